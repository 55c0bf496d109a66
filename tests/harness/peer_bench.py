"""Asynchronous peer-memory partitions (f2, csrc/peer_impl.cuh) on ONE B200:
BFS and PageRank on RMAT-<scale> (permuted ids) split into P partitions that
run as one persistent kernel.  All partitions share the SMs and HBM, so this
measures the protocol's overhead (remote pushes, summed termination), not
multi-GPU scaling.  Not the product path; parity is in tests/test_peer.py.

usage: python tests/harness/peer_bench.py [--scale 22] [--runs 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_2112_00132_b200 as atos  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--oracle", action="store_true")
a = ap.parse_args()
g = gg.rmat(a.scale, 16, seed=1, perm_seed=7)
src = int(np.argmax(np.diff(g.off)))  # the hub (ids are permuted)
deg = g.degrees()
xo = do = None
if a.oracle:
    import oracle
    do = oracle.bfs(g, src)
    xo = oracle.pagerank(g, 0.85)[0]
print(f"RMAT-{a.scale} permuted: n={g.n} m={g.m}")
print("| path | P | app | ms (median) | kernel ms | pops | edges | GTEPS | parity |")
print("|---|---|---|---|---|---|---|---|---|")
single = atos.Graph(g.off, g.col)
cases = [("single-partition warp workers", 1, single, dict(worker="warp", fetch_size=32)),
         ("single-partition CTA workers (bench config)", 1, single, dict())]
for P in (1, 2, 4, 8):
    cases.append((f"peer (f2)", P, atos.Graph.peer(g.off, g.col, P), dict(fetch_size=32)))
for name, P, Gx, kw in cases:
    for app in ("bfs", "pr"):
        ms, kms, st, out = [], [], None, None
        for _ in range(a.runs):
            if app == "bfs":
                out, st = atos.bfs(Gx, src, timeout_s=120, **kw)
            else:
                kw2 = dict(kw)
                if "worker" not in kw2 and P == 1 and name.startswith("single-partition CTA"):
                    kw2.update(fetch_size=128, cta_threads=1024)
                out, st = atos.pagerank(Gx, 0.85, 1e-6, timeout_s=120, **kw2)
            ms.append(st["ms"])
            kms.append(st["kernel_ms"])
        med, kmed = float(np.median(ms)), float(np.median(kms))
        if app == "bfs":
            e = int(deg[out != atos.UNREACHED].sum())
            par = "exact" if do is not None and np.array_equal(out, do) else ("-" if do is None else "MISMATCH")
        else:
            e = st["edges_processed"]
            par = f"{np.max(np.abs(out - xo)) / xo.max():.1e}" if xo is not None else "-"
        print(f"| {name} | {P} | {app} | {med:.2f} | {kmed:.2f} | {st['tasks_popped']} | {e} | "
              f"{e / kmed / 1e6:.1f} | {par} |", flush=True)

"""PageRank variant comparison on RMAT-<scale> (tuning experiments; not the product path).

Runs atos.pagerank through the C ABI for each named configuration, L2 flushed
before every run, and prints one markdown row per variant: median ms, pops,
pushes, edge pushes, GTEPS_raw, L_inf/max vs the fp64 Jacobi oracle (computed
once on all host cores; the oracle is test infrastructure)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import graphgen as gg
import paper_2112_00132_b200 as atos

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--variants", default='{"base": {}}', help="JSON {name: Config kwargs}")
ap.add_argument("--no-oracle", action="store_true")
ap.add_argument("--app", default="pr", choices=["pr", "bfs"])
a = ap.parse_args()
variants = json.loads(a.variants)
g = gg.rmat(a.scale, 16, seed=1)
G = atos.Graph(g.off, g.col)
dev = torch.device("cuda", 0)
out = torch.empty(g.n, dtype=torch.float32, device=dev)
flush = torch.empty(512 << 18, dtype=torch.float32, device=dev)
x = None
if not a.no_oracle:
    import oracle
    x = oracle.pagerank(g, 0.85)[0] if a.app == "pr" else oracle.bfs(g, 0)
print(f"RMAT-{a.scale}: n={g.n} m={g.m} app={a.app}")
if a.app == "bfs":
    out = torch.empty(g.n, dtype=torch.int32, device=dev)
print("| variant | ms (median) | pops | pushed | edge pushes | GTEPS_raw | Linf/max |")
print("|---|---|---|---|---|---|---|")
for name, kw in variants.items():
    base = dict(fetch_size=128, cta_threads=512 if a.app == "pr" else 256, timeout_s=120)
    base.update(kw)
    ms, st = [], None
    for _ in range(a.runs):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        if a.app == "pr":
            _, st = atos.pagerank(G, 0.85, 1e-6, out=out, **base)
        else:
            _, st = atos.bfs(G, 0, out=out, **base)
        ms.append(st["ms"])
    err = float("nan")
    if x is not None:
        if a.app == "pr":
            err = float(np.max(np.abs(out.cpu().numpy().astype(np.float64) - x)) / x.max())
        else:
            err = float(np.sum(out.cpu().numpy().view(np.uint32) != x))  # mismatching depths
    med = float(np.median(ms))
    print(f"| {name} | {med:.2f} | {st['tasks_popped']} | {st['tasks_pushed']} | {st['edges_processed']} | "
          f"{st['edges_processed'] / med / 1e6:.1f} | {err:.2e} |", flush=True)

"""PageRank fp32-residue precision vs time (experiments; DESIGN R34).

For the library selected by ATOS_LIB (default: the product build): RMAT-24
PageRank time and edge pushes (persistent CTA, bench config), and the L_inf
error (relative to max rank) of fp32-residue runs against an fp64-residue
run of the same library on the graphs where fp32 rounding bit before R34:
RMAT-16 with thread workers at FETCH 256 and the 40,001-vertex fan-in hub.
usage: ATOS_LIB=... python tools/pr_precision.py TAG
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import graphgen as gg  # noqa: E402
import paper_2112_00132_b200 as atos  # noqa: E402


def fan_in(k=40000, fan=64):
    e = [(s, 0) for s in range(1, k + 1)] + [(s, s + 1) for s in range(1, k)] + [(0, j) for j in range(1, fan + 1)]
    return gg.from_edges(k + 1, e)


def err(G, **kw):
    ref, _ = atos.pagerank(G, 0.85, 1e-6, pr_residue_fp64=True, **kw)
    r, st = atos.pagerank(G, 0.85, 1e-6, **kw)
    return float(np.max(np.abs(r.astype(np.float64) - ref)) / ref.max()), st["max_residue"]


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "product"
    out = {"tag": tag, "lib": atos.LIB_PATH}
    g16 = atos.Graph.from_csr(gg.rmat(16, 16, seed=1))
    out["rmat16_thread_f256"] = err(g16, worker="thread", fetch_size=256)
    out["rmat16_cta_f128"] = err(g16, fetch_size=128, cta_threads=1024)
    gf = atos.Graph.from_csr(fan_in())
    out["fanin_cta_f32"] = err(gf, fetch_size=32)
    out["fanin_thread_f256"] = err(gf, worker="thread", fetch_size=256)
    g = gg.rmat(24, 16, seed=1)
    G = atos.Graph(g.off, g.col)
    runs = []
    for i in range(4):
        r, st = atos.pagerank(G, 0.85, 1e-6, fetch_size=128, cta_threads=1024, timeout_s=120)
        if i:
            runs.append((st["kernel_ms"], st["ms"], st["edges_processed"], st["tasks_popped"], st["kernel_launches"]))
    out["rmat24"] = {"kernel_ms": float(np.median([x[0] for x in runs])), "ms": float(np.median([x[1] for x in runs])),
                     "pushes": int(np.median([x[2] for x in runs])), "pops": int(np.median([x[3] for x in runs])),
                     "launches": runs[-1][4]}
    if os.environ.get("PR_FP64"):
        ks = []
        for i in range(3):
            r, st = atos.pagerank(G, 0.85, 1e-6, fetch_size=128, cta_threads=1024, timeout_s=120, pr_residue_fp64=True)
            if i:
                ks.append((st["kernel_ms"], st["edges_processed"]))
        out["rmat24_fp64"] = {"kernel_ms": float(np.median([k[0] for k in ks])), "pushes": int(ks[-1][1])}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

"""High-diameter BFS latency: per-hop time
on the 4899x4899 grid (ecc. 9,796) and the 64x64 grid, persistent CTA
workers, for the product library or a variant (ATOS_LIB).  Not the product path.

usage: python tools/grid_latency.py [--runs 3] [--cells cta:256:128,...]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_2112_00132_b200 as atos  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--cells", default="cta:256:128,cta:128:16,cta:64:4")
ap.add_argument("--big", type=int, default=4899)
a = ap.parse_args()
cells = [(c.split(":")[0], int(c.split(":")[1]), int(c.split(":")[2])) for c in a.cells.split(",")]
print("| graph | worker | T | F | ms (median) | us / hop | pops / reached |")
print("|---|---|---|---|---|---|---|")
for name, g in [(f"grid {a.big}x{a.big}", gg.grid(a.big, a.big)), ("grid 64x64", gg.grid(64, 64))]:
    G = atos.Graph.from_csr(g)
    hops = 2 * (int(round(np.sqrt(g.n))) - 1)
    for w, t, f in cells:
        ms, st = [], None
        for _ in range(a.runs):
            d, st = atos.bfs(G, 0, worker=w, cta_threads=t, fetch_size=f, timeout_s=300)
            ms.append(st["ms"])
        assert int(d.max()) == hops
        med = float(np.median(ms))
        print(f"| {name} | {w} | {t} | {f} | {med:.2f} | {med * 1e3 / hops:.2f} | {st['tasks_popped'] / g.n:.3f} |",
              flush=True)

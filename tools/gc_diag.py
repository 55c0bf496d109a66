"""Colouring strategy diagnostic: persistent vs discrete
vs BSP x worker on a symmetrised RMAT graph — ms, rounds, tasks, colours and
per-round time, so the BSP/discrete numbers can be explained rather than
quoted.  Prints one markdown row per cell.  Not the product path.

usage: python tools/gc_diag.py [--scale 20] [--runs 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_2112_00132_b200 as atos  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--cells", default="")
a = ap.parse_args()
g = gg.rmat(a.scale, 16, seed=1, symmetrize=True)
G = atos.Graph.from_csr(g, symmetric=True)
out = torch.empty(g.n, dtype=torch.int32, device="cuda")
print(f"RMAT-{a.scale} symmetrised: n={g.n} m={g.m} max degree={int(np.diff(g.off).max())}")
print("| kernel | worker | F | ms (median) | rounds | ms / round | tasks popped | tasks / 2n | colours |")
print("|---|---|---|---|---|---|---|---|---|")
cells = [(k, w, f) for k in ("persistent", "discrete", "bsp") for w in ("thread", "warp", "cta") for f in (32, 128)]
if a.cells:
    cells = [tuple(c.split(":")[:2]) + (int(c.split(":")[2]),) for c in a.cells.split(",")]
for k, w, f in cells:
    ms, st, nc = [], None, 0
    for _ in range(a.runs):
        _, nc, st = atos.color(G, out=out, kernel=k, worker=w, fetch_size=f, cta_threads=256, timeout_s=120)
        ms.append(st["ms"])
    med = float(np.median(ms))
    r = max(1, st["rounds"])
    print(f"| {k} | {w} | {f} | {med:.2f} | {st['rounds']} | {med / r:.3f} | {st['tasks_popped']} | "
          f"{st['tasks_popped'] / (2 * g.n):.2f} | {nc} |", flush=True)

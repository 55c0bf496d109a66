"""Run one app a few times on RMAT-<scale> for ncu captures (not a benchmark)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import graphgen as gg
import paper_2112_00132_b200 as atos

ap = argparse.ArgumentParser()
ap.add_argument("--app", default="bfs")
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--ef", type=int, default=16)
ap.add_argument("--grid", type=int, default=0)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--worker", default="cta")
ap.add_argument("--kernel", default="persistent")
ap.add_argument("--fetch", type=int, default=256)
ap.add_argument("--threads", type=int, default=256)
ap.add_argument("--filter", type=int, default=1)
ap.add_argument("--window", type=int, default=0)
ap.add_argument("--check", type=int, default=8)
a = ap.parse_args()
g = gg.grid(a.grid, a.grid) if a.grid else gg.rmat(a.scale, a.ef, seed=1, symmetrize=(a.app == "color"))
G = atos.Graph.from_csr(g, symmetric=(a.app == "color"))
cfg = atos.Config(kernel=a.kernel, worker=a.worker, fetch_size=a.fetch, cta_threads=a.threads, bfs_filter=bool(a.filter), timeout_s=300, pr_activation=a.window, check_size=a.check)
for i in range(a.iters):
    if a.app == "bfs":
        d, st = atos.bfs(G, 0, cfg)
    elif a.app == "pr":
        d, st = atos.pagerank(G, 0.85, 1e-6, cfg)
    else:
        d, k, st = atos.color(G, cfg)
    print(a.app, {k: (round(v, 3) if isinstance(v, float) else v) for k, v in st.items()}, flush=True)

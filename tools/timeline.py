"""Timeline of one run (device trace): edges / items per time bucket."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import graphgen as gg
import paper_2112_00132_b200 as atos

ap = argparse.ArgumentParser()
ap.add_argument("--app", default="bfs")
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--grid", type=int, default=0)
ap.add_argument("--fetch", type=int, default=256)
ap.add_argument("--threads", type=int, default=256)
ap.add_argument("--worker", default="cta")
ap.add_argument("--buckets", type=int, default=40)
a = ap.parse_args()
g = gg.grid(a.grid, a.grid) if a.grid else gg.rmat(a.scale, 16, seed=1)
G = atos.Graph.from_csr(g)
tr = atos.Trace(1 << 22)
cfg = atos.Config(worker=a.worker, fetch_size=a.fetch, cta_threads=a.threads, trace=tr, timeout_s=300)
for it in range(2):
    if a.app == "bfs":
        _, st = atos.bfs(G, 0, cfg)
    else:
        _, st = atos.pagerank(G, 0.85, 1e-6, cfg)
r = tr.records(st)
t = (r["t_ns"] - r["t_ns"][0]) / 1e3
print(f"{a.app} ms={st['ms']:.3f} kernel_ms={st['kernel_ms']:.3f} records={len(r)} span_us={t[-1]:.1f} "
      f"items={int(r['items'].sum())} edges={int(r['edges'].astype(np.int64).sum())}")
edges_b = np.linspace(0, t[-1] + 1e-9, a.buckets + 1)
idx = np.clip(np.searchsorted(edges_b, t, side="right") - 1, 0, a.buckets - 1)
for b in range(a.buckets):
    m = idx == b
    print(f"{edges_b[b]:9.1f}us batches={int(m.sum()):6d} items={int(r['items'][m].sum()):9d} "
          f"edges={int(r['edges'][m].astype(np.int64).sum()):11d} sms={len(np.unique(r['sm'][m])):3d}")

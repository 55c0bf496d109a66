"""Compare single-GPU vs partitioned (world=1) work counters on RMAT-<scale>."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, graphgen as gg
import paper_2112_00132_b200 as atos
from paper_2112_00132_b200 import dist as adist
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g, fwd = gg.permute(gg.rmat(scale, 16, seed=1), 12345)
G = atos.Graph.from_csr(g)
for it in range(2):
    r, st = atos.pagerank(G, 0.85, 1e-6)
    print("single", {k: st[k] for k in ("ms", "tasks_popped", "edges_processed", "chunk_tasks")})
pg = adist.PartGraph.from_global(g, 1, 0)
for it in range(2):
    r2, st2 = adist.pagerank(pg, 0.85, 1e-6)
    print("part1 ", {k: st2[k] for k in ("ms", "tasks_popped", "edges_processed", "chunk_tasks", "rounds")})
print("maxdiff", float(np.max(np.abs(r - r2))))
for k in ("persistent", "discrete"):
    for it in range(2):
        r3, st3 = adist.pagerank(pg, 0.85, 1e-6, kernel=k)
        print("part1", k, {kk: st3[kk] for kk in ("ms", "tasks_popped", "edges_processed", "rounds")})

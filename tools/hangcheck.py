import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, graphgen as gg, paper_2112_00132_b200 as atos
app, scale = sys.argv[1], int(sys.argv[2])
g = gg.rmat(scale, 16, seed=1)
G = atos.Graph.from_csr(g)
for it in range(3):
    try:
        if app == "pr":
            r, st = atos.pagerank(G, 0.85, 1e-6, timeout_s=10)
        else:
            r, st = atos.bfs(G, 0, timeout_s=10)
        print(app, scale, it, "ok", st["ms"], st["tasks_popped"], st["chunk_tasks"], flush=True)
    except Exception as e:
        print(app, scale, it, "ERR", e, flush=True)

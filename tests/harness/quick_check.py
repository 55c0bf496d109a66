"""Quick parity smoke of a library variant (ATOS_LIB) on small graphs before
timing it: BFS exact, PageRank within 1e-4, colouring valid.  Not a test."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import graphgen as gg  # noqa: E402
import oracle  # noqa: E402
import paper_2112_00132_b200 as atos  # noqa: E402

for scale in (12, 16):
    g = gg.rmat(scale, 16, seed=1)
    G = atos.Graph.from_csr(g)
    for t in (256, 1024):
        d, _ = atos.bfs(G, 0, cta_threads=t, fetch_size=128, timeout_s=20)
        assert np.array_equal(d, oracle.bfs(g, 0)), ("bfs", scale, t)
        r, st = atos.pagerank(G, 0.85, 1e-6, cta_threads=t, fetch_size=128, timeout_s=20)
        x = oracle.pagerank(g, 0.85)[0]
        err = float(np.max(np.abs(r - x)) / x.max())
        assert err <= 1e-4 and st["max_residue"] <= 1e-6, ("pr", scale, t, err)
g = gg.grid(300, 300)
d, _ = atos.bfs(atos.Graph.from_csr(g), 0, timeout_s=20)
i, j = np.divmod(np.arange(g.n), 300)
assert np.array_equal(d.astype(np.int64), i + j)
print("quick_check ok", os.environ.get("ATOS_LIB", "product"))

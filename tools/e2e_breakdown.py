"""Break the bench's e2e step (public API from pinned host buffers) into its
parts: atos_graph_create (alloc + H2D + checks), atos_bfs, atos_pagerank (each
including its D2H of the result), atos_graph_destroy.  RMAT-24 as in bench.py.
Usage: python tools/e2e_breakdown.py [--iters 5]"""
import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--again", action="store_true", help="also time a second BFS on the same handle (warm workspace)")
    a = ap.parse_args()
    import torch
    import graphgen as gg
    import paper_2112_00132_b200 as atos
    g = gg.rmat(a.scale, 16, seed=1)
    off = torch.from_numpy(g.off).pin_memory()
    col = torch.from_numpy(g.col).pin_memory()
    depth = torch.empty(g.n, dtype=torch.int32).pin_memory()
    rk = torch.empty(g.n, dtype=torch.float32).pin_memory()
    cb = atos.Config(kernel="persistent", worker="cta", fetch_size=128, cta_threads=256, timeout_s=120)
    cp = atos.Config(kernel="persistent", worker="cta", fetch_size=128, cta_threads=1024, timeout_s=120)
    rows = []
    for i in range(a.iters):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        G = atos.Graph(off.numpy(), col.numpy())
        t1 = time.perf_counter()
        _, s1 = atos.bfs(G, 0, cb, out=depth.numpy().view("uint32"))
        t2 = time.perf_counter()
        if a.again:
            _, s2 = atos.bfs(G, 0, cb, out=depth.numpy().view("uint32"))
            tb = time.perf_counter()
            print("  bfs first: wall %.1f ms, device %.2f ms (kernel %.2f); again: wall %.1f ms, device %.2f ms (kernel %.2f)"
                  % ((t2 - t1) * 1e3, s1["ms"], s1["kernel_ms"], (tb - t2) * 1e3, s2["ms"], s2["kernel_ms"]), flush=True)
            t1 += time.perf_counter() - t2  # the bfs column keeps the first call only
            t2 = time.perf_counter()
        atos.pagerank(G, 0.85, 1e-6, cp, out=rk.numpy())
        t3 = time.perf_counter()
        G.close()
        t4 = time.perf_counter()
        rows.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3))
        print("iter %d: create %.1f ms  bfs %.1f ms  pagerank %.1f ms  destroy %.1f ms" %
              tuple([i] + [x * 1e3 for x in rows[-1]]), flush=True)
    med = [statistics.median(r[k] for r in rows[1:] or rows) * 1e3 for k in range(4)]
    print("median (iters 1..): create %.1f  bfs %.1f  pagerank %.1f  destroy %.1f ms; H2D %.2f GB" %
          (*med, (g.off.nbytes + g.col.nbytes) / 1e9))


if __name__ == "__main__":
    main()

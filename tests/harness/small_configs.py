"""BASELINE configs[0] (C1) and configs[1] (C2) on one B200, with parity beside each
number (the oracle is test infrastructure; this tool is a measurement driver, not the
product path).  Prints a markdown report.

C1: BFS from 0 on the 64x64 grid — device time, per-hop latency (t / eccentricity 126),
    bit-exact vs oracle and vs Manhattan distance; the same per-hop latency on a
    10^4-vertex path graph.
C2: RMAT-16 (ef 16, seed 1): PageRank alpha=.85 eps=1e-6 (ms, GTEPS_raw, GTEPS_norm =
    BSP-push edge pushes / t, L_inf/max vs fp64 Jacobi, max residue) and greedy
    colouring on the symmetrised graph (ms, colours vs ID-order first fit, overwork =
    tasks / 2n, validity).
"""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import graphgen as gg
import oracle
import paper_2112_00132_b200 as atos

REPS = 20


def med(f):
    out = [f() for _ in range(REPS + 1)][1:]
    return statistics.median(o[1]["ms"] for o in out), out[-1]


print("# Small configs (BASELINE configs[0], configs[1]) on one B200\n")
print("Device time = library CUDA events (init + run), median of 20 after 1 warm-up.\n")
# ---------------- C1
g = gg.grid(64, 64)
G = atos.Graph.from_csr(g)
ref = oracle.bfs(g, 0)
ij = np.add.outer(np.arange(64), np.arange(64)).ravel().astype(np.uint32)
print("## C1: BFS on grid 64x64 from vertex 0 (ecc 126)\n")
print("| worker | kernel | F | us | per-hop us | bit-exact vs oracle | == i+j |\n|---|---|---|---|---|---|---|")
for w, k, f, t in [("cta", "persistent", 128, 256), ("cta", "persistent", 16, 64), ("warp", "persistent", 4, 256),
                   ("thread", "persistent", 1, 256), ("cta", "discrete", 128, 256), ("cta", "bsp", 128, 256)]:
    ms, (d, st) = med(lambda: atos.bfs(G, 0, worker=w, kernel=k, fetch_size=f, cta_threads=t))
    print(f"| {w} | {k} | {f} | {ms*1e3:.1f} | {ms*1e3/126:.2f} | {np.array_equal(d, ref)} | {np.array_equal(d, ij)} |")
p = gg.path(10000)
P = atos.Graph.from_csr(p)
print("\nPath graph, 10,000 vertices, BFS from 0 (9,999 hops):\n")
print("| worker | F | ms | per-hop us | depth == index |\n|---|---|---|---|---|")
for w, f, t in [("cta", 128, 256), ("cta", 16, 64), ("warp", 4, 256), ("thread", 1, 256)]:
    ms, (d, st) = med(lambda: atos.bfs(P, 0, worker=w, fetch_size=f, cta_threads=t))
    print(f"| {w} | {f} | {ms:.2f} | {ms*1e3/9999:.2f} | {np.array_equal(d, np.arange(10000, dtype=np.uint32))} |")

# ---------------- C2 PageRank
r16 = gg.rmat(16, 16, seed=1)
R = atos.Graph.from_csr(r16)
x, it = oracle.pagerank(r16, 0.85)
_, bsp = atos.pagerank(R, 0.85, 1e-6, kernel="bsp")
norm_pushes = bsp["edges_processed"]
print(f"\n## C2: PageRank on RMAT-16 (n={r16.n}, m={r16.m}), alpha 0.85, eps 1e-6\n")
print(f"fp64 Jacobi oracle: {it} iterations to 1e-10.  GTEPS_norm uses the BSP-push run's "
      f"{norm_pushes} edge pushes (SURVEY §8d).\n")
print("| kernel | worker | F | ms | edge pushes | GTEPS_raw | GTEPS_norm | L_inf/max vs Jacobi | max residue |\n"
      "|---|---|---|---|---|---|---|---|---|")
for k, w, f, t in [("persistent", "cta", 128, 512), ("persistent", "cta", 32, 256), ("persistent", "warp", 8, 256),
                   ("discrete", "cta", 128, 256), ("bsp", "cta", 128, 256)]:
    ms, (r, st) = med(lambda: atos.pagerank(R, 0.85, 1e-6, kernel=k, worker=w, fetch_size=f, cta_threads=t))
    err = float(np.max(np.abs(r - x)) / x.max())
    e = st["edges_processed"]
    print(f"| {k} | {w} | {f} | {ms:.3f} | {e} | {e/ms/1e6:.1f} | {norm_pushes/ms/1e6:.1f} | {err:.2e} | {st['max_residue']:.2e} |")

# ---------------- C2 colouring
s16 = gg.rmat(16, 16, seed=1, symmetrize=True)
S = atos.Graph.from_csr(s16, symmetric=True)
oc, ok_n = oracle.greedy_color(s16)
print(f"\n## C2: greedy colouring on symmetrised RMAT-16 (n={s16.n}, m={s16.m}, max degree {int(s16.degrees().max())})\n")
print(f"Serial ID-order first fit (oracle): {ok_n} colours.\n")
print("| kernel | worker | F | ms | colours | overwork (tasks/2n) | monochromatic edges |\n|---|---|---|---|---|---|---|")
for k, w, f, t in [("persistent", "cta", 128, 256), ("persistent", "warp", 8, 256), ("discrete", "warp", 8, 256),
                   ("bsp", "cta", 128, 256)]:
    out = [atos.color(S, kernel=k, worker=w, fetch_size=f, cta_threads=t) for _ in range(REPS + 1)][1:]
    ms = statistics.median(o[2]["ms"] for o in out)
    c, kk, st = out[-1]
    bad, _ = oracle.check_coloring(s16, c)
    print(f"| {k} | {w} | {f} | {ms:.3f} | {kk} | {st['tasks_popped']/(2*s16.n):.2f} | {bad} |")

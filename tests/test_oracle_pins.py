"""Pins for the CPU oracle (runs with -m "not gpu").

The oracle (oracle/oracle.c) is checked against things other than itself:
closed forms, brute force on tiny inputs, a numpy dense linear solve, golden
fixtures from SPEC.md worked examples, and invariants — chosen so that a
dropped term, a wrong sign/index or a transposed operand fails one of them.
"""
import itertools
import os

import numpy as np
import pytest

import graphgen as gg
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
U = oracle.UNREACHED


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


# ------------------------------------------------------------------ BFS ---

def test_bfs_golden_path():
    rows = _rows("bfs_grid_1x5.txt")
    r, c, s = map(int, rows[0])
    g = gg.grid(r, c)
    assert oracle.bfs(g, s).tolist() == [int(x) for x in rows[1]]


def test_bfs_grid_manhattan():
    g = gg.grid(64, 64)
    d = oracle.bfs(g, 0)
    i, j = np.divmod(np.arange(64 * 64), 64)
    assert np.array_equal(d, (i + j).astype(np.uint32))
    assert d.max() == 126
    # from an interior source: |i-i0| + |j-j0|
    src = 37 * 64 + 11
    d = oracle.bfs(g, src)
    assert np.array_equal(d, (np.abs(i - 37) + np.abs(j - 11)).astype(np.uint32))


def test_bfs_small_closed_forms():
    assert oracle.bfs(gg.path(10), 0).tolist() == list(range(10))
    assert oracle.bfs(gg.path(10), 9).tolist() == list(range(9, -1, -1))
    st = gg.star(7)
    assert oracle.bfs(st, 0).tolist() == [0] + [1] * 7
    assert oracle.bfs(st, 3).tolist() == [1, 2, 2, 0, 2, 2, 2, 2]
    assert oracle.bfs(gg.complete(6), 2).tolist() == [1, 1, 0, 1, 1, 1]
    ch = gg.directed_chain(5)
    assert oracle.bfs(ch, 2).tolist() == [U, U, 0, 1, 2]
    e = gg.empty(4)
    assert oracle.bfs(e, 1).tolist() == [U, 0, U, U]


def _floyd_hops(g):
    n = g.n
    inf = 10 ** 9
    D = np.full((n, n), inf, dtype=np.int64)
    np.fill_diagonal(D, 0)
    for v in range(n):
        for w in g.col[g.off[v]:g.off[v + 1]]:
            D[v, w] = min(D[v, w], 1)
    for k in range(n):
        D = np.minimum(D, D[:, k:k + 1] + D[k:k + 1, :])
    return D, inf


def test_bfs_brute_force_floyd_warshall():
    rng = np.random.default_rng(7)
    for t in range(300):
        n = int(rng.integers(1, 13))
        g = gg.random_digraph(n, float(rng.uniform(0.05, 0.5)), seed=t)
        D, inf = _floyd_hops(g)
        for s in range(n):
            d = oracle.bfs(g, s).astype(np.int64)
            exp = np.where(D[s] >= inf, U, D[s])
            assert np.array_equal(d, exp), (t, s)


def test_bfs_permutation_invariance():
    g = gg.rmat(10, 8, seed=3)
    gp, fwd = gg.permute(g, 99)
    d0 = oracle.bfs(g, 0)
    d1 = oracle.bfs(gp, int(fwd[0]))
    assert np.array_equal(np.sort(d0), np.sort(d1))
    assert np.array_equal(d1[fwd], d0)


def test_bfs_validator_catches_corruption():
    g = gg.rmat(10, 8, seed=4)
    d = oracle.bfs(g, 0)
    assert oracle.check_bfs(g, 0, d) == 0
    reach = np.nonzero((d != U) & (d > 0))[0]
    bad = d.copy()
    bad[reach[5]] += 1
    assert oracle.check_bfs(g, 0, bad) > 0
    bad = d.copy()
    bad[reach[7]] -= 1
    assert oracle.check_bfs(g, 0, bad) > 0
    unr = np.nonzero(d == U)[0]
    if len(unr):
        bad = d.copy()
        bad[unr[0]] = 3
        assert oracle.check_bfs(g, 0, bad) > 0


# ------------------------------------------------------------- PageRank ---

def _graph_by_name(name, k):
    return {"star": lambda: gg.star(k), "chain": lambda: gg.directed_chain(k),
            "complete": lambda: gg.complete(k), "dcycle": lambda: gg.cycle(k, directed=True)}[name]()


def test_pagerank_closed_forms_golden():
    for name, k, a, v, exp in _rows("pagerank_closed_forms.txt"):
        g = _graph_by_name(name, int(k))
        x, _ = oracle.pagerank(g, float(a), tol=1e-15, max_iter=100000)
        assert abs(x[int(v)] - float(exp)) <= 1e-9 * max(1.0, float(exp)), (name, k, v, x[int(v)], exp)


@pytest.mark.parametrize("k", [1, 2, 5, 40])
def test_pagerank_star_all_leaves(k):
    a = 0.85
    x, _ = oracle.pagerank(gg.star(k), a, tol=1e-15, max_iter=100000)
    assert abs(x[0] - (1 + a * k) / (1 + a)) < 1e-9
    assert np.allclose(x[1:], (1 + a / k) / (1 + a), rtol=0, atol=1e-9)


def _dense_pagerank(g, a):
    n = g.n
    P = np.zeros((n, n))
    deg = g.degrees()
    for v in range(n):
        for w in g.col[g.off[v]:g.off[v + 1]]:
            P[w, v] += 1.0 / deg[v]
    return np.linalg.solve(np.eye(n) - a * P, np.full(n, 1 - a)), P


def test_pagerank_dense_solve():
    rng = np.random.default_rng(11)
    for t in range(60):
        n = int(rng.integers(1, 65))
        g = gg.random_digraph(n, float(rng.uniform(0.02, 0.3)), seed=1000 + t)
        a = float(rng.uniform(0.3, 0.95))
        x, _ = oracle.pagerank(g, a, tol=1e-14, max_iter=100000)
        xs, _ = _dense_pagerank(g, a)
        assert np.max(np.abs(x - xs)) <= 1e-9 * max(1.0, xs.max()), t


def test_pagerank_no_dangling_sums_to_n():
    g = gg.rmat(9, 8, seed=5, symmetrize=True)
    keep = g.degrees() > 0
    # isolated vertices have x = 1-a exactly; others: sum over a strongly-connected-free
    # symmetric graph with no dangling vertex -> total mass n
    x, _ = oracle.pagerank(g, 0.85, tol=1e-14, max_iter=100000)
    assert np.allclose(x[~keep], 0.15)
    assert abs(x.sum() - (keep.sum() + 0.15 * (~keep).sum())) < 1e-7 * g.n


def test_pagerank_thread_count_bit_identical():
    g = gg.rmat(12, 16, seed=2)
    x1, i1 = oracle.pagerank(g, 0.85, threads=1)
    x4, i4 = oracle.pagerank(g, 0.85, threads=4)
    assert i1 == i4 and np.array_equal(x1, x4)


def test_pagerank_push_bound_and_conservation():
    """Serial push PR (Alg. 4 with one worker): all residues <= eps at the end,
    0 <= x* - rank <= eps x*/(1-a) (P:525-540 with R4/R6), and the invariant
    rank + (I - aP)^{-1} residue = x* (reading R4 makes it hold at start)."""
    rng = np.random.default_rng(3)
    for t in range(25):
        n = int(rng.integers(2, 50))
        g = gg.random_digraph(n, float(rng.uniform(0.03, 0.3)), seed=500 + t)
        a, eps = 0.85, 1e-5
        r, s, pops, pushes = oracle.pagerank_push(g, a, eps)
        xs, P = _dense_pagerank(g, a)
        assert s.max() <= eps
        diff = xs - r
        assert diff.min() >= -1e-12
        assert np.all(diff <= eps * xs / (1 - a) + 1e-12)
        inv = r + np.linalg.solve(np.eye(n) - a * P, s)
        assert np.max(np.abs(inv - xs)) < 1e-10
        assert pops >= n


def test_pagerank_push_two_cycle_symmetric():
    # SPEC.md S:363 2-cycle: the fixed point is x = (1, 1); a serial (asynchronous-order)
    # push run is not symmetric (that is a BSP property) but each rank is within the
    # eps*x*/(1-a) bound below x*.
    g = gg.cycle(2, directed=True)
    r, s, _, _ = oracle.pagerank_push(g, 0.85, 1e-6)
    assert np.all(r <= 1.0 + 1e-15) and np.all(1.0 - r <= 1e-6 / 0.15)
    x, _ = oracle.pagerank(g, 0.85)
    assert np.allclose(x, 1.0)


def test_pagerank_push_rmat_vs_jacobi():
    g = gg.rmat(11, 16, seed=1)
    x, _ = oracle.pagerank(g, 0.85)
    r, s, _, pushes = oracle.pagerank_push(g, 0.85, 1e-6)
    assert np.max(np.abs(x - r)) <= 1e-6 / 0.15 * x.max()
    assert pushes > g.m


# ------------------------------------------------------------ colouring ---

def _crown(k):
    # u_i = 2i, v_i = 2i+1, edge u_i - v_j iff i != j
    e = [(2 * i, 2 * j + 1) for i in range(k) for j in range(k) if i != j]
    return gg.from_edges(2 * k, e, symmetrize=True)


def _graph_color(name, k):
    return {"complete": lambda: gg.complete(k), "edgeless": lambda: gg.empty(k),
            "cycle": lambda: gg.cycle(k), "crown": lambda: _crown(k), "grid": lambda: gg.grid(k, k)}[name]()


def test_coloring_golden_counts():
    for name, k, exp in _rows("coloring_small.txt"):
        g = _graph_color(name, int(k))
        c, nc = oracle.greedy_color(g)
        assert nc == int(exp), (name, k, nc)
        bad, nc2 = oracle.check_coloring(g, c)
        assert bad == 0 and nc2 == nc


def test_coloring_grid_parity_closed_form():
    g = gg.grid(64, 64)
    c, _ = oracle.greedy_color(g)
    i, j = np.divmod(np.arange(64 * 64), 64)
    assert np.array_equal(c, (i + j) % 2)


def _chromatic(g):
    n = g.n
    adj = [set(g.col[g.off[v]:g.off[v + 1]].tolist()) - {v} for v in range(n)]
    for k in range(1, n + 1):
        for assign in itertools.product(range(k), repeat=n):
            if all(assign[v] != assign[u] for v in range(n) for u in adj[v]):
                return k
    return n


def test_coloring_brute_force_chromatic_bound():
    rng = np.random.default_rng(5)
    for t in range(40):
        n = int(rng.integers(1, 8))
        g0 = gg.random_digraph(n, float(rng.uniform(0.1, 0.7)), seed=2000 + t)
        g = gg.from_edges(n, np.stack([np.repeat(np.arange(n), np.diff(g0.off)), g0.col], 1)
                          if g0.m else np.zeros((0, 2)), symmetrize=True)
        c, k = oracle.greedy_color(g)
        chi = _chromatic(g)
        assert oracle.check_coloring(g, c)[0] == 0
        assert chi <= k <= int(g.degrees().max(initial=0)) + 1


def test_coloring_validator_catches_conflict():
    g = gg.complete(3)
    bad, _ = oracle.check_coloring(g, np.array([0, 0, 1], dtype=np.int32))
    assert bad > 0
    bad, _ = oracle.check_coloring(g, np.array([0, 1, 2], dtype=np.int32))
    assert bad == 0
    # colour above deg(v) is out of range (palette <= deg+1 rule, R11)
    bad, _ = oracle.check_coloring(gg.path(3), np.array([0, 1, 5], dtype=np.int32))
    assert bad > 0


def test_coloring_rmat_palette_bound():
    g = gg.rmat(12, 16, seed=1, symmetrize=True)
    c, k = oracle.greedy_color(g)
    assert oracle.check_coloring(g, c)[0] == 0
    assert np.all(c <= g.degrees())

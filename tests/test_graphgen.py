"""Input generator checks (SPEC.md S:65-103 examples)."""
import os

import numpy as np

import graphgen as gg

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_grid_counts_golden():
    with open(os.path.join(GOLD, "grid_counts.txt")) as f:
        rows = [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]
    for r, c, n, m in rows:
        r, c, n, m = map(int, (r, c, n, m))
        assert r * c == n and 2 * (r * (c - 1) + c * (r - 1)) == m
        if n <= 1_000_000:
            g = gg.grid(r, c)
            assert (g.n, g.m) == (n, m)


def _check_csr(g):
    assert g.off[0] == 0 and g.off[-1] == g.m
    assert np.all(np.diff(g.off) >= 0)
    if g.m:
        assert g.col.min() >= 0 and g.col.max() < g.n
    for v in range(min(g.n, 2000)):
        row = g.col[g.off[v]:g.off[v + 1]]
        assert np.all(np.diff(row) > 0) and not np.any(row == v)


def test_rmat_deterministic_and_skewed():
    a = gg.rmat(14, 16, seed=1)
    b = gg.rmat(14, 16, seed=1)
    assert np.array_equal(a.off, b.off) and np.array_equal(a.col, b.col)
    _check_csr(a)
    deg = a.degrees()
    assert deg.max() >= 8 * deg.mean()
    c = gg.rmat(14, 16, seed=2)
    assert not np.array_equal(a.col[:1000], c.col[:1000])


def test_rmat_thread_count_independent():
    lib = gg._load()
    lib.gg_set_threads(1)
    a = gg.rmat(12, 16, seed=9, symmetrize=True)
    lib.gg_set_threads(4)
    b = gg.rmat(12, 16, seed=9, symmetrize=True)
    assert np.array_equal(a.off, b.off) and np.array_equal(a.col, b.col)


def test_symmetrize():
    g = gg.rmat(10, 8, seed=3, symmetrize=True)
    _check_csr(g)
    src = np.repeat(np.arange(g.n), g.degrees())
    fwd = set(zip(src.tolist(), g.col.tolist()))
    assert all((w, v) in fwd for v, w in fwd)


def test_permute_invariants():
    g = gg.rmat(10, 8, seed=3)
    p, fwd = gg.permute(g, 5)
    _check_csr(p)
    assert sorted(fwd.tolist()) == list(range(g.n))
    assert np.array_equal(np.sort(g.degrees()), np.sort(p.degrees()))
    assert np.array_equal(p.degrees()[fwd], g.degrees())


def test_road_like_grid_symmetric():
    g = gg.grid(50, 40, drop_prob=0.4, seed=3)
    _check_csr(g)
    assert 1.8 < g.m / g.n < 2.8
    src = np.repeat(np.arange(g.n), g.degrees())
    fwd = set(zip(src.tolist(), g.col.tolist()))
    assert all((w, v) in fwd for v, w in fwd)


def test_degenerate():
    g = gg.rmat(0, 1, seed=7)  # S:83 single vertex, self-loops dropped
    assert g.n == 1 and g.m == 0
    e = gg.empty(0)
    assert e.n == 0 and e.m == 0

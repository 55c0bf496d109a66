"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(SURVEY 8d C3/C4): RMAT-24 BFS bit-exact vs the serial oracle, PageRank within
1e-4 of max x* vs the multithreaded fp64 pull-Jacobi, colouring of the
symmetrised RMAT-24 checked exhaustively; the 4899x4899 grid against its closed
form depth = i + j.  The oracle is test infrastructure."""
import numpy as np
import pytest

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def atos():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2112_00132_b200 as m
    return m


@pytest.fixture(scope="module")
def rmat24():
    return gg.rmat(24, 16, seed=1)


def test_rmat24_bfs_bench_config(atos, rmat24):
    G = atos.Graph(rmat24.off, rmat24.col)
    d, st = atos.bfs(G, 0, kernel="persistent", worker="cta", fetch_size=128, cta_threads=256)
    exp = oracle.bfs(rmat24, 0)
    assert np.array_equal(d, exp), int(np.sum(d != exp))
    assert oracle.check_bfs(rmat24, 0, d) == 0


def test_rmat24_pagerank_bench_config(atos, rmat24):
    G = atos.Graph(rmat24.off, rmat24.col)
    r, st = atos.pagerank(G, 0.85, 1e-6, kernel="persistent", worker="cta", fetch_size=128, cta_threads=1024)
    x, _ = oracle.pagerank(rmat24, 0.85)
    err = float(np.max(np.abs(r.astype(np.float64) - x)) / x.max())
    assert err <= 1e-4, err
    assert st["max_residue"] <= 1e-6


def test_rmat24_color_bench_config(atos):
    s = gg.rmat(24, 16, seed=1, symmetrize=True)
    S = atos.Graph(s.off, s.col, symmetric=True)
    c, k, st = atos.color(S, kernel="persistent", worker="cta", fetch_size=128, cta_threads=256)
    bad, _ = oracle.check_coloring(s, c)
    assert bad == 0
    assert np.all(c >= 0) and np.all(c <= np.diff(s.off))  # palette <= deg + 1
    assert k == int(c.max()) + 1


def test_grid4899_bfs_closed_form(atos):
    n = 4899
    g = gg.grid(n, n)
    d, _ = atos.bfs(atos.Graph(g.off, g.col), 0, fetch_size=128, cta_threads=256)
    i, j = np.divmod(np.arange(n * n, dtype=np.int64), n)
    assert np.array_equal(d.astype(np.int64), i + j)
    assert int(d.max()) == 2 * (n - 1)

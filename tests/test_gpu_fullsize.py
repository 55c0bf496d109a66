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


@pytest.fixture(scope="module")
def rmat24_x(rmat24):
    return oracle.pagerank(rmat24, 0.85)[0]


@pytest.fixture(scope="module")
def rmat24_dev(atos, rmat24):
    return atos.Graph(rmat24.off, rmat24.col)


# bench config (R35 sweep-activated hubs, default), R34 threshold crossing at fp64 hubs,
# and the thread worker at FETCH 256 (the cell whose fp32 residues missed the gate in round 1)
@pytest.mark.parametrize("kw", [dict(worker="cta", fetch_size=128, cta_threads=1024),
                                dict(worker="cta", fetch_size=128, cta_threads=1024, pr_hub_check=0),
                                dict(worker="thread", fetch_size=256, cta_threads=256)],
                         ids=["bench", "hub_check0", "thread_f256"])
def test_rmat24_pagerank(atos, rmat24_dev, rmat24_x, kw):
    r, st = atos.pagerank(rmat24_dev, 0.85, 1e-6, kernel="persistent", timeout_s=120, **kw)
    x = rmat24_x
    err = float(np.max(np.abs(r.astype(np.float64) - x)) / x.max())
    assert err <= 1e-4, err
    assert st["max_residue"] <= 1e-6
    # one-sided bound 0 <= x* - rank (exact arithmetic), fp32 residue rounding allowance R36
    assert np.all(r <= x * (1 + 2048 * 2.0 ** -25) + 1e-6)


def test_fan_in_hub_full_size(atos):
    """A 2,000,000-way fan-in hub (every source of out-degree 2, equal pushes):
    the adversarial case for fp32 residues (R32), at RMAT-24-like size."""
    g = gg.fan_in(2_000_000)
    x = oracle.pagerank(g, 0.85)[0]
    G = atos.Graph(g.off, g.col)
    for kw in [dict(), dict(pr_hub_check=0), dict(worker="thread", fetch_size=256, cta_threads=256)]:
        r, st = atos.pagerank(G, 0.85, 1e-6, timeout_s=120, **kw)
        err = float(np.max(np.abs(r.astype(np.float64) - x)) / x.max())
        assert err <= 1e-4, (kw, err)
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

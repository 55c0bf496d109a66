"""Asynchronous peer-memory partitions (include/atos.h
atos_graph_create_peer): BFS and PageRank over P vertex
blocks with in-place remote atomics and remote queue pushes, no exchange
rounds.  On one GPU the P partitions run as one persistent kernel whose blocks
are split among them (the path a multi-GPU box runs as one kernel per device).
Parity against the oracle exactly as for the single-partition path: BFS
bit-exact, PageRank within 1e-4 of max x* with every residue <= eps."""
import numpy as np
import pytest

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu
PR_TOL = 1e-4
ONE_SIDED = 1 + 2.0 ** -30  # fp64 residues: < 2^20 adds per queue cycle x 2^-53 (R36)

_g = {}


def G(name):
    if name not in _g:
        _g[name] = {
            "rmat16": lambda: gg.rmat(16, 16, seed=1),
            "rmat16p": lambda: gg.rmat(16, 16, seed=1, perm_seed=7),
            "grid64": lambda: gg.grid(64, 64),
            "path": lambda: gg.path(3000),
            "star": lambda: gg.star(5000),
            "two": lambda: gg.from_edges(10, [(0, 1), (1, 2), (5, 6), (6, 7), (7, 8)]),
            "fanin": lambda: gg.fan_in(40000),
        }[name]()
    return _g[name]


@pytest.fixture(scope="module")
def atos():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2112_00132_b200 as m
    return m


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("gname,src", [("rmat16", 0), ("rmat16p", 11), ("grid64", 0), ("path", 1500), ("star", 3),
                                       ("two", 5)])
def test_peer_bfs_exact(atos, parts, gname, src):
    g = G(gname)
    P = atos.Graph.peer(g.off, g.col, parts)
    exp = oracle.bfs(g, src)
    for f in (1, 32):
        d, st = atos.bfs(P, src, fetch_size=f, timeout_s=60)
        assert np.array_equal(d, exp), (f, int(np.sum(d != exp)))
        assert st["tasks_popped"] >= 1


@pytest.mark.parametrize("parts", [1, 2, 4])
@pytest.mark.parametrize("gname", ["rmat16", "rmat16p", "grid64", "star", "fanin"])
def test_peer_pagerank(atos, parts, gname):
    g = G(gname)
    x = oracle.pagerank(g, 0.85)[0]
    P = atos.Graph.peer(g.off, g.col, parts)
    for f in (8, 64):
        r, st = atos.pagerank(P, 0.85, 1e-6, fetch_size=f, timeout_s=60)
        err = float(np.max(np.abs(r.astype(np.float64) - x)) / x.max())
        assert err <= PR_TOL, (f, err)
        assert st["max_residue"] <= 1e-6
        assert np.all(r <= x * ONE_SIDED + 1e-6)


def test_peer_remote_work_happens(atos):
    """With 4 blocks of an unpermuted RMAT graph most relaxations cross
    partitions: the run still pops each reached vertex about once."""
    g = G("rmat16p")
    P = atos.Graph.peer(g.off, g.col, 4)
    d, st = atos.bfs(P, 0, fetch_size=32, timeout_s=60)
    reached = int(np.sum(d != atos.UNREACHED))
    assert reached <= st["tasks_popped"] <= 2 * reached


def test_peer_errors(atos):
    g = G("grid64")
    for parts in (0, 9):
        with pytest.raises(atos.AtosError) as e:
            atos.Graph.peer(g.off, g.col, parts)
        assert e.value.name == "INVALID_ARGUMENT"
    small = G("two")
    d, _ = atos.bfs(atos.Graph.peer(small.off, small.col, 8), 0)  # n = 10 >= 8 parts: fine
    assert np.array_equal(d, oracle.bfs(small, 0))
    with pytest.raises(atos.AtosError) as e:
        atos.Graph.peer(np.array([0, 1], np.int64), np.array([0], np.int32), 2)  # n = 1 < parts
    assert e.value.name == "INVALID_ARGUMENT"
    with pytest.raises(atos.AtosError) as e:
        atos.Graph.peer(np.array([0, 1, 2], np.int64), np.array([1, 7], np.int32), 2, validate=True)
    assert e.value.name == "INVALID_GRAPH"
    with pytest.raises(atos.AtosError) as e:
        atos.Graph.peer(g.off, g.col, 2, devices=[0, 99])
    assert e.value.name == "INVALID_ARGUMENT"
    P = atos.Graph.peer(g.off, g.col, 2)
    with pytest.raises(atos.AtosError) as e:
        atos.color(P)
    assert e.value.name == "UNSUPPORTED"
    with pytest.raises(atos.AtosError) as e:
        atos.bfs(P, g.n)
    assert e.value.name == "INVALID_ARGUMENT"

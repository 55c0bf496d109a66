"""1-D partition multi-process tests.

CPU (gloo, world 2/3): partition bookkeeping invariants and the Python
orchestration (message grouping, all-to-all splits, termination) with a numpy
stand-in for the device library.  GPU: the CUDA partitioned path through the C
ABI — world 1, and world 2/3 as separate processes sharing cuda:0 with gloo
staging — checked against the unpartitioned oracle."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import graphgen as gg
import oracle

HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return str(p)


def _spawn(world, mode, app, tmp_path, timeout=300):
    port = _port()
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "dist_worker.py"), str(r), str(world), port, mode,
                               str(app), str(tmp_path)]) for r in range(world)]
    for p in procs:
        assert p.wait(timeout=timeout) == 0
    parts = [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]
    return np.concatenate([p["res"] for p in parts]), parts


def test_partition_invariants():
    from paper_2112_00132_b200 import dist as adist
    g, fwd = gg.permute(gg.rmat(10, 8, seed=1), 3)
    for world in (1, 2, 3, 8):
        b = adist.block_bounds(g.n, world)
        assert b[0] == 0 and b[-1] == g.n and np.all(np.diff(b) >= 0)
        owners = np.searchsorted(b, np.arange(g.n), side="right") - 1
        assert np.array_equal(np.bincount(owners, minlength=world), np.diff(b))  # each vertex owned once
        m = 0
        for r in range(world):
            lo, lc = adist.local_csr(g.off, g.col, int(b[r]), int(b[r + 1]))
            assert lo[0] == 0 and lo.shape[0] == b[r + 1] - b[r] + 1
            v = int(b[r]) + 3 if b[r + 1] - b[r] > 3 else int(b[r])
            if v < b[r + 1]:
                assert np.array_equal(lc[lo[v - b[r]]:lo[v - b[r] + 1]], g.col[g.off[v]:g.off[v + 1]])
            m += lc.shape[0]
        assert m == g.m


@pytest.mark.parametrize("world", [2, 3])
def test_orchestration_gloo_fake_engine(world, tmp_path):
    """Real gloo all-to-all / all-reduce, numpy stand-in for the kernels."""
    depth, parts = _spawn(world, "fake", 0, tmp_path)
    g, fwd = gg.permute(gg.rmat(12, 8, seed=3), 7)
    assert np.array_equal(depth, oracle.bfs(g, int(parts[0]["src"])))
    assert int(parts[0]["rounds"]) == 0  # fake engine reports no stats


def _check_partitioned_coloring(colors, parts):
    g, fwd = gg.permute(gg.rmat(12, 8, seed=3, symmetrize=True), 7)
    bad, k = oracle.check_coloring(g, colors)
    assert bad == 0  # proper: zero monochromatic edges (exhaustive scan)
    assert np.all(colors >= 0) and np.all(colors <= g.degrees())  # first fit: colour <= degree
    assert all(int(p["num_colors"]) == k for p in parts)  # every rank reports the global count
    return g, k


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_coloring_protocol_gloo_fake_engine(world, tmp_path):
    """The cross-rank colouring protocol (ghost replica, changed-colour
    messages, larger endpoint recolours) with real gloo collectives and a serial
    numpy stand-in for each rank's kernel: the union is a proper colouring."""
    colors, parts = _spawn(world, "fake", 2, tmp_path)
    g, k = _check_partitioned_coloring(colors, parts)
    assert k <= int(g.degrees().max()) + 1


@pytest.mark.gpu
@pytest.mark.parametrize("world,mode,worker", [(2, "gpu", "cta"), (3, "gpu", "cta"), (3, "gpu", "warp"),
                                               (2, "gpu", "thread"), (2, "gpu-discrete", "warp")])
def test_gpu_partitioned_coloring_multiprocess(world, mode, worker, tmp_path, monkeypatch):
    monkeypatch.setenv("ATOS_TEST_WORKER", worker)
    colors, parts = _spawn(world, mode, 2, tmp_path)
    _check_partitioned_coloring(colors, parts)
    assert sum(int(p["bytes"]) for p in parts) > 0  # ghost colours were exchanged


@pytest.mark.gpu
@pytest.mark.parametrize("world,mode", [(2, "gpu"), (3, "gpu"), (3, "gpu-discrete")])
def test_gpu_partitioned_bfs_multiprocess(world, mode, tmp_path):
    depth, parts = _spawn(world, mode, 0, tmp_path)
    g, fwd = gg.permute(gg.rmat(12, 8, seed=3), 7)
    assert np.array_equal(depth, oracle.bfs(g, int(parts[0]["src"])))
    assert sum(int(p["bytes"]) for p in parts) > 0  # remote traffic happened


@pytest.mark.gpu
@pytest.mark.parametrize("world,mode", [(2, "gpu"), (3, "gpu"), (2, "gpu-discrete")])
def test_gpu_partitioned_pagerank_multiprocess(world, mode, tmp_path):
    rank, parts = _spawn(world, mode, 1, tmp_path)
    g, fwd = gg.permute(gg.rmat(12, 8, seed=3), 7)
    x, _ = oracle.pagerank(g, 0.85)
    assert np.max(np.abs(rank - x)) / x.max() <= 1e-4


@pytest.mark.gpu
def test_gpu_partitioned_world1():
    import paper_2112_00132_b200 as atos
    from paper_2112_00132_b200 import dist as adist
    g = gg.rmat(14, 16, seed=2)
    pg = adist.PartGraph.from_global(g, 1, 0)
    d, st = adist.bfs(pg, 0)
    assert np.array_equal(d, oracle.bfs(g, 0))
    r, st = adist.pagerank(pg, 0.85, 1e-6)
    x, _ = oracle.pagerank(g, 0.85)
    assert np.max(np.abs(r - x)) / x.max() <= 1e-4
    with pytest.raises(atos.AtosError):  # bounds[world] != global_n
        adist.PartGraph(g.n, 2, 0, [0, 5, 3], g.off[:6], g.col[:g.off[5]])
    with pytest.raises(atos.AtosError):  # a partitioned handle is not a single-GPU graph
        atos.bfs(pg, 0)
    with pytest.raises(atos.AtosError) as e:  # colouring needs a symmetric graph
        adist.color(pg)
    assert e.value.name == "INVALID_GRAPH"
    s = gg.rmat(13, 16, seed=2, symmetrize=True)
    ps = adist.PartGraph.from_global(s, 1, 0)
    for w in ("cta", "warp", "thread"):
        c, st = adist.color(ps, worker=w)
        bad, k = oracle.check_coloring(s, c)
        assert bad == 0 and st["num_colors"] == k

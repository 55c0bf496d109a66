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


@pytest.fixture(scope="module")
def harness(tmp_path_factory):
    """The library's round loop (csrc/rounds.h) built with serial CPU engines."""
    so = tmp_path_factory.mktemp("harness") / "libharness.so"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I", os.path.join(os.path.dirname(HERE), "include"),
                           "-o", str(so), os.path.join(HERE, "round_harness.cpp")])
    return str(so)


@pytest.mark.parametrize("world", [2, 3])
def test_round_loop_bfs_gloo(world, harness, tmp_path, monkeypatch):
    """rounds.h over real gloo collectives (host callbacks) with a serial BFS
    engine per rank: the union of the ranks' depths is the oracle's."""
    monkeypatch.setenv("ATOS_HARNESS", harness)
    depth, parts = _spawn(world, "harness", 0, tmp_path)
    g, fwd = gg.permute(gg.rmat(12, 8, seed=3), 7)
    assert np.array_equal(depth.astype(np.uint32), oracle.bfs(g, int(parts[0]["src"])))
    assert all(int(p["rc"]) == 0 for p in parts)
    assert len({int(p["rounds"]) for p in parts}) == 1 and int(parts[0]["rounds"]) > 1  # all ranks agree
    assert sum(int(p["bytes"]) for p in parts) > 0


@pytest.mark.parametrize("world", [2, 3])
def test_round_loop_pagerank_closing_flush_gloo(world, harness, tmp_path, monkeypatch):
    """PageRank rounds: remote contributions below eps accumulate and are only
    sent by the closing flush round; the result meets the 1e-4 gate."""
    monkeypatch.setenv("ATOS_HARNESS", harness)
    rank, parts = _spawn(world, "harness", 1, tmp_path)
    g, fwd = gg.permute(gg.rmat(12, 8, seed=3), 7)
    x, _ = oracle.pagerank(g, 0.85)
    assert all(int(p["rc"]) == 0 for p in parts)
    assert np.max(np.abs(rank - x)) / x.max() <= 1e-4


def test_round_loop_collective_error_gloo(harness, tmp_path, monkeypatch):
    """An abort on one rank fails the call on EVERY rank in the same round (no
    rank is left waiting in a collective)."""
    monkeypatch.setenv("ATOS_HARNESS", harness)
    _, parts = _spawn(3, "harness-fail", 0, tmp_path)
    assert [int(p["rc"]) for p in parts] == [7, 7, 7]  # ATOS_ERR_TIMEOUT everywhere
    assert {int(p["rounds"]) for p in parts} == {2}


def _check_partitioned_coloring(colors, parts):
    g, fwd = gg.permute(gg.rmat(12, 8, seed=3, symmetrize=True), 7)
    bad, k = oracle.check_coloring(g, colors)
    assert bad == 0  # proper: zero monochromatic edges (exhaustive scan)
    assert np.all(colors >= 0) and np.all(colors <= g.degrees())  # first fit: colour <= degree
    assert all(int(p["num_colors"]) == k for p in parts)  # every rank reports the global count
    return g, k


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
    assert len({int(p["rounds"]) for p in parts}) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("world,mode", [(2, "gpu"), (3, "gpu"), (2, "gpu-discrete")])
def test_gpu_partitioned_pagerank_multiprocess(world, mode, tmp_path):
    rank, parts = _spawn(world, mode, 1, tmp_path)
    g, fwd = gg.permute(gg.rmat(12, 8, seed=3), 7)
    x, _ = oracle.pagerank(g, 0.85)
    assert np.max(np.abs(rank - x)) / x.max() <= 1e-4
    assert np.all(rank <= x * (1 + 1e-5) + 1e-6)


@pytest.mark.gpu
@pytest.mark.parametrize("world,mode,r64", [(2, "gpu", "0"), (3, "gpu", "0"), (2, "gpu-discrete", "0"), (2, "gpu", "1")])
def test_gpu_partitioned_pagerank_fan_in_hub(world, mode, r64, tmp_path, monkeypatch):
    """The 40,001-vertex fan-in hub across ranks: its 40,000 in-edges are mostly
    remote, so the hub's mass arrives through the fp64 remote accumulators and
    the compensated fp32 adds of the receiver (R30, R34)."""
    monkeypatch.setenv("ATOS_TEST_R64", r64)
    rank, parts = _spawn(world, mode, 3, tmp_path)
    import graphgen as ggm
    k, fan = 40000, 64
    e = [(s, 0) for s in range(1, k + 1)] + [(s, s + 1) for s in range(1, k)] + [(0, j) for j in range(1, fan + 1)]
    x, _ = oracle.pagerank(ggm.from_edges(k + 1, e), 0.85)
    assert np.max(np.abs(rank - x)) / x.max() <= 1e-4
    assert np.all(rank <= x * (1 + 1e-5) + 1e-6)


def _world1_comm(atos):
    """A one-rank NCCL communicator created through the C ABI alone."""
    import ctypes
    from paper_2112_00132_b200 import dist as adist
    L = atos.lib()
    uid = (ctypes.c_uint8 * 128)()
    atos._check(L.atos_comm_unique_id(uid), "atos_comm_unique_id")
    h = ctypes.c_void_p()
    atos._check(L.atos_comm_init(0, 1, uid, ctypes.byref(h)), "atos_comm_init")
    return adist.Comm(h, 0, 1)


@pytest.mark.gpu
def test_gpu_partitioned_world1_nccl():
    import paper_2112_00132_b200 as atos
    from paper_2112_00132_b200 import dist as adist
    comm = _world1_comm(atos)
    g = gg.rmat(14, 16, seed=2)
    pg = adist.PartGraph.from_global(g, comm)
    for kernel in ("persistent", "discrete"):
        d, st = adist.bfs(pg, 0, kernel=kernel)
        assert np.array_equal(d, oracle.bfs(g, 0)) and st["rounds"] >= 1
        r, st = adist.pagerank(pg, 0.85, 1e-6, kernel=kernel)
        x, _ = oracle.pagerank(g, 0.85)
        assert np.max(np.abs(r - x)) / x.max() <= 1e-4
    with pytest.raises(atos.AtosError) as e:  # colouring needs a symmetric graph
        adist.color(pg)
    assert e.value.name == "INVALID_GRAPH"
    with pytest.raises(atos.AtosError) as e:  # ranges must tile [0, global_n)
        adist.PartGraph(comm, g.n, 0, 5, g.off[:6], g.col[:g.off[5]])
    assert e.value.name == "INVALID_ARGUMENT"
    s = gg.rmat(13, 16, seed=2, symmetrize=True)
    ps = adist.PartGraph.from_global(s, comm)
    for w in ("cta", "warp", "thread"):
        c, st = adist.color(ps, worker=w)
        bad, k = oracle.check_coloring(s, c)
        assert bad == 0 and st["num_colors"] == k
    ps.close()
    pg.close()
    comm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2])
def test_c_program_partitioned_bfs(world, tmp_path):
    """A gcc-built C program linking libatos.so runs partitioned BFS through
    atos_bfs alone: world 1 over an NCCL communicator, world 2 as two forked
    processes exchanging through atos_comm_init_host callbacks over a socket pair."""
    import paper_2112_00132_b200 as atos
    g = gg.rmat(12, 8, seed=5)
    g.off.astype(np.int64).tofile(tmp_path / "off.bin")
    g.col.astype(np.int32).tofile(tmp_path / "col.bin")
    exe = tmp_path / "cbfs"
    libdir = os.path.dirname(atos.LIB_PATH)
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(os.path.dirname(HERE), "include"), "-o", str(exe),
                           os.path.join(HERE, "c_partitioned_bfs.c"), "-L", libdir, "-latos",
                           f"-Wl,-rpath,{libdir}"])
    subprocess.check_call([str(exe), str(world), str(g.n), str(g.m), str(tmp_path)], timeout=300)
    depth = np.concatenate([np.fromfile(tmp_path / f"depth{r}.bin", dtype=np.uint32) for r in range(world)])
    assert np.array_equal(depth, oracle.bfs(g, 0))

"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element
by element on the same seeded inputs.

Acceptance (BASELINE.json north_star):
  BFS        bit-exact depths;
  PageRank   ||rank - x*||_inf <= 1e-4 * max(x*) vs the fp64 Jacobi oracle, and
             every residue <= eps (device-reported);
  colouring  zero monochromatic edges (exhaustive scan), color[v] <= deg(v);
             colour count reported beside the oracle's, not asserted equal.
"""
import itertools
import os

import numpy as np
import pytest

import graphgen as gg
import oracle

pytestmark = pytest.mark.gpu
PR_TOL = 1e-4
# One-sided bound of push PageRank: 0 <= x* - rank in exact arithmetic (Alg. 4
# invariant).  fp32 residue adds round to nearest (relative 2^-24
# per add, half an ulp) and a non-hub vertex (in-degree < 2048, R34) takes
# < 2048 adds per queue cycle, so the mass it forwards is off by < 2048 * 2^-25
# relative; by positivity of (I - aP)^-1 so is rank (DESIGN R36).  + 1e-6: fp32 output.
ONE_SIDED = 1 + 2048 * 2.0 ** -25

KERNELS = ["persistent", "discrete", "bsp"]
WORKERS = ["thread", "warp", "cta"]
FETCH = [1, 4, 32, 256]


@pytest.fixture(scope="module")
def atos():
    import torch
    assert torch.cuda.is_available()
    import paper_2112_00132_b200 as a
    a.lib()
    return a


_cache = {}


def T(worker, fetch):
    """cta_threads (the library shrinks staging blocks to fit shared memory)."""
    return 256


def G(name):
    """Seeded test graphs (host CSR, cached)."""
    if name not in _cache:
        f = {
            "grid64": lambda: gg.grid(64, 64),
            "rmat16": lambda: gg.rmat(16, 16, seed=1),
            "rmat16s": lambda: gg.rmat(16, 16, seed=1, symmetrize=True),
            "rmat12": lambda: gg.rmat(12, 16, seed=1),
            "rmat12s": lambda: gg.rmat(12, 16, seed=1, symmetrize=True),
            "road": lambda: gg.grid(120, 90, drop_prob=0.4, seed=5),
            "path": lambda: gg.path(3000),
            "star": lambda: gg.star(5000),
            "K9": lambda: gg.complete(9),
            "hub": lambda: gg.hub_graph(70000, extra=300),
            "two": lambda: gg.from_edges(10, [(0, 1), (1, 2), (5, 6), (6, 7), (7, 5)], symmetrize=True),
            "empty5": lambda: gg.empty(5),
        }[name]
        _cache[name] = f()
    return _cache[name]


_dev = {}


def D(atos, name, symmetric=False):
    key = (name, symmetric)
    if key not in _dev:
        _dev[key] = atos.Graph.from_csr(G(name), symmetric=symmetric)
    return _dev[key]


# ------------------------------------------------------------------ BFS ---

def expandable(g, depth, src):
    """Vertices a BFS must pop with sink deferral (R29): the reached vertices
    with out-degree > 0, plus the source (always enqueued)."""
    deg = np.diff(g.off)
    reach = depth != oracle.UNREACHED
    return int(np.sum(reach & (deg > 0))) + int(deg[src] == 0)


@pytest.mark.parametrize("kernel,worker,fetch", list(itertools.product(KERNELS, WORKERS, FETCH)))
@pytest.mark.parametrize("gname", ["grid64", "rmat16"])
def test_bfs_matrix(atos, gname, kernel, worker, fetch):
    g = G(gname)
    d, st = atos.bfs(D(atos, gname), 0, kernel=kernel, worker=worker, fetch_size=fetch,
                     cta_threads=T(worker, fetch))
    exp = oracle.bfs(g, 0)
    assert np.array_equal(d, exp), f"{int(np.sum(d != exp))} mismatches"
    assert st["tasks_popped"] >= expandable(g, exp, 0)  # overwork >= 1


def test_bfs_grid_manhattan(atos):
    d, _ = atos.bfs(D(atos, "grid64"), 0)
    i, j = np.divmod(np.arange(64 * 64), 64)
    assert np.array_equal(d, (i + j).astype(np.uint32)) and d.max() == 126


@pytest.mark.parametrize("seed", range(20))
def test_bfs_small_rmat_seeds(atos, seed):
    # SPEC S:556 acceptance 1: oracle equivalence, 20 seeds
    g = gg.rmat(10, 8, seed=seed)
    G_ = atos.Graph.from_csr(g)
    for cfg in [dict(), dict(worker="warp", fetch_size=4), dict(worker="thread", fetch_size=1, kernel="discrete")]:
        d, _ = atos.bfs(G_, seed % g.n, **cfg)
        assert np.array_equal(d, oracle.bfs(g, seed % g.n)), cfg


@pytest.mark.parametrize("gname,src", [("path", 0), ("path", 1500), ("star", 0), ("star", 17), ("K9", 4),
                                       ("hub", 0), ("two", 0), ("two", 5), ("two", 9), ("empty5", 2), ("road", 0)])
@pytest.mark.parametrize("worker", WORKERS)
def test_bfs_special_graphs(atos, gname, src, worker):
    g = G(gname)
    d, _ = atos.bfs(D(atos, gname), src, worker=worker, fetch_size=32)
    assert np.array_equal(d, oracle.bfs(g, src))


def test_bfs_serial_order_identity(atos):
    """One warp worker, FETCH 1, one CTA: FIFO order => Dijkstra order =>
    every reachable vertex is popped exactly once (overwork 1.0);
    with sink deferral (R29) every reachable non-dangling vertex."""
    for name in ["grid64", "rmat12", "road"]:
        g = G(name)
        exp = oracle.bfs(g, 0)
        for defer in (False, True):
            d, st = atos.bfs(D(atos, name), 0, worker="warp", fetch_size=1, num_blocks=1, cta_threads=32,
                             sink_defer=defer)
            assert np.array_equal(d, exp)
            want = expandable(g, exp, 0) if defer else int(np.sum(exp != oracle.UNREACHED))
            assert st["tasks_popped"] == want, (name, defer)


@pytest.mark.parametrize("name", ["rmat12s", "grid64", "K9", "two"])
def test_color_serial_order_identity(atos, name):
    """One warp worker, FETCH 1, one CTA: the queue is strictly FIFO, so every
    ASSIGN(v) (queued in id order, R22) runs after every ASSIGN(u < v) and
    before any CHECK — exactly the oracle's serial id-order greedy:
    the same colour for every vertex, not just the same count.  More tasks in
    flight raise the count (tests/harness/experiments.py colorq)."""
    g = G(name)
    exp, k_or = oracle.greedy_color(g)
    c, k, st = atos.color(D(atos, name, symmetric=True), worker="warp", fetch_size=1, num_blocks=1, cta_threads=32)
    assert np.array_equal(c, exp)
    assert k == k_or
    assert st["tasks_popped"] == 2 * g.n  # one ASSIGN and one CHECK each, no conflict


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("worker", WORKERS)
def test_bfs_sink_defer(atos, kernel, worker):
    """R29: dangling vertices get their depth from the atomicMin and are never
    pushed; depths stay bit-exact, pops drop to the expandable vertices."""
    g = G("rmat16")
    exp = oracle.bfs(g, 0)
    pops = {}
    for defer in (False, True):
        d, st = atos.bfs(D(atos, "rmat16"), 0, kernel=kernel, worker=worker, fetch_size=32,
                         cta_threads=T(worker, 32), sink_defer=defer)
        assert np.array_equal(d, exp), (defer, int(np.sum(d != exp)))
        pops[defer] = st["tasks_popped"]
    assert pops[True] >= expandable(g, exp, 0)
    assert pops[True] < pops[False], pops
    # a dangling source is still popped once; its neighbours-less task ends the run
    h = gg.from_edges(4, [(1, 0), (2, 0)])
    d, st = atos.bfs(atos.Graph.from_csr(h), 0, kernel=kernel, worker=worker)
    assert list(d) == [0, oracle.UNREACHED, oracle.UNREACHED, oracle.UNREACHED] and st["tasks_popped"] == 1


def test_bfs_deep_path_beyond_u16_mirror(atos):
    """Depths above 65,534 saturate the 2-byte dist mirror used by the edge
    filter; the filter must then defer to the 32-bit atomicMin (R25 notes)."""
    g = gg.path(70000)
    for cfg in [dict(), dict(worker="warp", fetch_size=4), dict(kernel="bsp")]:
        d, _ = atos.bfs(atos.Graph.from_csr(g), 0, **cfg)
        assert np.array_equal(d, np.arange(70000, dtype=np.uint32)), cfg


def test_trace_records(atos):
    g = G("rmat16")
    tr = atos.Trace(1 << 22)
    d, st = atos.bfs(D(atos, "rmat16"), 0, trace=tr)
    assert np.array_equal(d, oracle.bfs(g, 0))  # tracing writes from the hot loop: results must not change
    r = tr.records(st)
    assert st["trace_records"] == len(r) > 0
    assert np.all(np.diff(r["t_ns"].astype(np.int64)) >= 0)
    # every popped task is in exactly one record (chunk tasks included)
    assert int(r["items"].sum()) == st["tasks_popped"] + st["chunk_tasks"]
    assert int(r["edges"].astype(np.int64).sum()) == st["edges_processed"]
    assert set(np.unique(r["kind"]).tolist()) == {0}
    # PageRank and colouring with the timeline on: parity and record accounting
    x = jacobi("rmat16")
    rk, st = atos.pagerank(D(atos, "rmat16"), 0.85, 1e-6, trace=tr)
    assert np.max(np.abs(rk.astype(np.float64) - x)) / x.max() <= PR_TOL and st["max_residue"] <= 1e-6
    r = tr.records(st)
    assert int(r["items"].sum()) == st["tasks_popped"] + st["chunk_tasks"] and set(np.unique(r["kind"]).tolist()) == {1}
    c, k, st = atos.color(D(atos, "rmat16s", symmetric=True), trace=tr)
    assert oracle.check_coloring(G("rmat16s"), c)[0] == 0
    r = tr.records(st)
    assert int(r["items"].sum()) == st["tasks_popped"] and set(np.unique(r["kind"]).tolist()) == {2}


def test_stats_invariants(atos):
    g = G("rmat16")
    exp = oracle.bfs(g, 0)
    reach = exp != oracle.UNREACHED
    for cfg in [dict(), dict(worker="warp"), dict(worker="thread", fetch_size=1), dict(kernel="discrete"),
                dict(kernel="bsp")]:
        d, st = atos.bfs(D(atos, "rmat16"), 0, **cfg)
        assert st["tasks_pushed"] == st["tasks_popped"] - 1 or cfg.get("kernel") == "bsp", cfg  # src + pushes
        assert st["edges_processed"] >= int(g.degrees()[reach].sum()), cfg
        assert st["kernel_launches"] >= 1 and st["ms"] > 0


@pytest.mark.parametrize("worker", WORKERS)
def test_discrete_device_loop(atos, worker):
    """Discrete strategy with the round loop in a CUDA-graph WHILE node."""
    for name in ["rmat16", "grid64", "path"]:
        d, st = atos.bfs(D(atos, name), 0, kernel="discrete", device_loop=True, worker=worker, fetch_size=16)
        assert np.array_equal(d, oracle.bfs(G(name), 0)), name
        d2, st2 = atos.bfs(D(atos, name), 0, kernel="discrete", worker=worker, fetch_size=16)
        assert st["rounds"] == st2["rounds"], name  # same rounds as the host-driven loop
    x = jacobi("rmat16")
    r, st = atos.pagerank(D(atos, "rmat16"), 0.85, 1e-6, kernel="discrete", device_loop=True, worker=worker,
                          fetch_size=32)
    assert np.max(np.abs(r - x)) / x.max() <= PR_TOL and st["max_residue"] <= 1e-6
    c, k, st = atos.color(D(atos, "rmat16s", symmetric=True), kernel="discrete", device_loop=True, worker=worker)
    assert oracle.check_coloring(G("rmat16s"), c)[0] == 0


def test_bfs_adaptive_fetch_off(atos):
    d, st = atos.bfs(D(atos, "rmat16"), 0, adaptive_fetch=False)
    assert np.array_equal(d, oracle.bfs(G("rmat16"), 0))


def test_bfs_device_output_and_torch_borrow(atos):
    import torch
    g = G("rmat12")
    off = torch.from_numpy(g.off).cuda()
    col = torch.from_numpy(g.col).cuda()
    Gt = atos.Graph(off, col)
    d, _ = atos.bfs(Gt, 3, device=True)
    assert d.is_cuda
    assert np.array_equal(d.cpu().numpy().view(np.uint32), oracle.bfs(g, 3))


@pytest.mark.parametrize("stage", [0, 256, 1024, 8192])
@pytest.mark.parametrize("gname,src", [("rmat16", 0), ("hub", 0), ("road", 17), ("star", 3)])
def test_bfs_column_staging(atos, gname, src, stage):
    """Persistent CTA workers with TMA-staged column lists: every
    staging capacity (0 = off, 256 = most items fall back to global loads,
    8192 = whole batches staged) gives the oracle's depths."""
    for fetch, thr in [(128, 256), (7, 64), (1024, 512)]:
        d, _ = atos.bfs(D(atos, gname), src, fetch_size=fetch, cta_threads=thr, stage_edges=stage)
        assert np.array_equal(d, oracle.bfs(G(gname), src)), (fetch, thr)


def test_staging_borrowed_unpadded_columns(atos):
    """A borrowed column array has no padding: the list ending at m must not be
    bulk-copied past the allocation (it falls back to global loads)."""
    import torch
    g = gg.from_edges(6, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 0), (5, 1)])  # m = 7: last list ends at m
    assert g.m % 4 != 0
    off = torch.from_numpy(g.off).cuda()
    col = torch.from_numpy(g.col[:]).cuda()
    Gt = atos.Graph(off, col)
    d, _ = atos.bfs(Gt, 0, stage_edges=1024)
    assert np.array_equal(d, oracle.bfs(g, 0))
    x = oracle.pagerank(g, 0.85)[0]
    r, st = atos.pagerank(Gt, 0.85, 1e-6, stage_edges=1024)
    assert np.max(np.abs(r - x)) / x.max() <= PR_TOL


@pytest.mark.parametrize("gname", ["rmat16", "star", "two"])
def test_tagged_vs_borrowed_columns(atos, gname):
    """R34/R37: a library-owned CSR carries HUB/SINK tags in bits 31/30 of its
    column entries; a borrowed (caller-owned) one is never written and uses the
    bitmaps and fp64 residues.  Both give the oracle's answers, and the sink
    tag defers exactly the dangling vertices the bitmap does (same pops for
    the deterministic single-worker BFS)."""
    import torch
    g = G(gname)
    Gt = atos.Graph(torch.from_numpy(g.off).cuda(), torch.from_numpy(g.col.copy()).cuda())
    Go = D(atos, gname)
    x, src = jacobi(gname), 0
    for Gx in (Go, Gt):
        d, sb = atos.bfs(Gx, src, worker="thread", fetch_size=1, num_blocks=1, cta_threads=32)
        assert np.array_equal(d, oracle.bfs(g, src))
        r, st = atos.pagerank(Gx, 0.85, 1e-6, fetch_size=64)
        assert np.max(np.abs(r.astype(np.float64) - x)) / x.max() <= PR_TOL
        assert st["max_residue"] <= 1e-6
    _, s1 = atos.bfs(Go, src, worker="thread", fetch_size=1, num_blocks=1, cta_threads=32)
    _, s2 = atos.bfs(Gt, src, worker="thread", fetch_size=1, num_blocks=1, cta_threads=32)
    assert s1["tasks_popped"] == s2["tasks_popped"]


@pytest.mark.parametrize("stage", [0, 512, 4096])
def test_pagerank_column_staging(atos, stage):
    x = jacobi("rmat16")
    for fetch, thr in [(128, 512), (16, 128)]:
        r, st = atos.pagerank(D(atos, "rmat16"), 0.85, 1e-6, fetch_size=fetch, cta_threads=thr, stage_edges=stage)
        assert np.max(np.abs(r - x)) / x.max() <= PR_TOL
        assert st["max_residue"] <= 1e-6


def test_stage_edges_invalid(atos):
    with pytest.raises(atos.AtosError) as e:
        atos.bfs(D(atos, "K9"), 0, stage_edges=-2)
    assert e.value.name == "INVALID_ARGUMENT"


def test_bfs_queue_wraparound(atos):
    g = G("grid64")
    d, st = atos.bfs(D(atos, "grid64"), 0, queue_capacity=256, worker="warp", fetch_size=4)
    assert np.array_equal(d, oracle.bfs(g, 0))
    assert st["tasks_pushed"] > 256  # wrapped the ring


def hub_chain(k=300, deg=5000):
    """k hubs in a chain: hub i has `deg` parallel edges to hub i+1, so every hub is
    split into chunk tasks (R24) while the frontier stays one vertex wide."""
    off = np.arange(k + 2, dtype=np.int64) * deg
    off[-1] = off[-2]  # the last vertex has no edges
    col = np.repeat(np.arange(1, k + 1, dtype=np.int32), deg)
    return off, col


@pytest.mark.parametrize("gname,cap", [("grid64", 256), ("road", 256), ("hubchain", 256)])
@pytest.mark.parametrize("fetch,threads", [(128, 256), (16, 64), (512, 1024)])
def test_bfs_cta_queue_wraparound(atos, gname, cap, fetch, threads):
    """Persistent CTA workers (queue agent, hub chunk tasks) on a small ring:
    the agent reads every claimed slot before it pushes, chunk
    entries live exactly as long as their slots; exact depths, no hang."""
    if gname == "hubchain":
        off, col = hub_chain()
        Gd = atos.Graph(off, col)
        exp = np.arange(301, dtype=np.uint32)
    else:
        Gd, exp = D(atos, gname), oracle.bfs(G(gname), 0)
    d, st = atos.bfs(Gd, 0, queue_capacity=cap, fetch_size=fetch, cta_threads=threads, timeout_s=60)
    assert np.array_equal(d, exp)
    assert st["tasks_pushed"] + st["chunk_tasks"] > cap  # wrapped the ring
    if gname == "hubchain":
        assert st["chunk_tasks"] >= 300


@pytest.mark.parametrize("worker", WORKERS)
def test_pagerank_queue_wraparound(atos, worker):
    """PageRank on a 2n-slot ring (threshold activation keeps <= 2 live copies
    per vertex, R16): the pushes wrap the ring several times."""
    g = G("rmat12")
    x = jacobi("rmat12")
    r, st = atos.pagerank(D(atos, "rmat12"), 0.85, 1e-6, worker=worker, fetch_size=32, queue_capacity=2 * g.n,
                          timeout_s=60)
    assert np.max(np.abs(r.astype(np.float64) - x)) / x.max() <= PR_TOL
    assert st["tasks_pushed"] > 4 * g.n


def test_bfs_queue_overflow(atos):
    with pytest.raises(atos.AtosError) as e:
        atos.bfs(D(atos, "star"), 0, queue_capacity=32, num_blocks=1)
    assert e.value.name == "QUEUE_OVERFLOW"
    # the handle stays usable
    d, _ = atos.bfs(D(atos, "star"), 0)
    assert np.array_equal(d, oracle.bfs(G("star"), 0))


def test_bfs_errors(atos):
    with pytest.raises(atos.AtosError) as e:
        atos.bfs(D(atos, "grid64"), 4096)
    assert e.value.name == "INVALID_ARGUMENT"
    with pytest.raises(atos.AtosError):
        atos.bfs(D(atos, "grid64"), 0, cta_threads=48)
    with pytest.raises(atos.AtosError):
        atos.bfs(D(atos, "grid64"), 0, fetch_size=0)
    E = atos.Graph(np.zeros(1, np.int64), np.zeros(0, np.int32))
    d, _ = atos.bfs(E, 0)  # n == 0: OK, nothing written
    assert d.size == 0
    with pytest.raises(atos.AtosError) as e:
        atos.Graph(np.array([0, 2, 1], np.int64), np.array([0, 1], np.int32), validate=True)
    assert e.value.name == "INVALID_GRAPH"
    with pytest.raises(atos.AtosError) as e:
        atos.Graph(np.array([0, 1, 2], np.int64), np.array([0, 7], np.int32), validate=True)
    assert e.value.name == "INVALID_GRAPH"


def test_watchdog_timeout(atos):
    with pytest.raises(atos.AtosError) as e:
        atos.pagerank(D(atos, "rmat16"), 0.85, 1e-9, timeout_s=1e-6, worker="thread", fetch_size=1)
    assert e.value.name == "TIMEOUT"
    r, st = atos.pagerank(D(atos, "rmat12"), 0.85, 1e-6)  # library still healthy
    assert st["max_residue"] <= 1e-6


# ------------------------------------------------------------- PageRank ---

_jac = {}


def jacobi(name, alpha=0.85):
    if (name, alpha) not in _jac:
        _jac[(name, alpha)] = oracle.pagerank(G(name), alpha)[0]
    return _jac[(name, alpha)]


@pytest.mark.parametrize("kernel,worker,fetch", [(k, w, f) for k in KERNELS for w in WORKERS for f in (1, 32, 256)])
def test_pagerank_matrix(atos, kernel, worker, fetch):
    x = jacobi("rmat16")
    # fp32 residues in every cell: thread workers with a large FETCH hold claimed
    # vertices long enough for their residue to grow to O(10), which rounded
    # away 6.6e-4 of max x* before the compensated adds (DESIGN R34)
    r, st = atos.pagerank(D(atos, "rmat16"), 0.85, 1e-6, kernel=kernel, worker=worker, fetch_size=fetch,
                          cta_threads=T(worker, fetch))
    err = np.max(np.abs(r.astype(np.float64) - x)) / x.max()
    assert err <= PR_TOL, err
    assert st["max_residue"] <= 1e-6
    # one-sided bound 0 <= x* - rank <= eps x*/(1-a) (Alg. 4 invariant; R34 keeps it through fp32)
    assert np.all(r <= x * ONE_SIDED + 1e-6)


@pytest.mark.parametrize("worker", WORKERS)
def test_pagerank_fp64_residue(atos, worker):
    x = jacobi("rmat16")
    for kernel in KERNELS:
        r, st = atos.pagerank(D(atos, "rmat16"), 0.85, 1e-6, kernel=kernel, worker=worker, fetch_size=32,
                              pr_residue_fp64=True)
        assert np.max(np.abs(r - x)) / x.max() <= PR_TOL
        assert st["max_residue"] <= 1e-6


@pytest.mark.parametrize("kernel", ["persistent", "discrete"])
@pytest.mark.parametrize("worker", WORKERS)
def test_pagerank_sink_defer(atos, kernel, worker):
    """R29: dangling vertices are never pushed on activation; their residue is
    absorbed after quiescence.  Same fixed point (Jacobi), fewer
    pushed tasks than the literal Alg. 4 activation (rmat16: 38% dangling)."""
    x = jacobi("rmat16")
    g = G("rmat16")
    dangling = np.diff(g.off) == 0
    assert dangling.mean() > 0.2
    pushed = {}
    for defer in (False, True):
        r, st = atos.pagerank(D(atos, "rmat16"), 0.85, 1e-6, kernel=kernel, worker=worker, fetch_size=32,
                              cta_threads=T(worker, 32), sink_defer=defer)
        assert np.max(np.abs(r.astype(np.float64) - x)) / x.max() <= PR_TOL
        assert st["max_residue"] <= 1e-6
        assert np.all(r <= x * ONE_SIDED + 1e-6)
        pushed[defer] = st["tasks_pushed"]
    assert pushed[True] < pushed[False], pushed


def test_pagerank_sink_defer_edge_cases(atos):
    a = 0.85
    # every vertex dangling: nothing propagates, rank = 1 - a
    r, st = atos.pagerank(atos.Graph.from_csr(gg.empty(37)), a, 1e-6)
    assert np.allclose(r, 1 - a) and st["tasks_pushed"] == 0
    # directed chain 0->...->k: only the last vertex is dangling; x_i = 1 - a^(i+1)
    for defer in (False, True):
        r, _ = atos.pagerank(atos.Graph.from_csr(gg.directed_chain(6)), a, 1e-7, sink_defer=defer)
        assert np.allclose(r, 1 - a ** (np.arange(6) + 1), atol=1e-5)


@pytest.mark.parametrize("gname", ["rmat16", "hub", "star", "fanin"])
@pytest.mark.parametrize("deg,factor", [(1, 1000), (16, 4), (1024, 8)])
def test_pagerank_hub_deferral(atos, gname, deg, factor):
    """R31: deferring popped hubs with small residues (re-queued once with
    DEFER_BIT) reaches the same fixed point; (1, 1000) defers nearly every pop."""
    g = fan_in_graph() if gname == "fanin" else G(gname)
    x = oracle.pagerank(g, 0.85)[0]
    Gd = atos.Graph.from_csr(g) if gname == "fanin" else D(atos, gname)
    # deferring the fan-in hub lets its fp32 residue grow for a second queue cycle while
    # eps-sized pushes arrive (1.1e-4 / 1.8e-4 of max x* rounded away before R34)
    r, st = atos.pagerank(Gd, 0.85, 1e-6, fetch_size=64, pr_defer_degree=deg, pr_defer_factor=factor)
    assert np.max(np.abs(r.astype(np.float64) - x)) / x.max() <= PR_TOL
    assert st["max_residue"] <= 1e-6
    assert np.all(r <= x * ONE_SIDED + 1e-6)


def fan_in_graph(k=40000, fan=64):
    """k sources s -> 0 and s -> s+1 (chain), plus 0 -> 1..fan: vertex 0's
    seeding residue (R4) is k adds of the same c = (1-a)a/2 onto a sum growing
    to ~2,550, whose fp32 rounding errors are correlated (R30)."""
    if "graph" not in _fan:
        _fan["graph"] = gg.fan_in(k, fan)
    return _fan["graph"]


@pytest.mark.parametrize("r64", [False, True])
@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("worker", WORKERS)
def test_pagerank_fan_in_hub(atos, kernel, worker, r64):
    """A 40,000-way fan-in hub (x* = 11,930) fed by 40,000 equal pushes per
    sweep: fp32 residues rounded them the same way every time (1.8e-4 to
    5.8e-4 of max x* before the compensated adds, DESIGN R32/R34).  Both
    residue precisions must meet the gate and the one-sided bound."""
    g = fan_in_graph()
    x = fan_in_x()
    r, st = atos.pagerank(fan_in_dev(atos), 0.85, 1e-6, kernel=kernel, worker=worker, fetch_size=32,
                          cta_threads=T(worker, 32), pr_residue_fp64=r64)
    err = np.max(np.abs(r.astype(np.float64) - x)) / x.max()
    assert err <= PR_TOL, err
    assert st["max_residue"] <= 1e-6
    assert np.all(r <= x * ONE_SIDED + 1e-6)


_fan = {}


def fan_in_x():
    if "x" not in _fan:
        _fan["x"] = oracle.pagerank(fan_in_graph(), 0.85)[0]
    return _fan["x"]


def fan_in_dev(atos):
    if "g" not in _fan:
        _fan["g"] = atos.Graph.from_csr(fan_in_graph())
    return _fan["g"]


@pytest.mark.parametrize("fetch", [1, 32, 256, 1024])
@pytest.mark.parametrize("worker", WORKERS)
def test_pagerank_fan_in_fetch_sweep(atos, worker, fetch):
    """Large FETCH holds claimed vertices (and their growing residues) longest."""
    x = fan_in_x()
    r, st = atos.pagerank(fan_in_dev(atos), 0.85, 1e-6, worker=worker, fetch_size=fetch,
                          cta_threads=T(worker, fetch))
    assert np.max(np.abs(r.astype(np.float64) - x)) / x.max() <= PR_TOL
    assert st["max_residue"] <= 1e-6


@pytest.mark.parametrize("hub_check", [0, 1, 16, 1000])
@pytest.mark.parametrize("gname", ["rmat16", "fanin", "hub", "star"])
def test_pagerank_hub_sweep(atos, gname, hub_check):
    """R35: hub targets (in-degree >= 2048) take fire-and-forget fp64 adds and are
    activated by sweeps (hub_check hubs per processed batch; 0 = threshold
    crossing, R34); quiescence needs a clean sweep of every hub.  Same fixed
    point, every residue <= eps at return."""
    g = fan_in_graph() if gname == "fanin" else G(gname)
    x = fan_in_x() if gname == "fanin" else jacobi(gname)
    Gd = fan_in_dev(atos) if gname == "fanin" else D(atos, gname)
    for kw in [dict(fetch_size=128, cta_threads=1024), dict(fetch_size=1, cta_threads=96)]:
        r, st = atos.pagerank(Gd, 0.85, 1e-6, pr_hub_check=hub_check, timeout_s=60, **kw)
        assert np.max(np.abs(r.astype(np.float64) - x)) / x.max() <= PR_TOL
        assert st["max_residue"] <= 1e-6
        assert np.all(r <= x * ONE_SIDED + 1e-6)


@pytest.mark.parametrize("check_size", [1, 8, 32])
@pytest.mark.parametrize("gname", ["rmat16", "grid64", "star", "road", "hub", "two"])
def test_pagerank_window_activation(atos, gname, check_size):
    """Alg. 4's Check_Size window activation: red adds,
    sweeping-cursor re-activation, full-sweep termination (R9)."""
    x = jacobi(gname)
    r, st = atos.pagerank(D(atos, gname), 0.85, 1e-6, pr_activation=1, check_size=check_size, fetch_size=64)
    assert np.max(np.abs(r - x)) / x.max() <= PR_TOL
    assert st["max_residue"] <= 1e-6


def seed_tiles_graph():
    """Merge-path tile edge cases for the R4 seeding pass (k_pr_seed, 2,048
    vertices + edges per tile): a 5,000-vertex run of isolated vertices, one
    vertex of out-degree 7,000 spanning several tiles, another isolated run,
    a 3,000-way fan-in onto the last vertex (in-degree >= 2048: a hub, fp64
    seeding into its replicas) and a seeded random tail."""
    n = 20000
    rng = np.random.default_rng(7)
    e = [(5000, int(t)) for t in rng.choice(np.arange(5001, n), 7000, replace=False)]
    e += [(int(v), n - 1) for v in range(12000, 15000)]
    tail = rng.integers(15000, n, size=(20000, 2))
    e += [(int(a), int(b)) for a, b in tail if a != b]
    return gg.from_edges(n, e)


@pytest.mark.parametrize("gname", ["tiles", "cycle1024", "cycle2048", "K9", "empty5"])
@pytest.mark.parametrize("fp64", [False, True])
def test_pagerank_seeding_tiles(atos, gname, fp64):
    """R4 seeding over merge-path tiles: graphs whose n + m is below one tile,
    exactly one or two tiles (directed cycles: n + m = 2n), and a graph whose
    vertex runs and out-degree hub cross tile boundaries.  Both storages:
    fp32 with fp64 hubs (tagged) and all-fp64 residues."""
    g = {"tiles": seed_tiles_graph, "cycle1024": lambda: gg.cycle(1024, directed=True),
         "cycle2048": lambda: gg.cycle(2048, directed=True), "K9": lambda: G("K9"),
         "empty5": lambda: G("empty5")}[gname]()
    x = oracle.pagerank(g, 0.85)[0]
    r, st = atos.pagerank(atos.Graph.from_csr(g), 0.85, 1e-6, pr_residue_fp64=fp64, timeout_s=60)
    assert np.max(np.abs(r.astype(np.float64) - x)) / x.max() <= PR_TOL
    assert st["max_residue"] <= 1e-6
    assert np.all(r <= x * ONE_SIDED + 1e-6)


def test_pagerank_cta_threads_floor(atos):
    # persistent CTA PageRank runs two queue-agent warps per CTA: at least one worker warp more
    with pytest.raises(atos.AtosError) as e:
        atos.pagerank(D(atos, "K9"), 0.85, 1e-6, cta_threads=64)
    assert e.value.name == "INVALID_ARGUMENT"
    r, st = atos.pagerank(D(atos, "K9"), 0.85, 1e-6, cta_threads=96, fetch_size=1)
    assert np.allclose(r, 1.0, atol=1e-5)


def test_pagerank_window_unsupported_combos(atos):
    for kw in [dict(kernel="discrete"), dict(worker="warp"), dict(pr_residue_fp64=True)]:
        with pytest.raises(atos.AtosError) as e:
            atos.pagerank(D(atos, "K9"), 0.85, 1e-6, pr_activation=1, **kw)
        assert e.value.name == "UNSUPPORTED"


@pytest.mark.parametrize("gname", ["grid64", "star", "K9", "path", "two", "road", "hub"])
def test_pagerank_special(atos, gname):
    x = jacobi(gname)
    for cfg in [dict(), dict(worker="warp", fetch_size=8, kernel="discrete")]:
        r, st = atos.pagerank(D(atos, gname), 0.85, 1e-6, **cfg)
        assert np.max(np.abs(r - x)) / x.max() <= PR_TOL
        assert st["max_residue"] <= 1e-6


def test_pagerank_closed_forms(atos):
    a = 0.85
    r, _ = atos.pagerank(atos.Graph.from_csr(gg.star(5)), a, 1e-7)
    assert abs(r[0] - (1 + a * 5) / (1 + a)) < 1e-4 and np.allclose(r[1:], (1 + a / 5) / (1 + a), atol=1e-5)
    r, _ = atos.pagerank(atos.Graph.from_csr(gg.directed_chain(6)), a, 1e-7)
    assert np.allclose(r, 1 - a ** (np.arange(6) + 1), atol=1e-5)
    r, _ = atos.pagerank(atos.Graph.from_csr(gg.complete(8)), a, 1e-7)
    assert np.allclose(r, 1.0, atol=1e-5)


def test_pagerank_errors(atos):
    for al, ep in [(0.0, 1e-6), (1.0, 1e-6), (0.85, 0.0), (0.85, float("nan"))]:
        with pytest.raises(atos.AtosError) as e:
            atos.pagerank(D(atos, "K9"), al, ep)
        assert e.value.name == "INVALID_ARGUMENT"
    with pytest.raises(atos.AtosError) as e:
        atos.pagerank(D(atos, "rmat16"), 0.85, 1e-6, queue_capacity=1024)
    assert e.value.name == "QUEUE_OVERFLOW"


# ------------------------------------------------------------ colouring ---

@pytest.mark.parametrize("kernel,worker,fetch", [(k, w, f) for k in KERNELS for w in WORKERS for f in (1, 32, 256)])
def test_color_matrix(atos, kernel, worker, fetch):
    g = G("rmat16s")
    c, k, st = atos.color(D(atos, "rmat16s", symmetric=True), kernel=kernel, worker=worker, fetch_size=fetch,
                           cta_threads=T(worker, fetch))
    bad, kk = oracle.check_coloring(g, c)
    assert bad == 0
    assert kk == k
    _, k_or = oracle.greedy_color(g)
    print(f"colours gpu={k} oracle={k_or} tasks={st['tasks_popped']} overwork={st['tasks_popped'] / (2 * g.n):.2f}")


@pytest.mark.parametrize("worker", WORKERS)
def test_color_closed_forms(atos, worker):
    for kn in [2, 5, 9, 33]:
        c, k, _ = atos.color(atos.Graph.from_csr(gg.complete(kn), symmetric=True), worker=worker)
        assert k == kn and sorted(c.tolist()) == list(range(kn))
    c, k, _ = atos.color(atos.Graph.from_csr(gg.empty(7), symmetric=True), worker=worker)
    assert k == 1 and np.all(c == 0)
    for name in ["grid64", "road", "path", "star", "two"]:
        g = G(name)
        c, k, _ = atos.color(D(atos, name, symmetric=True), worker=worker)
        assert oracle.check_coloring(g, c)[0] == 0
        assert k <= int(g.degrees().max()) + 1


def test_color_requires_symmetric(atos):
    with pytest.raises(atos.AtosError) as e:
        atos.color(D(atos, "rmat16"))
    assert e.value.name == "INVALID_GRAPH"


def test_pool_reuse_across_graphs(atos):
    """Graph-lifetime arrays come from a retained stream-ordered pool (DESIGN §5
    Allocation): a destroyed graph's HBM is handed to the next create, so every
    array must be initialised per call.  Alternate a large and a small graph,
    destroying each after use, and check exact BFS / PageRank / colouring."""
    big, small = G("rmat16"), G("grid64")
    x_big, x_small = jacobi("rmat16"), oracle.pagerank(small, 0.85)[0]
    for _ in range(3):
        for g, x in ((big, x_big), (small, x_small)):
            Gd = atos.Graph.from_csr(g)
            d, _ = atos.bfs(Gd, 0)
            assert np.array_equal(d, oracle.bfs(g, 0))
            r, st = atos.pagerank(Gd, 0.85, 1e-6)
            assert np.max(np.abs(r.astype(np.float64) - x)) / x.max() <= PR_TOL
            Gd.close()
    gs = G("rmat12s")
    for _ in range(2):
        Gd = atos.Graph.from_csr(gs, symmetric=True)
        c, k, _ = atos.color(Gd)
        bad, kk = oracle.check_coloring(gs, c)
        assert bad == 0 and kk == k
        Gd.close()

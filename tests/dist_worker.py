"""Worker for multi-process partitioned tests (spawned by tests/test_dist.py; one process per rank).

mode "harness": the library's round loop (csrc/rounds.h) compiled into
  tests/round_harness.cpp with serial CPU engines, exchanging over gloo (no GPU).
mode "gpu" / "gpu-discrete": the CUDA partitioned path through the C ABI
  (atos_bfs / atos_pagerank / atos_color on atos_graph_create_partitioned),
  ranks sharing cuda:0, exchanges through a host communicator over gloo.
Writes this rank's result slice to <outdir>/rank<r>.npz."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

APP_FANIN = 3


def graph(app):
    import graphgen as gg
    if app == 2:
        g, fwd = gg.permute(gg.rmat(12, 8, seed=3, symmetrize=True), 7)
        return g, 0
    if app == APP_FANIN:
        k, fan = 40000, 64
        e = [(s, 0) for s in range(1, k + 1)] + [(s, s + 1) for s in range(1, k)] + [(0, j) for j in range(1, fan + 1)]
        return gg.from_edges(k + 1, e), 0
    g, fwd = gg.permute(gg.rmat(12, 8, seed=3), 7)
    return g, int(fwd[0])


def main():
    rank, world, port, mode, app, outdir = sys.argv[1:7]
    rank, world, app = int(rank), int(world), int(app)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2112_00132_b200 import dist as adist
    g, src = graph(app)
    b = adist.block_bounds(g.n, world)
    vb, ve = int(b[rank]), int(b[rank + 1])
    if mode.startswith("harness"):
        H = ctypes.CDLL(os.environ["ATOS_HARNESS"])
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        from paper_2112_00132_b200 import ALLGATHER_FN, ALLTOALLV_FN
        H.harness_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ALLGATHER_FN, ALLTOALLV_FN, i64, vp, vp,
                                  vp, i64, ctypes.c_double, ctypes.c_double, ctypes.c_int, vp, vp, vp]
        H.harness_run.restype = ctypes.c_int
        ag, a2a = adist.host_callbacks()
        lo, lc = adist.local_csr(g.off, g.col, vb, ve)
        out = np.zeros(ve - vb, dtype=np.float64)
        rounds, nbytes = ctypes.c_int64(0), ctypes.c_int64(0)
        fail = 2 if (mode == "harness-fail" and rank == world - 1) else -1
        rc = H.harness_run(min(app, 1), rank, world, ag, a2a, g.n, b.ctypes.data, lo.ctypes.data,
                           lc.ctypes.data if lc.size else None, src, 0.85, 1e-6, fail, out.ctypes.data,
                           ctypes.addressof(rounds), ctypes.addressof(nbytes))
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), res=out, rc=rc, rounds=rounds.value, bytes=nbytes.value,
                 src=src)
        dist.barrier()
        dist.destroy_process_group()
        return
    import paper_2112_00132_b200 as atos
    torch.cuda.set_device(0)
    comm = adist.Comm.host()
    pg = adist.PartGraph.from_global(g, comm, validate=True)
    kernel = "discrete" if mode == "gpu-discrete" else "persistent"
    worker = os.environ.get("ATOS_TEST_WORKER", "cta")
    kw = dict(kernel=kernel, worker=worker, fetch_size=32, timeout_s=120)
    if app == 0:
        res, st = adist.bfs(pg, src, **kw)
    elif app == 2:
        res, st = adist.color(pg, **kw)
    else:
        res, st = adist.pagerank(pg, 0.85, 1e-6, pr_residue_fp64=os.environ.get("ATOS_TEST_R64") == "1", **kw)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), res=res, src=src, rounds=st["rounds"], bytes=st["bytes_sent"],
             num_colors=st.get("num_colors", 0), launches=st["kernel_launches"])
    pg.close()
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    del atos


if __name__ == "__main__":
    main()

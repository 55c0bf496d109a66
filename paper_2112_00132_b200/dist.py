"""Multi-GPU BFS / PageRank / colouring over a 1-D vertex partition.

One process per GPU.  Each rank owns a contiguous block of (pre-permuted)
vertex ids.  ``atos_bfs`` / ``atos_pagerank`` / ``atos_color`` on a
partitioned handle run every exchange round inside the library (include/atos.h
"multi-GPU"; csrc/rounds.h): NCCL over NVLink/NVSwitch with ``Comm.nccl``, or
host callbacks with ``Comm.host`` (a gloo process group — used by the tests,
which run several ranks on one GPU).  This module only marshals arguments and,
for ``Comm.host``, forwards the library's two collective callbacks to
``torch.distributed``.
"""
from __future__ import annotations

import ctypes
import traceback

import numpy as np

from . import ALLGATHER_FN, ALLTOALLV_FN, CStats, Config, _cfg, _check, _out, _ptr, lib


def block_bounds(n: int, world: int) -> np.ndarray:
    """Contiguous block split: rank r owns [bounds[r], bounds[r+1])."""
    return np.array([r * n // world for r in range(world + 1)], dtype=np.int64)


def local_csr(off: np.ndarray, col: np.ndarray, vb: int, ve: int):
    """Rows [vb, ve) of a global CSR as a local CSR with global column ids."""
    lo = np.ascontiguousarray(off[vb:ve + 1] - off[vb], dtype=np.int64)
    lc = np.ascontiguousarray(col[off[vb]:off[ve]], dtype=np.int32)
    return lo, lc


def host_callbacks(group=None):
    """The two collective callbacks of atos_comm_init_host, forwarded to torch.distributed
    on host memory (argument marshalling only).  Returns (allgather, alltoallv) ctypes
    function objects; the caller keeps them alive while the communicator exists."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)

    def _bytes(ptr, n):
        if n == 0:
            return torch.empty(0, dtype=torch.uint8)
        return torch.frombuffer(bytearray(ctypes.string_at(ptr, n)), dtype=torch.uint8)

    def allgather(_user, send, recv, nbytes):
        try:
            t = _bytes(send, nbytes)
            outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(outs, t, group=group)
            if nbytes:
                allb = torch.cat(outs).numpy()  # kept alive across the copy
                ctypes.memmove(recv, allb.ctypes.data, nbytes * world)
            return 0
        except Exception:
            traceback.print_exc()
            return 1

    def alltoallv(_user, send, sbytes, recv, rbytes):
        try:
            sb = [int(sbytes[i]) for i in range(world)]
            rb = [int(rbytes[i]) for i in range(world)]
            inp = _bytes(send, sum(sb))
            out = torch.empty(sum(rb), dtype=torch.uint8)
            dist.all_to_all_single(out, inp, output_split_sizes=rb, input_split_sizes=sb, group=group)
            if sum(rb):
                outb = out.numpy()
                ctypes.memmove(recv, outb.ctypes.data, sum(rb))
            return 0
        except Exception:
            traceback.print_exc()
            return 1

    return ALLGATHER_FN(allgather), ALLTOALLV_FN(alltoallv)


class Comm:
    """An atos communicator (atos_comm)."""

    def __init__(self, handle, rank: int, world: int, keep=None):
        self.h, self.rank, self.world, self._keep = handle, rank, world, keep

    @classmethod
    def nccl(cls, group=None):
        """NCCL communicator over the ranks of a torch.distributed group (one GPU per rank):
        rank 0 creates the NCCL unique id, the group broadcasts it, every rank joins."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = (ctypes.c_uint8 * 128)()
        if rank == 0:
            _check(lib().atos_comm_unique_id(uid), "atos_comm_unique_id")
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(obj[0])
        h = ctypes.c_void_p()
        _check(lib().atos_comm_init(rank, world, uid, ctypes.byref(h)), "atos_comm_init")
        return cls(h, rank, world)

    @classmethod
    def host(cls, group=None):
        """Communicator whose exchanges run through torch.distributed on host memory (e.g. gloo)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        ag, a2a = host_callbacks(group)
        h = ctypes.c_void_p()
        _check(lib().atos_comm_init_host(rank, world, ag, a2a, None, ctypes.byref(h)), "atos_comm_init_host")
        return cls(h, rank, world, keep=(ag, a2a))

    @classmethod
    def auto(cls, group=None):
        """NCCL for an NCCL process group, host callbacks otherwise."""
        import torch.distributed as dist
        return cls.nccl(group) if dist.get_backend(group) == "nccl" else cls.host(group)

    def close(self):
        if getattr(self, "h", None):
            lib().atos_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PartGraph:
    """This rank's partition (atos_graph_create_partitioned, collective over `comm`)."""

    def __init__(self, comm: Comm, global_n: int, v_begin: int, v_end: int, local_off, local_col,
                 validate: bool = False, symmetric: bool = False):
        self.comm = comm
        self.global_n, self.v_begin, self.v_end = int(global_n), int(v_begin), int(v_end)
        self.rank, self.world = comm.rank, comm.world
        lo = np.ascontiguousarray(local_off, dtype=np.int64)
        lc = np.ascontiguousarray(local_col, dtype=np.int32)
        self.n = int(lo.shape[0] - 1)
        h = ctypes.c_void_p()
        _check(lib().atos_graph_create_partitioned(comm.h, self.global_n, self.v_begin, self.v_end, lo.ctypes.data,
                                                   lc.ctypes.data if lc.size else None, lc.shape[0],
                                                   (4 if validate else 0) | (8 if symmetric else 0), ctypes.byref(h)),
               "atos_graph_create_partitioned")
        self.h = h

    @classmethod
    def from_global(cls, g, comm: Comm, bounds=None, **kw):
        b = block_bounds(g.n, comm.world) if bounds is None else np.asarray(bounds, dtype=np.int64)
        vb, ve = int(b[comm.rank]), int(b[comm.rank + 1])
        lo, lc = local_csr(g.off, g.col, vb, ve)
        kw.setdefault("symmetric", bool(getattr(g, "symmetric", False)))
        return cls(comm, g.n, vb, ve, lo, lc, **kw)

    def close(self):
        if getattr(self, "h", None):
            lib().atos_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def bfs(pg: PartGraph, src: int, cfg: Config | None = None, device: bool = False, out=None, **kw):
    """Partitioned BFS from GLOBAL vertex src (collective).  Returns (depths of the owned vertices, stats)."""
    c = _cfg(cfg, kw)
    d = _out(pg.n, np.uint32, device, out)
    st = CStats()
    _check(lib().atos_bfs(pg.h, src, ctypes.byref(c), _ptr(d) if pg.n else None, ctypes.byref(st)), "atos_bfs")
    return d, st.to_dict()


def pagerank(pg: PartGraph, alpha: float = 0.85, eps: float = 1e-6, cfg: Config | None = None, device: bool = False,
             out=None, **kw):
    """Partitioned push PageRank (collective).  Returns (ranks of the owned vertices, stats)."""
    c = _cfg(cfg, kw)
    r = _out(pg.n, np.float32, device, out)
    st = CStats()
    _check(lib().atos_pagerank(pg.h, alpha, eps, ctypes.byref(c), _ptr(r) if pg.n else None, ctypes.byref(st)),
           "atos_pagerank")
    return r, st.to_dict()


def color(pg: PartGraph, cfg: Config | None = None, device: bool = False, out=None, **kw):
    """Partitioned speculative greedy colouring of a symmetric graph (collective).
    Returns (colours of the owned vertices, stats); stats["num_colors"] counts all ranks."""
    c = _cfg(cfg, kw)
    col = _out(pg.n, np.int32, device, out)
    k = ctypes.c_int32(0)
    st = CStats()
    _check(lib().atos_color(pg.h, ctypes.byref(c), _ptr(col) if pg.n else None, ctypes.byref(k), ctypes.byref(st)),
           "atos_color")
    d = st.to_dict()
    d["num_colors"] = k.value
    return col, d

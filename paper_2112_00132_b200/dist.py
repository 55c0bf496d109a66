"""Multi-GPU BFS / PageRank over a 1-D vertex partition.

One process per GPU.  Each rank owns a contiguous block of (pre-permuted)
vertex ids and runs the library's persistent queue kernel on it to local
quiescence (``atos_part_run``); remote activations come back as one packed
message buffer per round, exchanged here with ``torch.distributed``
all-to-all (NCCL over NVLink/NVSwitch on GPUs; gloo stages through host memory
for CPU-side tests), applied with ``atos_part_apply``; a round in which no rank
sends anything ends the run.  This module only marshals buffers and issues the
collectives — every update runs in the CUDA kernels.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import CStats, Config, _check, _cfg, lib

APP_BFS, APP_PR, APP_GC = 0, 1, 2


def block_bounds(n: int, world: int) -> np.ndarray:
    """Contiguous block split: rank r owns [bounds[r], bounds[r+1])."""
    return np.array([r * n // world for r in range(world + 1)], dtype=np.int64)


def local_csr(off: np.ndarray, col: np.ndarray, vb: int, ve: int):
    """Rows [vb, ve) of a global CSR as a local CSR with global column ids."""
    lo = np.ascontiguousarray(off[vb:ve + 1] - off[vb], dtype=np.int64)
    lc = np.ascontiguousarray(col[off[vb]:off[ve]], dtype=np.int32)
    return lo, lc


class PartGraph:
    """This rank's partition (atos_graph_create_partitioned)."""

    def __init__(self, global_n: int, world: int, rank: int, bounds, local_off, local_col, validate=False,
                 symmetric=False):
        L = lib()
        self.global_n, self.world, self.rank = int(global_n), int(world), int(rank)
        self.bounds = np.ascontiguousarray(bounds, dtype=np.int64)
        lo = np.ascontiguousarray(local_off, dtype=np.int64)
        lc = np.ascontiguousarray(local_col, dtype=np.int32)
        self.n = int(lo.shape[0] - 1)
        h = ctypes.c_void_p()
        _check(L.atos_graph_create_partitioned(self.global_n, self.world, self.rank, self.bounds.ctypes.data,
                                               lo.ctypes.data, lc.ctypes.data if lc.size else None, lc.shape[0],
                                               (4 if validate else 0) | (8 if symmetric else 0), ctypes.byref(h)),
               "atos_graph_create_partitioned")
        self.h = h

    @classmethod
    def from_global(cls, g, world: int, rank: int, bounds=None, **kw):
        b = block_bounds(g.n, world) if bounds is None else np.asarray(bounds, dtype=np.int64)
        lo, lc = local_csr(g.off, g.col, int(b[rank]), int(b[rank + 1]))
        kw.setdefault("symmetric", bool(getattr(g, "symmetric", False)))
        return cls(g.n, world, rank, b, lo, lc, **kw)

    def close(self):
        if getattr(self, "h", None):
            lib().atos_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ptr(t):
    return t.data_ptr() if hasattr(t, "data_ptr") else t.ctypes.data


def run(pg: PartGraph, app: int, src: int = 0, alpha: float = 0.85, eps: float = 1e-6,
        cfg: Config | None = None, group=None, **kw):
    """Run a partitioned BFS (app 0), PageRank (app 1) or colouring (app 2) on this rank.

    Returns (local result numpy array, stats dict).  Collective: every rank of
    ``group`` must call it with the same arguments."""
    import torch
    import torch.distributed as dist

    L = lib()
    c = _cfg(cfg, kw)
    world = pg.world
    host = (dist.get_backend(group) == "gloo") if world > 1 else True
    dev = torch.device("cpu") if host else torch.device("cuda", torch.cuda.current_device())
    _check(L.atos_part_begin(pg.h, app, src, alpha, eps, ctypes.byref(c)), "atos_part_begin")
    counts_all = np.zeros(world + 1, dtype=np.int64)  # [world] = local tasks still queued
    counts = counts_all[:world]
    flush_all = 0
    while True:
        _check(L.atos_part_run(pg.h, flush_all, counts_all.ctypes.data), "atos_part_run")
        if world == 1:
            if counts_all[world] == 0:
                break
            continue
        send_counts = torch.from_numpy(counts.copy()).to(dev)
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=group)
        total = torch.tensor([int(counts_all.sum())], dtype=torch.int64, device=dev)
        dist.all_reduce(total, group=group)
        if int(total.item()) == 0:
            if app != APP_PR or flush_all:
                break
            flush_all = 1  # PageRank: close with a round that sends every pending contribution
            continue
        flush_all = 0

        ns = int(counts.sum())
        send = torch.empty(max(ns, 1), dtype=torch.int64, device=dev)
        _check(L.atos_part_pack(pg.h, _ptr(send), ns), "atos_part_pack")
        rc = recv_counts.cpu().tolist()
        recv = torch.empty(max(sum(rc), 1), dtype=torch.int64, device=dev)
        dist.all_to_all_single(recv[:sum(rc)], send[:ns], output_split_sizes=rc,
                               input_split_sizes=counts.tolist(), group=group)
        if not host:
            torch.cuda.current_stream().synchronize()
        _check(L.atos_part_apply(pg.h, _ptr(recv), sum(rc)), "atos_part_apply")
    out = np.empty(pg.n, dtype={APP_BFS: np.uint32, APP_PR: np.float32, APP_GC: np.int32}[app])
    st = CStats()
    _check(L.atos_part_finish(pg.h, out.ctypes.data if pg.n else None, ctypes.byref(st)), "atos_part_finish")
    return out, st.to_dict()


def bfs(pg: PartGraph, src: int, cfg: Config | None = None, group=None, **kw):
    return run(pg, APP_BFS, src=src, cfg=cfg, group=group, **kw)


def pagerank(pg: PartGraph, alpha: float = 0.85, eps: float = 1e-6, cfg: Config | None = None, group=None, **kw):
    return run(pg, APP_PR, alpha=alpha, eps=eps, cfg=cfg, group=group, **kw)


def color(pg: PartGraph, cfg: Config | None = None, group=None, **kw):
    """Partitioned speculative greedy colouring of a symmetric
    graph.  Returns (local colours int32[n_local], stats) — stats["num_colors"] is
    the colour count over all ranks (a MAX all-reduce)."""
    import torch
    import torch.distributed as dist

    out, st = run(pg, APP_GC, cfg=cfg, group=group, **kw)
    k = int(out.max()) + 1 if out.size else 0
    if pg.world > 1:
        host = dist.get_backend(group) == "gloo"
        t = torch.tensor([k], dtype=torch.int64,
                         device="cpu" if host else torch.device("cuda", torch.cuda.current_device()))
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        k = int(t.item())
    st["num_colors"] = k
    return out, st

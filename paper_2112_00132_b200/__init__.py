"""paper_2112_00132_b200 — B200-native Atos hot path (arxiv 2112.00132).

Thin Python binding over ``libatos.so`` (C ABI in include/atos.h): argument
marshalling only — every step of BFS / PageRank / colouring runs in the CUDA
kernels of ``csrc/``.  PyTorch supplies device memory, streams and process
groups.  There is no CPU fallback: if the library is missing or no GPU is
present, calls raise.

    import paper_2112_00132_b200 as atos
    g = atos.Graph(off, col)                    # numpy (host) or torch CUDA tensors
    depth, st = atos.bfs(g, 0)                  # persistent CTA workers by default
    rank, st = atos.pagerank(g, 0.85, 1e-6, kernel="discrete", worker="warp")
    color, ncol, st = atos.color(gsym)
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ATOS_LIB selects a tuning variant built by tools/build_variant.py (experiments only; the
# product library is never overwritten)
LIB_PATH = os.environ.get("ATOS_LIB") or os.path.join(_HERE, "libatos.so")

# ---- C enums (include/atos.h) ---------------------------------------------
OK = 0
STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "INVALID_GRAPH", 3: "OUT_OF_MEMORY", 4: "CUDA", 5: "NCCL",
          6: "QUEUE_OVERFLOW", 7: "TIMEOUT", 8: "UNSUPPORTED"}
KERNELS = {"persistent": 0, "discrete": 1, "bsp": 2}
WORKERS = {"thread": 0, "warp": 1, "cta": 2}
GRAPH_DEVICE_PTRS, GRAPH_BORROW, GRAPH_VALIDATE, GRAPH_SYMMETRIC = 1, 2, 4, 8
UNREACHED = 0xFFFFFFFF

EXPORTS = [
    "atos_config_default", "atos_graph_create", "atos_graph_destroy", "atos_graph_info", "atos_bfs",
    "atos_pagerank", "atos_color", "atos_status_string", "atos_last_error", "atos_version",
    "atos_comm_unique_id", "atos_comm_init", "atos_comm_init_host", "atos_comm_info", "atos_comm_destroy",
    "atos_graph_create_partitioned", "atos_graph_create_peer", "atos_pool_trim", "atos_pool_reserved",
]

# callback types of atos_comm_init_host (include/atos.h)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)
ALLTOALLV_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
                                ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64))


class AtosError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{where}: ATOS_ERR_{self.name}: {detail}")


class CConfig(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("kernel", ctypes.c_int32), ("worker", ctypes.c_int32),
                ("cta_threads", ctypes.c_int32), ("fetch_size", ctypes.c_int32), ("num_blocks", ctypes.c_int32),
                ("bfs_filter", ctypes.c_int32), ("pr_activation", ctypes.c_int32), ("check_size", ctypes.c_int32),
                ("gc_literal", ctypes.c_int32), ("pr_residue_fp64", ctypes.c_int32),
                ("adaptive_fetch", ctypes.c_int32), ("device_loop", ctypes.c_int32),
                ("queue_capacity", ctypes.c_int64), ("timeout_s", ctypes.c_double),
                ("stream", ctypes.c_void_p), ("trace", ctypes.c_void_p), ("trace_capacity", ctypes.c_int64),
                ("stage_edges", ctypes.c_int32), ("sink_defer", ctypes.c_int32),
                ("pr_defer_degree", ctypes.c_int32), ("pr_defer_factor", ctypes.c_int32),
                ("hub_split", ctypes.c_int32), ("pr_hub_check", ctypes.c_int32)]


class CStats(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("ms", ctypes.c_double), ("kernel_ms", ctypes.c_double),
                ("kernel_launches", ctypes.c_int64), ("tasks_popped", ctypes.c_int64),
                ("tasks_pushed", ctypes.c_int64), ("edges_processed", ctypes.c_int64), ("rounds", ctypes.c_int64),
                ("queue_high_water", ctypes.c_int64), ("bytes_sent", ctypes.c_int64), ("num_colors", ctypes.c_int32),
                ("_pad", ctypes.c_int32), ("max_residue", ctypes.c_double), ("chunk_tasks", ctypes.c_int64),
                ("trace_records", ctypes.c_int64)]

    def to_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k not in ("struct_size", "_pad")}


_lib = None


def lib():
    """Load libatos.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: build it with `python -c 'import __graft_entry__ as e; e.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
        cfgp, stp = ctypes.POINTER(CConfig), ctypes.POINTER(CStats)
        L.atos_config_default.argtypes = [cfgp]
        L.atos_config_default.restype = None
        L.atos_graph_create.argtypes = [vp, vp, i64, i64, u32, ctypes.POINTER(vp)]
        L.atos_graph_destroy.argtypes = [vp]
        L.atos_graph_info.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.atos_bfs.argtypes = [vp, i64, cfgp, vp, stp]
        L.atos_pagerank.argtypes = [vp, ctypes.c_float, ctypes.c_float, cfgp, vp, stp]
        L.atos_color.argtypes = [vp, cfgp, vp, ctypes.POINTER(i32), stp]
        L.atos_status_string.argtypes = [ctypes.c_int]
        L.atos_status_string.restype = ctypes.c_char_p
        L.atos_last_error.restype = ctypes.c_char_p
        L.atos_version.restype = ctypes.c_char_p
        L.atos_comm_unique_id.argtypes = [vp]
        L.atos_comm_init.argtypes = [i32, i32, vp, ctypes.POINTER(vp)]
        L.atos_comm_init_host.argtypes = [i32, i32, ALLGATHER_FN, ALLTOALLV_FN, vp, ctypes.POINTER(vp)]
        L.atos_comm_info.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)]
        L.atos_comm_destroy.argtypes = [vp]
        L.atos_graph_create_partitioned.argtypes = [vp, i64, i64, i64, vp, vp, i64, u32, ctypes.POINTER(vp)]
        L.atos_graph_create_peer.argtypes = [i32, vp, vp, vp, i64, i64, u32, ctypes.POINTER(vp)]
        L.atos_pool_trim.argtypes = [ctypes.c_uint64]
        L.atos_pool_reserved.argtypes = [ctypes.POINTER(ctypes.c_uint64)]
        for f in ("atos_graph_create", "atos_graph_destroy", "atos_graph_info", "atos_bfs", "atos_pagerank",
                  "atos_color", "atos_comm_unique_id", "atos_comm_init", "atos_comm_init_host", "atos_comm_info",
                  "atos_comm_destroy", "atos_graph_create_partitioned", "atos_graph_create_peer", "atos_pool_trim",
                  "atos_pool_reserved"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(rc: int, where: str):
    if rc != OK:
        raise AtosError(rc, where, lib().atos_last_error().decode(errors="replace"))


def version() -> str:
    return lib().atos_version().decode()


# ---- configuration ---------------------------------------------------------
@dataclass
class Config:
    """Scheduler configuration (the paper's launch* arguments)."""
    kernel: str = "persistent"     # persistent | discrete | bsp
    worker: str = "cta"            # thread | warp | cta
    cta_threads: int = 256         # numThread
    fetch_size: int = 256          # FETCH_SIZE
    num_blocks: int = 0            # numBlock (0 = resident maximum)
    bfs_filter: bool = True
    pr_activation: int = 0
    check_size: int = 32
    gc_literal: bool = False
    pr_residue_fp64: bool = False  # fp64 residues (see engine.cuh PrAppT)
    adaptive_fetch: bool = True    # pop min(FETCH, ceil(queued/workers))
    device_loop: bool = False      # discrete rounds driven on the device (CUDA-graph WHILE node)
    queue_capacity: int = 0
    timeout_s: float = 60.0
    stream: int | None = None      # raw cudaStream_t; None = torch current stream
    trace: object = None           # Trace() buffer for the timeline, or None
    stage_edges: int = 0           # TMA column staging per batch buffer (edges); 0 off, -1 auto
    sink_defer: bool = True        # never push dangling vertices (BFS: no-op tasks; PR: one final pass) (R29)
    pr_defer_degree: int = 0       # PR hub deferral (R31): min out-degree; 0 = off
    pr_defer_factor: int = 4       # ... defer while residue < factor * eps
    hub_split: int = -1            # hub chunk tasks (R24): -1 app default (BFS on, PR off, R33), 0 off, 1 on
    pr_hub_check: int = 4          # PR hubs activated by sweeps, hubs checked per batch (R35); 0 = off (R34)

    def to_c(self) -> CConfig:
        c = CConfig()
        lib().atos_config_default(ctypes.byref(c))
        c.kernel = KERNELS[self.kernel]
        c.worker = WORKERS[self.worker]
        c.cta_threads = self.cta_threads
        c.fetch_size = self.fetch_size
        c.num_blocks = self.num_blocks
        c.bfs_filter = int(self.bfs_filter)
        c.pr_activation = self.pr_activation
        c.check_size = self.check_size
        c.gc_literal = int(self.gc_literal)
        c.pr_residue_fp64 = int(self.pr_residue_fp64)
        c.adaptive_fetch = int(self.adaptive_fetch)
        c.device_loop = int(self.device_loop)
        c.queue_capacity = self.queue_capacity
        c.timeout_s = self.timeout_s
        c.stage_edges = self.stage_edges
        c.sink_defer = int(self.sink_defer)
        c.pr_defer_degree = self.pr_defer_degree
        c.pr_defer_factor = self.pr_defer_factor
        c.hub_split = self.hub_split
        c.pr_hub_check = self.pr_hub_check
        s = self.stream
        if s is None:
            import torch
            if torch.cuda.is_available():
                s = torch.cuda.current_stream().cuda_stream
        c.stream = s or None
        if self.trace is not None:
            c.trace = self.trace.buf.data_ptr()
            c.trace_capacity = self.trace.capacity
        return c


def _cfg(cfg: Config | None, kw) -> CConfig:
    cfg = cfg or Config()
    if kw:
        cfg = Config(**{**cfg.__dict__, **kw})
    return cfg.to_c()


class Trace:
    """Device timeline buffer (atos_trace_rec records, one per processed batch).

    After a call with ``Config(trace=tr)``: ``tr.records(stats)`` returns a
    numpy structured array (t_ns, items, edges, sm, kind) sorted by time — the
    cumulative-work-vs-time view of the paper's Figs. 4-6."""
    DTYPE = np.dtype([("t_ns", "<u8"), ("items", "<u4"), ("edges", "<u4"), ("sm", "<u4"), ("kind", "<u4")])

    def __init__(self, capacity: int = 1 << 20):
        import torch
        self.capacity = int(capacity)
        self.buf = torch.zeros(self.capacity * 24, dtype=torch.uint8, device="cuda")

    def records(self, stats: dict):
        k = min(int(stats.get("trace_records", 0)), self.capacity)
        raw = self.buf[: k * 24].cpu().numpy()
        r = raw.view(self.DTYPE)
        return np.sort(r, order="t_ns")


# ---- graph -----------------------------------------------------------------
class Graph:
    """Device CSR graph handle (atos_graph_create).

    ``off`` int64[n+1] and ``col`` int32[m]: numpy arrays (copied host->device)
    or torch CUDA tensors (borrowed zero-copy; the tensors are kept alive)."""

    def __init__(self, off, col, symmetric: bool = False, validate: bool = False):
        self._keep = None
        flags = (GRAPH_SYMMETRIC if symmetric else 0) | (GRAPH_VALIDATE if validate else 0)
        try:
            import torch
            is_t = isinstance(off, torch.Tensor)
        except ImportError:  # pragma: no cover
            is_t = False
        if is_t:
            if off.dtype != torch.int64 or col.dtype != torch.int32 or not off.is_cuda or not col.is_cuda:
                raise TypeError("torch inputs must be CUDA int64 offsets and int32 columns")
            off, col = off.contiguous(), col.contiguous()
            self._keep = (off, col)
            flags |= GRAPH_DEVICE_PTRS | GRAPH_BORROW
            po, pc, n, m = off.data_ptr(), col.data_ptr(), off.numel() - 1, col.numel()
        else:
            off = np.ascontiguousarray(off, dtype=np.int64)
            col = np.ascontiguousarray(col, dtype=np.int32)
            self._keep = (off, col)
            po, pc, n, m = off.ctypes.data, col.ctypes.data, off.shape[0] - 1, col.shape[0]
        h = ctypes.c_void_p()
        _check(lib().atos_graph_create(po, pc or None, n, m, flags, ctypes.byref(h)), "atos_graph_create")
        self.h = h
        self.n, self.m = int(n), int(m)
        self.symmetric = symmetric
        if not is_t:
            self._keep = None  # copied; host arrays may be freed

    @classmethod
    def peer(cls, off, col, parts: int, devices=None, validate: bool = False):
        """Asynchronous peer-memory partitions (atos_graph_create_peer): `parts`
        contiguous vertex blocks on `devices` (None: all on the current device, one launch over
        every partition).  atos_bfs / atos_pagerank run with no exchange rounds."""
        self = cls.__new__(cls)
        off = np.ascontiguousarray(off, dtype=np.int64)
        col = np.ascontiguousarray(col, dtype=np.int32)
        dv = None if devices is None else np.ascontiguousarray(devices, dtype=np.int32)
        h = ctypes.c_void_p()
        _check(lib().atos_graph_create_peer(parts, dv.ctypes.data if dv is not None else None, off.ctypes.data,
                                            col.ctypes.data if col.size else None, off.shape[0] - 1, col.shape[0],
                                            GRAPH_VALIDATE if validate else 0, ctypes.byref(h)),
               "atos_graph_create_peer")
        self._keep = None
        self.h = h
        self.n, self.m = int(off.shape[0] - 1), int(col.shape[0])
        self.symmetric = False
        return self

    @classmethod
    def from_csr(cls, g, **kw):
        """From a graphgen.CSR-like object with .off/.col."""
        return cls(g.off, g.col, symmetric=kw.pop("symmetric", getattr(g, "symmetric", False)), **kw)

    def info(self):
        n, m, d = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().atos_graph_info(self.h, ctypes.byref(n), ctypes.byref(m), ctypes.byref(d)), "atos_graph_info")
        return n.value, m.value, d.value

    def close(self):
        if getattr(self, "h", None):
            lib().atos_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _out(n: int, dtype, device: bool, out):
    if out is not None:
        return out
    if device:
        import torch
        tdt = {np.uint32: torch.int32, np.float32: torch.float32, np.int32: torch.int32}[dtype]
        return torch.empty(n, dtype=tdt, device="cuda")
    return np.empty(n, dtype=dtype)


def _ptr(a):
    return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data


def bfs(g: Graph, src: int, cfg: Config | None = None, device: bool = False, out=None, **kw):
    """Speculative BFS (Alg. 2).  Returns (depth uint32[n] — a torch int32 view
    when device=True — , stats dict).  Unreachable = 0xFFFFFFFF."""
    c = _cfg(cfg, kw)
    d = _out(g.n, np.uint32, device, out)
    st = CStats()
    _check(lib().atos_bfs(g.h, src, ctypes.byref(c), _ptr(d) if g.n else None, ctypes.byref(st)), "atos_bfs")
    return d, st.to_dict()


def pagerank(g: Graph, alpha: float = 0.85, eps: float = 1e-6, cfg: Config | None = None, device: bool = False,
             out=None, **kw):
    """Push PageRank (Alg. 4; BSP Alg. 3).  Returns (rank float32[n], stats)."""
    c = _cfg(cfg, kw)
    r = _out(g.n, np.float32, device, out)
    st = CStats()
    _check(lib().atos_pagerank(g.h, alpha, eps, ctypes.byref(c), _ptr(r) if g.n else None, ctypes.byref(st)),
           "atos_pagerank")
    return r, st.to_dict()


def color(g: Graph, cfg: Config | None = None, device: bool = False, out=None, **kw):
    """Speculative greedy colouring (Alg. 6; BSP Alg. 5).  Returns (color int32[n], ncolors, stats)."""
    c = _cfg(cfg, kw)
    col = _out(g.n, np.int32, device, out)
    k = ctypes.c_int32(0)
    st = CStats()
    _check(lib().atos_color(g.h, ctypes.byref(c), _ptr(col) if g.n else None, ctypes.byref(k), ctypes.byref(st)),
           "atos_color")
    return col, k.value, st.to_dict()


def pool_trim(keep_bytes: int = 0):
    """Release the library's retained graph memory down to keep_bytes (atos_pool_trim)."""
    _check(lib().atos_pool_trim(keep_bytes), "atos_pool_trim")


def pool_reserved() -> int:
    v = ctypes.c_uint64()
    _check(lib().atos_pool_reserved(ctypes.byref(v)), "atos_pool_reserved")
    return v.value


__all__ = ["pool_trim", "pool_reserved", "Graph", "Config", "Trace", "bfs", "pagerank", "color", "AtosError", "lib", "version", "UNREACHED", "EXPORTS"]

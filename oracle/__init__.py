"""CPU oracle for the Atos hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2112_00132_b200``) never imports it and shares no code with it.

Each function is a plain definition from the paper (arxiv 2112.00132,
PAPER.md cited as P:n) written in serial C (oracle.c), fp64 for PageRank.
Parity pins live in tests/test_oracle_pins.py.  All functions here are pinned
(see oracle.c header); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

UNREACHED = 0xFFFFFFFF  # P:421 MAX_UINT32


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        vp, i64, dbl, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        lib.or_bfs.restype = ci
        lib.or_bfs.argtypes = [i64, vp, vp, i64, vp]
        lib.or_pagerank_jacobi.restype = ci
        lib.or_pagerank_jacobi.argtypes = [i64, vp, vp, dbl, dbl, ci, ci, vp]
        lib.or_pagerank_push.restype = ci
        lib.or_pagerank_push.argtypes = [i64, vp, vp, dbl, dbl, vp, vp, vp, vp]
        lib.or_greedy_color.restype = ci
        lib.or_greedy_color.argtypes = [i64, vp, vp, vp]
        lib.or_check_bfs.restype = i64
        lib.or_check_bfs.argtypes = [i64, vp, vp, i64, vp, vp]
        lib.or_check_coloring.restype = i64
        lib.or_check_coloring.argtypes = [i64, vp, vp, vp, vp, vp]
        _lib = lib
    return _lib


def _csr(g):
    off = np.ascontiguousarray(g.off, dtype=np.int64)
    col = np.ascontiguousarray(g.col, dtype=np.int32)
    return off.shape[0] - 1, off, col


def bfs(g, src: int) -> np.ndarray:
    """Serial FIFO BFS depths (uint32; unreachable = 0xFFFFFFFF). P:417-434."""
    n, off, col = _csr(g)
    d = np.empty(n, dtype=np.uint32)
    if _load().or_bfs(n, off.ctypes.data, col.ctypes.data, src, d.ctypes.data) != 0:
        raise ValueError("or_bfs: bad arguments")
    return d


def pagerank(g, alpha: float = 0.85, tol: float = 1e-10, max_iter: int = 10000, threads: int = 0):
    """fp64 Jacobi fixed point of x = (1-a)1 + a P x. Returns (x, iterations). P:481-505."""
    n, off, col = _csr(g)
    x = np.empty(n, dtype=np.float64)
    it = _load().or_pagerank_jacobi(n, off.ctypes.data, col.ctypes.data, alpha, tol, max_iter, threads,
                                    x.ctypes.data)
    if it < 0:
        raise ValueError("or_pagerank_jacobi failed")
    return x, it


def pagerank_push(g, alpha: float = 0.85, eps: float = 1e-6):
    """Serial fp64 push PageRank (Alg. 4 with one worker, threshold activation).

    Returns (rank, residue, pops, edge_pushes)."""
    n, off, col = _csr(g)
    r = np.empty(n, dtype=np.float64)
    s = np.empty(n, dtype=np.float64)
    pops = ctypes.c_int64(0)
    pushes = ctypes.c_int64(0)
    rc = _load().or_pagerank_push(n, off.ctypes.data, col.ctypes.data, alpha, eps, r.ctypes.data, s.ctypes.data,
                                  ctypes.addressof(pops), ctypes.addressof(pushes))
    if rc != 0:
        raise ValueError("or_pagerank_push failed")
    return r, s, pops.value, pushes.value


def greedy_color(g):
    """Serial first-fit colouring in id order. Returns (color int32[n], ncolors). P:560-623."""
    n, off, col = _csr(g)
    c = np.empty(n, dtype=np.int32)
    k = _load().or_greedy_color(n, off.ctypes.data, col.ctypes.data, c.ctypes.data)
    if k < 0:
        raise MemoryError("or_greedy_color failed")
    return c, k


def check_bfs(g, src: int, depth) -> int:
    """Number of BFS-certificate violations (0 = valid depth labelling)."""
    n, off, col = _csr(g)
    d = np.ascontiguousarray(depth, dtype=np.uint32)
    bad = ctypes.c_int64(-1)
    return int(_load().or_check_bfs(n, off.ctypes.data, col.ctypes.data, src, d.ctypes.data, ctypes.addressof(bad)))


def check_coloring(g, color):
    """Returns (violations, ncolors): monochromatic edges + out-of-range colours."""
    n, off, col = _csr(g)
    c = np.ascontiguousarray(color, dtype=np.int32)
    k = ctypes.c_int32(0)
    bad = ctypes.c_int64(-1)
    v = _load().or_check_coloring(n, off.ctypes.data, col.ctypes.data, c.ctypes.data, ctypes.addressof(k),
                                  ctypes.addressof(bad))
    return int(v), int(k.value)

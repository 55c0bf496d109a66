"""Seeded synthetic graph inputs shared by the oracle and the CUDA path.

Holds none of the Atos method's arithmetic (arxiv 2112.00132): it only builds
CSR graphs shaped like the paper's workloads (tbl:dataset)
— RMAT/Kronecker scale-free graphs and 2-D grid / road-like meshes.  The C
generator (gen.c) is deterministic for a seed, independent of thread count.

Every graph is returned as ``(row_offsets: int64[n+1], col: int32[m])`` numpy
arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libgraphgen.so")
_lib = None

GRAPH500_ABC = (0.57, 0.19, 0.19)


def build(force: bool = False) -> str:
    """Compile gen.c into libgraphgen.so (gcc -O3 -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        vp, i64, u64, dbl, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_int
        lib.gg_n.restype = i64
        lib.gg_n.argtypes = [vp]
        lib.gg_m.restype = i64
        lib.gg_m.argtypes = [vp]
        lib.gg_copy.argtypes = [vp, vp, vp]
        lib.gg_free.argtypes = [vp]
        lib.gg_set_threads.argtypes = [ci]
        lib.gg_grid.restype = vp
        lib.gg_grid.argtypes = [i64, i64, dbl, u64]
        lib.gg_rmat.restype = vp
        lib.gg_rmat.argtypes = [ci, i64, u64, dbl, dbl, dbl, ci, u64]
        lib.gg_from_edges.restype = vp
        lib.gg_from_edges.argtypes = [i64, i64, vp, vp, ci]
        lib.gg_permute.restype = vp
        lib.gg_permute.argtypes = [i64, vp, vp, u64, vp]
        _lib = lib
    return _lib


@dataclass
class CSR:
    """Host CSR graph: ``off`` int64[n+1], ``col`` int32[m]."""
    off: np.ndarray
    col: np.ndarray
    name: str = ""
    symmetric: bool = False

    @property
    def n(self) -> int:
        return int(self.off.shape[0] - 1)

    @property
    def m(self) -> int:
        return int(self.col.shape[0])

    def degrees(self) -> np.ndarray:
        return np.diff(self.off)


def _take(h, name: str, symmetric: bool) -> CSR:
    lib = _load()
    if not h:
        raise MemoryError(f"graphgen: generator failed for {name}")
    try:
        n, m = lib.gg_n(h), lib.gg_m(h)
        off = np.empty(n + 1, dtype=np.int64)
        col = np.empty(m, dtype=np.int32)
        lib.gg_copy(h, off.ctypes.data, col.ctypes.data)
    finally:
        lib.gg_free(h)
    return CSR(off, col, name, symmetric)


def grid(rows: int, cols: int, drop_prob: float = 0.0, seed: int = 0) -> CSR:
    """2-D lattice, 4-neighbourhood, both directions, row-major ids.

    ``drop_prob`` > 0 gives the road-like variant (each undirected edge deleted
    independently, seeded)."""
    h = _load().gg_grid(rows, cols, float(drop_prob), seed)
    return _take(h, f"grid{rows}x{cols}" + (f"_drop{drop_prob}" if drop_prob else ""), True)


def rmat(scale: int, edge_factor: int = 16, seed: int = 1, abc=GRAPH500_ABC,
         symmetrize: bool = False, perm_seed: int = 0) -> CSR:
    """RMAT/Kronecker graph, 2^scale vertices, edge_factor*2^scale tuples (Graph500 a,b,c,d)."""
    a, b, c = abc
    h = _load().gg_rmat(scale, edge_factor, seed, a, b, c, int(symmetrize), perm_seed)
    nm = f"rmat{scale}_ef{edge_factor}_s{seed}" + ("_sym" if symmetrize else "") + (f"_p{perm_seed}" if perm_seed else "")
    return _take(h, nm, symmetrize)


def from_edges(n: int, edges, symmetrize: bool = False, name: str = "edges") -> CSR:
    """CSR from an explicit edge list (self-loops dropped, rows sorted/deduped)."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    if e.size and (e.min() < 0 or e.max() >= n):
        raise ValueError("edge endpoint out of range")
    src = np.ascontiguousarray(e[:, 0], dtype=np.uint32)
    dst = np.ascontiguousarray(e[:, 1], dtype=np.uint32)
    h = _load().gg_from_edges(n, len(src), src.ctypes.data, dst.ctypes.data, int(symmetrize))
    return _take(h, name, symmetrize)


def fan_in(k: int, fan: int = 64) -> CSR:
    """Fan-in hub: k sources s -> 0 and s -> s+1 (a chain, so every source has
    out-degree 2, the last one 1), plus 0 -> 1..fan.  Vertex 0 receives k equal
    pushes per sweep (the adversarial case for fp32 residue accumulation)."""
    s = np.arange(1, k + 1, dtype=np.int64)
    e = np.concatenate([np.stack([s, np.zeros(k, np.int64)], 1), np.stack([s[:-1], s[:-1] + 1], 1),
                        np.stack([np.zeros(fan, np.int64), np.arange(1, fan + 1, dtype=np.int64)], 1)])
    return from_edges(k + 1, e, name=f"fanin{k}")


def permute(g: CSR, perm_seed: int):
    """Relabel by a seeded uniform permutation; returns (graph, forward) where forward[old] = new."""
    fwd = np.empty(g.n, dtype=np.int32)
    h = _load().gg_permute(g.n, g.off.ctypes.data, g.col.ctypes.data, perm_seed, fwd.ctypes.data)
    return _take(h, g.name + f"_p{perm_seed}", g.symmetric), fwd


# ---- small named graphs (test fixtures) ---------------------------------

def path(k: int) -> CSR:
    """Undirected path 0-1-...-(k-1)."""
    return from_edges(k, [(i, i + 1) for i in range(k - 1)], symmetrize=True, name=f"path{k}")


def directed_chain(k: int) -> CSR:
    """Directed chain 0->1->...->(k-1)."""
    return from_edges(k, [(i, i + 1) for i in range(k - 1)], name=f"chain{k}")


def star(leaves: int) -> CSR:
    """Undirected star, centre 0, leaves 1..leaves."""
    return from_edges(leaves + 1, [(0, i) for i in range(1, leaves + 1)], symmetrize=True, name=f"star{leaves}")


def complete(k: int) -> CSR:
    """Complete graph K_k (both directions)."""
    return from_edges(k, [(i, j) for i in range(k) for j in range(k) if i != j], name=f"K{k}", symmetrize=True)


def cycle(k: int, directed: bool = False) -> CSR:
    return from_edges(k, [(i, (i + 1) % k) for i in range(k)], symmetrize=not directed,
                      name=("dcycle" if directed else "cycle") + str(k))


def empty(n: int) -> CSR:
    return CSR(np.zeros(n + 1, dtype=np.int64), np.zeros(0, dtype=np.int32), f"empty{n}", True)


def random_digraph(n: int, p: float, seed: int) -> CSR:
    """Erdos-Renyi directed graph (numpy seeded); for brute-force pins."""
    rng = np.random.default_rng(seed)
    a = rng.random((n, n)) < p
    np.fill_diagonal(a, False)
    s, d = np.nonzero(a)
    return from_edges(n, np.stack([s, d], 1), name=f"er{n}_{seed}")


def hub_graph(n_leaves: int, extra: int = 0) -> CSR:
    """Directed fan-out hub 0 -> 1..n_leaves plus a chain among the leaves
    (a hub with degree above CTA x FETCH, SURVEY §4 layer 2)."""
    e = [(0, i) for i in range(1, n_leaves + 1)]
    e += [(i, i + 1) for i in range(1, min(n_leaves, 1 + extra))]
    return from_edges(n_leaves + 1, e, name=f"hub{n_leaves}")

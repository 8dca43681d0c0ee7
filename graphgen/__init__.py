"""Seeded synthetic graph inputs (SURVEY.md §2.5 M1, §8(d) input recipe).

This module is shared by the oracle tests, the GPU parity tests and ``bench.py``.  It holds
none of DAWN's arithmetic (no frontier, no distances): it only generates normalised CSR
arrays, their transpose, the largest-WCC source set and seeded source samples.

All arrays are numpy: ``row_ptr`` int64[n+1], ``col`` int32[m]; rows sorted, no self-loops,
no duplicates.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "graphgen.cpp")
_LIB = os.path.join(_HERE, "libgraphgen.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile libgraphgen.so in-tree (g++ -O3, pthreads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O3", "-march=x86-64-v2", "-std=c++17", "-shared", "-fPIC",
                               "-pthread", _SRC, "-o", _LIB + ".tmp"])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        vp, i64, i32p, i64p = ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p
        L.gg_n.restype = i64; L.gg_n.argtypes = [vp]
        L.gg_m.restype = i64; L.gg_m.argtypes = [vp]
        L.gg_copy.restype = None; L.gg_copy.argtypes = [vp, i64p, i32p]
        L.gg_free.restype = None; L.gg_free.argtypes = [vp]
        L.gg_from_edges.restype = vp
        L.gg_from_edges.argtypes = [i64, i64, i32p, i32p, ctypes.c_int]
        L.gg_kron.restype = vp
        L.gg_kron.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_int]
        L.gg_er.restype = vp; L.gg_er.argtypes = [i64, i64, ctypes.c_uint64]
        L.gg_grid.restype = vp; L.gg_grid.argtypes = [i64, i64]
        L.gg_transpose.restype = None
        L.gg_transpose.argtypes = [i64, i64, i64p, i32p, i64p, i32p]
        L.gg_wcc_largest.restype = i64
        L.gg_wcc_largest.argtypes = [i64, i64p, i32p, i32p, ctypes.POINTER(ctypes.c_int64)]
        L.gg_weights.restype = None
        L.gg_weights.argtypes = [i64, i64p, i32p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int,
                                 vp]
        L.gg_sample_sources.restype = i64
        L.gg_sample_sources.argtypes = [i64, i64p, i64, ctypes.c_uint64, i32p]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Graph:
    """Normalised directed CSR (symmetric graphs store both arcs)."""
    n: int
    row_ptr: np.ndarray   # int64[n+1]
    col: np.ndarray       # int32[m]
    symmetric: bool
    name: str = ""

    @property
    def m(self) -> int:
        return int(self.row_ptr[-1])

    def degrees(self) -> np.ndarray:
        return np.diff(self.row_ptr)

    def transpose(self) -> tuple[np.ndarray, np.ndarray]:
        """CSC (in-edges): (col_ptr int64[n+1], row int32[m])."""
        if self.symmetric:
            return self.row_ptr, self.col
        L = _load()
        ptr = np.empty(self.n + 1, np.int64)
        idx = np.empty(self.m, np.int32)
        L.gg_transpose(self.n, self.m, _ptr(self.row_ptr), _ptr(self.col), _ptr(ptr), _ptr(idx))
        return ptr, idx

    def largest_wcc(self) -> tuple[np.ndarray, int]:
        """(vertices of the largest WCC ascending, E_wcc) — SURVEY Q15."""
        L = _load()
        out = np.empty(self.n, np.int32)
        e = ctypes.c_int64(0)
        k = L.gg_wcc_largest(self.n, _ptr(self.row_ptr), _ptr(self.col), _ptr(out),
                             ctypes.byref(e))
        return out[:k].copy(), int(e.value)

    def weights(self, seed: int = 1, wmax: int = 255) -> np.ndarray:
        """Seeded integer arc weights in [1, wmax] aligned with col (uint32[m]); both arcs of a
        symmetric graph's edge get the same weight."""
        w = np.empty(self.m, np.uint32)
        _load().gg_weights(self.n, _ptr(self.row_ptr), _ptr(self.col), seed, wmax,
                           1 if self.symmetric else 0, _ptr(w))
        return w

    def sample_sources(self, k: int, seed: int = 1) -> np.ndarray:
        """k seeded sources, uniform over vertices with out-degree > 0."""
        L = _load()
        out = np.empty(k, np.int32)
        got = L.gg_sample_sources(self.n, _ptr(self.row_ptr), k, seed, _ptr(out))
        return out[:got].copy()


def _take(h, symmetric: bool, name: str) -> Graph:
    L = _load()
    if not h:
        raise ValueError("graphgen: invalid arguments")
    n, m = L.gg_n(h), L.gg_m(h)
    row_ptr = np.empty(n + 1, np.int64)
    col = np.empty(m, np.int32)
    L.gg_copy(h, _ptr(row_ptr), _ptr(col))
    L.gg_free(h)
    return Graph(n, row_ptr, col, symmetric, name)


def from_edges(n: int, edges, symmetric: bool = False, name: str = "") -> Graph:
    e = np.asarray(edges, dtype=np.int32).reshape(-1, 2)
    src = np.ascontiguousarray(e[:, 0])
    dst = np.ascontiguousarray(e[:, 1])
    h = _load().gg_from_edges(n, len(e), _ptr(src), _ptr(dst), 1 if symmetric else 0)
    return _take(h, symmetric, name)


def kron(scale: int, edge_factor: int = 16, seed: int | None = None) -> Graph:
    """Graph500 Kronecker, symmetrised; default seed = scale (SURVEY §8(d) seeds)."""
    seed = scale if seed is None else seed
    h = _load().gg_kron(scale, edge_factor, seed, 1)
    return _take(h, True, f"kron{scale}_ef{edge_factor}_s{seed}")


def er(n: int, m: int, seed: int = 1) -> Graph:
    """Directed Erdos-Renyi G(n, m) (configs[0]: n=1000, m=8000)."""
    return _take(_load().gg_er(n, m, seed), False, f"er{n}_{m}_s{seed}")


def grid(W: int, H: int | None = None) -> Graph:
    H = W if H is None else H
    return _take(_load().gg_grid(W, H), True, f"grid{W}x{H}")


def er_prob(n: int, p: float, seed: int) -> Graph:
    """Directed G(n, p) for the property corpus, via numpy's seeded PCG64."""
    rng = np.random.default_rng(seed)
    a = rng.random((n, n)) < p
    np.fill_diagonal(a, False)
    u, v = np.nonzero(a)
    return from_edges(n, np.stack([u, v], 1) if len(u) else np.zeros((0, 2), np.int32),
                      False, f"gnp{n}_{p}_s{seed}")


# ---------------------------------------------------------------- the five BASELINE configs
CONFIGS = {
    "C1": "SSSP from vertex 0, directed ER n=1000 m=8000 (seed 1)",
    "C2": "SSSP, Graph500 Kronecker scale 20 ef 16 (seed 20), 64 sources",
    "C3": "SSSP from vertex 0 on the 4096x4096 grid",
    "C4": "SSSP, Graph500 Kronecker scale 24 ef 16 (seed 24), 64 sources",
    "C5": "APSP over the largest WCC of Kronecker scale 18 ef 16 (seed 18)",
}


def config_graph(name: str) -> Graph:
    if name == "C1":
        return er(1000, 8000, 1)
    if name == "C2":
        return kron(20, 16, 20)
    if name == "C3":
        return grid(4096, 4096)
    if name == "C4":
        return kron(24, 16, 24)
    if name == "C5":
        return kron(18, 16, 18)
    raise KeyError(name)

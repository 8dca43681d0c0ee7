"""CPU oracle for DAWN unweighted shortest paths — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2208_04514_b200``) never imports it, and it never imports the product path.

Thin ctypes wrapper over ``oracle.c`` (plain C, built with gcc); see the header of
``oracle.c`` for the paper passage each function follows.  Parity pins live in
``tests/test_oracle.py``; DESIGN.md lists the readings (Q1-Q25) they rely on.
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

UNREACHED = 0xFFFFFFFF
REC_DTYPE = np.dtype([("source", "<u4"), ("ecc", "<u4"), ("reached", "<u4"), ("pad", "<u4"),
                      ("sum_dist", "<u8"), ("hash", "<u8")])


class _Stats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_uint32), ("rounds", ctypes.c_uint32),
                ("edge_inspections", ctypes.c_uint64), ("node_inspections", ctypes.c_uint64)]


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc -O2; plain C, pthreads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread", _SRC,
                               "-o", _LIB + ".tmp"])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        for name in ("oracle_sovm", "oracle_bovm", "oracle_bfs_fifo"):
            f = getattr(L, name)
            f.restype = ctypes.c_int
            f.argtypes = [i64, vp, vp, i64, vp, ctypes.POINTER(_Stats)]
        L.oracle_floyd_warshall.restype = ctypes.c_int
        L.oracle_floyd_warshall.argtypes = [i64, vp, vp, vp]
        L.oracle_first_hit.restype = ctypes.c_int
        L.oracle_first_hit.argtypes = [i64, vp, vp, vp, i64, vp]
        L.oracle_record.restype = None
        L.oracle_record.argtypes = [i64, vp, i64, vp, vp, ctypes.POINTER(ctypes.c_uint64)]
        L.oracle_certify.restype = ctypes.c_int
        L.oracle_certify.argtypes = [i64, vp, vp, vp, vp, i64, vp, ctypes.POINTER(ctypes.c_int64)]
        L.oracle_records.restype = ctypes.c_int
        L.oracle_records.argtypes = [i64, vp, vp, i64, vp, ctypes.c_int, vp]
        L.oracle_largest_wcc.restype = ctypes.c_int64
        L.oracle_largest_wcc.argtypes = [i64, vp, vp, vp, ctypes.POINTER(ctypes.c_uint64)]
        L.oracle_minplus.restype = ctypes.c_int
        L.oracle_minplus.argtypes = [i64, vp, vp, vp, i64, vp, ctypes.POINTER(_Stats)]
        L.oracle_dijkstra.restype = ctypes.c_int
        L.oracle_dijkstra.argtypes = [i64, vp, vp, vp, i64, vp]
        L.oracle_floyd_warshall_w.restype = ctypes.c_int
        L.oracle_floyd_warshall_w.argtypes = [i64, vp, vp, vp, vp]
        L.oracle_certify_w.restype = ctypes.c_int
        L.oracle_certify_w.argtypes = [i64, vp, vp, vp, i64, vp, ctypes.POINTER(ctypes.c_int64)]
        L.oracle_hash_term.restype = ctypes.c_uint64
        L.oracle_hash_term.argtypes = [ctypes.c_uint32, ctypes.c_uint32]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def _csr(row_ptr, col):
    return (np.ascontiguousarray(row_ptr, dtype=np.int64),
            np.ascontiguousarray(col, dtype=np.int32))


def _run(fname, n, ptr, idx, s):
    ptr, idx = _csr(ptr, idx)
    dist = np.empty(n, np.uint32)
    st = _Stats()
    rc = getattr(_load(), fname)(n, _p(ptr), _p(idx), s, _p(dist), ctypes.byref(st))
    if rc:
        raise ValueError(f"{fname}: error {rc}")
    return dist, {"iterations": st.iterations, "rounds": st.rounds,
                  "edge_inspections": st.edge_inspections,
                  "node_inspections": st.node_inspections}


def sovm(n, row_ptr, col, s):
    """Algorithm 2 (SOVM) literally; returns (dist uint32[n], stats)."""
    return _run("oracle_sovm", n, row_ptr, col, s)


def bovm(n, col_ptr, row, s):
    """Algorithm 1 (BOVM) on CSC; returns (dist uint32[n], stats)."""
    return _run("oracle_bovm", n, col_ptr, row, s)


def bfs_fifo(n, row_ptr, col, s):
    """Algorithm 3 (General BFS, FIFO); returns (dist uint32[n], stats)."""
    return _run("oracle_bfs_fifo", n, row_ptr, col, s)


def floyd_warshall(n, row_ptr, col):
    ptr, idx = _csr(row_ptr, col)
    D = np.empty((n, n), np.uint32)
    if _load().oracle_floyd_warshall(n, _p(ptr), _p(idx), _p(D)):
        raise ValueError("floyd_warshall: n must be in [1, 512]")
    return D


def first_hit(n, row_ptr, col, kq: int = 0):
    """Theorem 1 distances via saturating matrix powers (n <= 32); optionally A^kq."""
    ptr, idx = _csr(row_ptr, col)
    D = np.empty((n, n), np.uint32)
    C = np.zeros((n, n), np.uint64)
    if _load().oracle_first_hit(n, _p(ptr), _p(idx), _p(D), kq, _p(C)):
        raise ValueError("first_hit: n must be in [1, 32]")
    return (D, C) if kq else D


def record(n, row_ptr, s, dist):
    """(record as a REC_DTYPE scalar array, edges_reach)."""
    ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    dist = np.ascontiguousarray(dist, dtype=np.uint32)
    out = np.zeros(1, REC_DTYPE)
    er = ctypes.c_uint64(0)
    _load().oracle_record(n, _p(ptr), s, _p(dist), _p(out), ctypes.byref(er))
    return out[0], int(er.value)


def certify(n, row_ptr, col, in_ptr, in_idx, s, dist):
    """0 if dist is the exact BFS vector of s, else (invariant number, vertex)."""
    ptr, idx = _csr(row_ptr, col)
    iptr, iidx = _csr(in_ptr, in_idx)
    dist = np.ascontiguousarray(dist, dtype=np.uint32)
    bad = ctypes.c_int64(-1)
    rc = _load().oracle_certify(n, _p(ptr), _p(idx), _p(iptr), _p(iidx), s, _p(dist),
                                ctypes.byref(bad))
    return 0 if rc == 0 else (rc, int(bad.value))


def records(n, row_ptr, col, sources, threads: int | None = None):
    """oracle_sovm + record for every source, on a pthread pool -> REC_DTYPE[k]."""
    ptr, idx = _csr(row_ptr, col)
    src = np.ascontiguousarray(sources, dtype=np.int32)
    out = np.zeros(len(src), REC_DTYPE)
    threads = threads or len(os.sched_getaffinity(0))
    rc = _load().oracle_records(n, _p(ptr), _p(idx), len(src), _p(src), threads, _p(out))
    if rc:
        raise ValueError(f"oracle_records: error {rc}")
    return out


def largest_wcc(n, row_ptr, col):
    """(vertices of the largest WCC ascending as int64[S_wcc], E_wcc): PAPER Table 1,
    "largest" per reading Q15 (most nodes, then most arcs, then the smaller minimum id)."""
    ptr, idx = _csr(row_ptr, col)
    out = np.empty(max(1, n), np.int64)
    arcs = ctypes.c_uint64(0)
    k = _load().oracle_largest_wcc(n, _p(ptr), _p(idx), _p(out), ctypes.byref(arcs))
    if k < 0:
        raise MemoryError("oracle_largest_wcc")
    return out[:k].copy(), int(arcs.value)


def hash_term(v: int, d: int) -> int:
    return int(_load().oracle_hash_term(v, d))


# ------------------------------------------------------------------ weighted (min,+), NEXT-4
UNREACHED64 = 0xFFFFFFFFFFFFFFFF


def _wcsr(row_ptr, col, w):
    rp, c = _csr(row_ptr, col)
    return rp, c, np.ascontiguousarray(w, dtype=np.uint32)


def minplus(n, row_ptr, col, w, s):
    """(min,+) SOVM with synchronous rounds (oracle.c oracle_minplus; reading Q26).
    Returns (uint64 distances, stats dict)."""
    rp, c, ww = _wcsr(row_ptr, col, w)
    d = np.empty(n, np.uint64)
    st = _Stats()
    rc = _load().oracle_minplus(n, _p(rp), _p(c), _p(ww), int(s), _p(d), ctypes.byref(st))
    if rc:
        raise ValueError(f"oracle_minplus rc={rc}")
    return d, {f: getattr(st, f) for f, _ in _Stats._fields_}


def dijkstra(n, row_ptr, col, w, s):
    rp, c, ww = _wcsr(row_ptr, col, w)
    d = np.empty(n, np.uint64)
    rc = _load().oracle_dijkstra(n, _p(rp), _p(c), _p(ww), int(s), _p(d))
    if rc:
        raise ValueError(f"oracle_dijkstra rc={rc}")
    return d


def floyd_warshall_w(n, row_ptr, col, w):
    rp, c, ww = _wcsr(row_ptr, col, w)
    D = np.empty((n, n), np.uint64)
    rc = _load().oracle_floyd_warshall_w(n, _p(rp), _p(c), _p(ww), _p(D))
    if rc:
        raise ValueError(f"oracle_floyd_warshall_w rc={rc}")
    return D


def certify_w(n, row_ptr, col, w, s, dist):
    """0 if dist (uint64) is the exact weighted distance vector from s (weights >= 1)."""
    rp, c, ww = _wcsr(row_ptr, col, w)
    d = np.ascontiguousarray(dist, dtype=np.uint64)
    bad = ctypes.c_int64(-1)
    rc = _load().oracle_certify_w(n, _p(rp), _p(c), _p(ww), int(s), _p(d), ctypes.byref(bad))
    return rc, bad.value

"""dawn-b200: DAWN (arXiv 2208.04514) unweighted shortest paths on B200 (sm_100a).

Thin ctypes binding over ``libdawn.so`` (C ABI in ``include/dawn.h``).  This module only
marshals arguments: every step of the path (init, push/pull levels, direction choice,
frontier-empty test, records) runs in the CUDA kernels of ``csrc/``.  PyTorch provides device
memory (tensors), the current stream and ``torch.distributed`` for the APSP gather.

There is no CPU fallback: if ``libdawn.so`` is missing or fails to load, importing the
compute entry points raises.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np
import torch

__all__ = ["build", "Graph", "sssp", "sssp_batch", "msssp", "apsp", "apsp_rows", "apsp_shard",
           "wsssp", "wsssp_batch", "dist_u8", "dist_u4", "unpack_u4", "part_range", "part_build", "PartGraph", "part_exchange", "part_sssp", "part_sssp_local",
           "part_fused_local", "part_sssp_fused", "largest_wcc",
           "check", "DawnError", "UNREACHED", "AUTO", "PUSH", "PULL", "MS_BATCH", "REC_DTYPE",
           "records_to_numpy", "stats_to_dict", "gather_records"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_CSRC = os.path.join(_HERE, "csrc")
_LIB = os.path.join(_HERE, "libdawn.so")  # always the in-tree build (no override)
_INCLUDE = os.path.join(os.path.dirname(_HERE), "include")

UNREACHED = 0xFFFFFFFF
MS_BATCH = 256  # DAWN_MS_BATCH: sources per bit-parallel pass / APSP shard unit
AUTO, PUSH, PULL = 0, 1, 2
_VARIANTS = {"auto": AUTO, "push": PUSH, "pull": PULL, AUTO: AUTO, PUSH: PUSH, PULL: PULL}
REC_DTYPE = np.dtype([("source", "<u4"), ("ecc", "<u4"), ("reached", "<u4"), ("pad", "<u4"),
                      ("sum_dist", "<u8"), ("hash", "<u8")])
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3"]

_STATUS = {0: "DAWN_OK", 1: "DAWN_ERR_INVALID_ARGUMENT", 2: "DAWN_ERR_BOUNDS",
           3: "DAWN_ERR_CONFIG", 4: "DAWN_ERR_CAPACITY", 5: "DAWN_ERR_WORKSPACE",
           6: "DAWN_ERR_INVALID_GRAPH", 7: "DAWN_ERR_CUDA"}


class DawnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


def _sources():
    return [os.path.join(_CSRC, f) for f in sorted(os.listdir(_CSRC))
            if f.endswith((".cu", ".cuh", ".h"))] + [os.path.join(_INCLUDE, "dawn.h")]


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile libdawn.so in-tree for sm_100a (nvcc; cross-compiles without a GPU).
    `out`/`defines` build an experimental variant (e.g. defines=("DAWN_PULL_J=4",))."""
    target = out or _LIB
    srcs = _sources()
    newest = max(os.path.getmtime(s) for s in srcs)
    if force or out or not os.path.exists(target) or os.path.getmtime(target) < newest:
        cmd = ["nvcc", *NVCC_FLAGS, *[f"-D{d}" for d in defines],
               os.path.join(_CSRC, "dawn.cu"), "-o", target + ".tmp"]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        os.replace(target + ".tmp", target)
    return target


_lib = None
# dawn_row_sink: int (*)(void *user, int64_t first_row, int64_t rows, const uint32_t *host_rows)
_ROW_SINK = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                             ctypes.c_void_p)


class _SsspStats(ctypes.Structure):
    _fields_ = [("levels", ctypes.c_uint32), ("reached", ctypes.c_uint32),
                ("edges_reach", ctypes.c_uint64), ("edges_examined", ctypes.c_uint64),
                ("push_levels", ctypes.c_uint32), ("pull_levels", ctypes.c_uint32)]


def lib():
    """The loaded libdawn.so (raises if it cannot be loaded: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"libdawn.so not built ({_LIB}); run paper_2208_04514_b200.build()")
        L = ctypes.CDLL(_LIB)
        vp, i64, u32, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint32, ctypes.c_int32
        st = ctypes.c_int
        L.dawn_workspace_bytes.restype = ctypes.c_size_t
        L.dawn_workspace_bytes.argtypes = [i64, i64, u32]
        L.dawn_graph_load_csr.restype = st
        L.dawn_graph_load_csr.argtypes = [i64, i64, vp, vp, vp, vp, u32, vp, ctypes.c_size_t, vp,
                                          ctypes.POINTER(vp)]
        L.dawn_graph_destroy.restype = st
        L.dawn_graph_destroy.argtypes = [vp]
        L.dawn_graph_get_param.restype = st
        L.dawn_graph_get_param.argtypes = [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
        L.dawn_graph_set_param.restype = st
        L.dawn_graph_set_param.argtypes = [vp, ctypes.c_int, ctypes.c_double]
        L.dawn_sssp.restype = st
        L.dawn_sssp.argtypes = [vp, i64, u32, vp, vp, vp]
        L.dawn_sssp_batch.restype = st
        L.dawn_sssp_batch.argtypes = [vp, vp, i64, u32, vp, vp, vp]
        L.dawn_msssp.restype = st
        L.dawn_msssp.argtypes = [vp, vp, i64, vp, vp, vp]
        L.dawn_apsp_shard.restype = st
        L.dawn_apsp_shard.argtypes = [i64, i32, i32, vp, i64, ctypes.POINTER(ctypes.c_int64)]
        L.dawn_apsp.restype = st
        L.dawn_apsp.argtypes = [vp, vp, i64, i32, i32, vp, i64, ctypes.POINTER(ctypes.c_int64), vp]
        L.dawn_last_error.restype = ctypes.c_char_p
        L.dawn_last_error.argtypes = []
        L.dawn_graph_trace.restype = st
        L.dawn_graph_trace.argtypes = [vp, vp, i64, ctypes.POINTER(ctypes.c_int64), vp]
        L.dawn_version.restype = ctypes.c_char_p
        L.dawn_version.argtypes = []
        L.dawn_graph_check.restype = st
        L.dawn_graph_check.argtypes = [vp, vp]
        L.dawn_graph_ms_counters.restype = st
        L.dawn_graph_ms_counters.argtypes = [vp, vp, vp]
        L.dawn_apsp_rows.restype = st
        L.dawn_apsp_rows.argtypes = [vp, vp, i64, i64, vp, vp, _ROW_SINK, vp, vp]
        L.dawn_wsssp_batch.restype = st
        L.dawn_wsssp_batch.argtypes = [vp, vp, i64, vp, vp, vp, vp]
        L.dawn_dist_u8.restype = st
        L.dawn_dist_u8.argtypes = [vp, i64, vp, vp, vp]
        L.dawn_dist_u4.restype = st
        L.dawn_dist_u4.argtypes = [vp, i64, vp, vp, vp]
        L.dawn_wsssp.restype = st
        L.dawn_wsssp.argtypes = [vp, i64, vp, vp, vp, vp]
        L.dawn_part_range.restype = st
        L.dawn_part_range.argtypes = [i64, i32, i32, ctypes.POINTER(ctypes.c_int64),
                                      ctypes.POINTER(ctypes.c_int64)]
        L.dawn_part_build.restype = st
        L.dawn_part_build.argtypes = [i64, i64, vp, vp, i32, i32, ctypes.POINTER(ctypes.c_int64),
                                      vp, vp, vp, vp, vp]
        L.dawn_part_workspace_bytes.restype = ctypes.c_size_t
        L.dawn_part_workspace_bytes.argtypes = [i64, i64, i32, i32]
        L.dawn_part_load.restype = st
        L.dawn_part_load.argtypes = [i64, i64, i32, i32, i64, vp, vp, vp, vp, vp, vp,
                                     ctypes.c_size_t, vp, ctypes.POINTER(vp)]
        L.dawn_part_destroy.restype = st
        L.dawn_part_destroy.argtypes = [vp]
        L.dawn_part_exchange.restype = st
        L.dawn_part_exchange.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp),
                                         ctypes.POINTER(ctypes.c_int64)]
        L.dawn_part_begin.restype = st
        L.dawn_part_begin.argtypes = [vp, i64, u32, vp, vp]
        L.dawn_part_step.restype = st
        L.dawn_part_step.argtypes = [vp, vp]
        L.dawn_part_done.restype = st
        L.dawn_part_done.argtypes = [vp, ctypes.POINTER(ctypes.c_int32), vp]
        L.dawn_part_fused_peers.restype = st
        L.dawn_part_fused_peers.argtypes = [vp, i32, vp, vp]
        L.dawn_part_fused_sssp.restype = st
        L.dawn_part_fused_sssp.argtypes = [vp, i64, u32, vp, vp, i32, vp]
        L.dawn_part_finish.restype = st
        L.dawn_part_finish.argtypes = [vp, vp, vp]
        L.dawn_largest_wcc.restype = st
        L.dawn_largest_wcc.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_int64),
                                       ctypes.POINTER(ctypes.c_uint64), vp]
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise DawnError(status, lib().dawn_last_error().decode())


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "expected a contiguous CUDA tensor"
    return t.data_ptr()


class Graph:
    """A device-resident graph handle (dawn_graph_load_csr).

    row_ptr int64[n+1], col int32[m] (CUDA tensors, or numpy arrays that are uploaded).
    For directed graphs pass the CSC (in_row_ptr, in_col) to enable pull / auto switching.
    The handle keeps references to every tensor it uses (graph arrays + workspace).
    """

    def __init__(self, row_ptr, col, symmetric: bool, in_row_ptr=None, in_col=None,
                 validate: bool = False, device=None, stream=None, trace: bool = False,
                 lean: bool = False):
        dev = torch.device(device) if device is not None else torch.device("cuda",
                                                                            torch.cuda.current_device())
        to = lambda a, dt: (a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
                            ).to(device=dev, dtype=dt).contiguous()
        self.row_ptr = to(row_ptr, torch.int64)
        self.col = to(col, torch.int32)
        self.n = int(self.row_ptr.numel() - 1)
        self.m = int(self.col.numel())
        self.symmetric = bool(symmetric)
        self.in_row_ptr = to(in_row_ptr, torch.int64) if in_row_ptr is not None else None
        self.in_col = to(in_col, torch.int32) if in_col is not None else None
        # lean: DAWN_GRAPH_LEAN (no multi-source words / degree-ordered in-rows / arc array)
        flags = ((1 if symmetric else 0) | (2 if validate else 0) | (4 if trace else 0) |
                 (8 if lean else 0))
        nbytes = lib().dawn_workspace_bytes(self.n, self.m, flags)
        if nbytes == 0:
            raise DawnError(4, "unsupported graph size")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        self.device = dev
        h = ctypes.c_void_p()
        with torch.cuda.device(dev):
            _check(lib().dawn_graph_load_csr(
                self.n, self.m, _dptr(self.row_ptr), _dptr(self.col) if self.m else None,
                _dptr(self.in_row_ptr), _dptr(self.in_col), flags, _dptr(self.workspace),
                nbytes, _stream(stream), ctypes.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def trace(self, stream=None) -> np.ndarray:
        """Per-level trace of the last sssp call (graph built with trace=True)."""
        dt = np.dtype([("t_ns", "<u8"), ("level", "<u4"), ("dir", "<u4"), ("nf", "<u4"),
                       ("rep", "<u4"), ("mf", "<u8"), ("t_first", "<u8"), ("t_last", "<u8"),
                       ("cyc", "<u8", (4,))])
        buf = np.zeros(1 << 16, dt)
        cnt = ctypes.c_int64(0)
        _check(lib().dawn_graph_trace(self._h, buf.ctypes.data_as(ctypes.c_void_p), len(buf),
                                      ctypes.byref(cnt), _stream(stream)))
        self.timeline = buf[-1].copy()  # (t_ns: k_sssp entry, t_first: init done, t_last: end)
        return buf[: min(cnt.value, len(buf) - 1)].copy()

    _PARAMS = {"alpha": 0, "beta": 1, "ms_alpha": 2, "bitmap_push_edges": 3, "solo_edges": 4,
               "cluster_start": 5, "cluster_handover_edges": 6, "bitmap_push_grow_edges": 7,
               "narrow_queue_cap": 8, "batch_lanes": 9, "dense_max_entries": 10, "ms_lanes": 11, "weight_delta": 12,
               "batch_dynamic": 13}

    def get_tuning(self, key: str) -> float:
        """dawn_graph_get_param (e.g. "batch_lanes", "ms_lanes")."""
        v = ctypes.c_double(0)
        _check(lib().dawn_graph_get_param(self._h, self._PARAMS[key], ctypes.byref(v)))
        return v.value

    def set_tuning(self, **kw):
        """dawn_graph_set_param for each keyword (alpha, beta, ms_alpha, bitmap_push_edges,
        solo_edges, cluster_start, cluster_handover_edges, bitmap_push_grow_edges).  Speed only; results never change."""
        for k, v in kw.items():
            _check(lib().dawn_graph_set_param(self._h, self._PARAMS[k], float(v)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.dawn_graph_destroy(h)
            self._h = None


def sssp(g: Graph, source: int, variant="auto", stats: bool = False, out: torch.Tensor | None = None,
         stream=None):
    """dawn_sssp: distances as an int32 CUDA tensor (uint32 bits; UNREACHED reads as -1).

    With stats=True also returns a 32-byte CUDA tensor holding dawn_sssp_stats
    (see stats_to_dict)."""
    dist = out if out is not None else torch.empty(g.n, dtype=torch.int32, device=g.device)
    assert dist.numel() == g.n and dist.dtype == torch.int32
    st = torch.zeros(4, dtype=torch.int64, device=g.device) if stats else None
    _check(lib().dawn_sssp(g.handle, int(source), _VARIANTS[variant], _dptr(dist), _dptr(st),
                           _stream(stream)))
    return (dist, st) if stats else dist


def sssp_batch(g: Graph, sources: torch.Tensor, variant="auto", stats: bool = False,
               out: torch.Tensor | None = None, stream=None, check: bool = False):
    """dawn_sssp_batch: k single-source searches with no host work between them (include/dawn.h:
    concurrent one-CTA searches on tiny graphs, one grid-wide launch running them one after the
    other otherwise).  `sources`: uint32/int32 CUDA tensor [k] of vertex ids in [0, n).
    Returns dist int32 [k, n] (and stats int64 [k, 4] = k dawn_sssp_stats when stats=True)."""
    assert sources.is_cuda and sources.dtype in (torch.int32, torch.uint32)
    k = sources.numel()
    dist = out if out is not None else torch.empty((k, g.n), dtype=torch.int32, device=g.device)
    assert dist.shape == (k, g.n) and dist.dtype == torch.int32 and dist.is_contiguous()
    st = torch.zeros((k, 4), dtype=torch.int64, device=g.device) if stats else None
    _check(lib().dawn_sssp_batch(g.handle, _dptr(sources), k, _VARIANTS[variant], _dptr(dist),
                                 _dptr(st), _stream(stream)))
    if check:  # synchronise and surface a device-side source-id error (DAWN_ERR_BOUNDS)
        globals()["check"](g, stream)
    return (dist, st) if stats else dist


def check(g: Graph, stream=None):
    """dawn_graph_check: synchronise the stream; raise DawnError(DAWN_ERR_BOUNDS) if a
    dawn_sssp_batch since the last check met a source id outside [0, n) (it wrote nothing)."""
    _check(lib().dawn_graph_check(g.handle, _stream(stream)))


def ms_counters(g: Graph, stream=None) -> dict:
    """dawn_graph_ms_counters: executed-schedule counters of the bit-parallel kernel since the
    last read (levels, adjacency entries gathered, word reductions, batches); resets them."""
    out = np.zeros(4, np.uint64)
    _check(lib().dawn_graph_ms_counters(g.handle, out.ctypes.data_as(ctypes.c_void_p),
                                        _stream(stream)))
    return {"levels": int(out[0]), "gathered": int(out[1]), "reductions": int(out[2]),
            "batches": int(out[3])}


def largest_wcc(g: Graph, stream=None):
    """dawn_largest_wcc (device union-find): (vertices of the largest WCC ascending as int64
    numpy array, E_wcc).  PAPER Table 1; ties per DESIGN.md reading Q15."""
    out = np.empty(g.n, np.int64)
    k = ctypes.c_int64(0)
    arcs = ctypes.c_uint64(0)
    _check(lib().dawn_largest_wcc(g.handle, out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(k),
                                  ctypes.byref(arcs), _stream(stream)))
    return out[: k.value].copy(), int(arcs.value)


def stats_to_dict(st: torch.Tensor) -> dict:
    raw = st.cpu().numpy().tobytes()
    s = _SsspStats.from_buffer_copy(raw)
    return {f: getattr(s, f) for f, _ in _SsspStats._fields_}


def records_to_numpy(rec: torch.Tensor) -> np.ndarray:
    return np.frombuffer(rec.cpu().numpy().tobytes(), dtype=REC_DTYPE)


def msssp(g: Graph, sources, dist: bool = True, records: bool = True, stream=None,
          d_out: torch.Tensor | None = None):
    """dawn_msssp (bit-parallel kernel, DAWN_MS_BATCH = 256 sources per pass).  Returns
    (dist int32[k, n] | None, records int64[k, 4] CUDA tensor (32-byte dawn_record rows) | None).
    `d_out`: optional preallocated contiguous int32 [k, n] CUDA tensor for the distances."""
    src = np.ascontiguousarray(np.asarray(sources, dtype=np.int64).reshape(-1))
    k = len(src)
    d = None
    if dist:
        d = d_out if d_out is not None else torch.empty((k, g.n), dtype=torch.int32, device=g.device)
        assert d.shape == (k, g.n) and d.dtype == torch.int32 and d.is_contiguous()
    r = torch.empty((k, 4), dtype=torch.int64, device=g.device) if records else None
    _check(lib().dawn_msssp(g.handle, src.ctypes.data_as(ctypes.c_void_p), k, _dptr(d), _dptr(r),
                            _stream(stream)))
    return d, r


def apsp_rows(g: Graph, sources, sink, chunk: int = MS_BATCH, stream=None):
    """dawn_apsp_rows: the distance rows of every source streamed to host memory.  `sink(first,
    rows)` is called in order with `rows` a uint32 numpy array [r, n] (rows first .. first+r-1),
    valid only during the call (copy what you keep); return False to stop early.  Uses two
    device pieces of chunk x n and two pinned host pieces (allocated here, torch)."""
    src = np.ascontiguousarray(np.asarray(sources, dtype=np.int64).reshape(-1))
    k = len(src)
    c = max(1, min(int(chunk), max(1, k)))
    dev = torch.empty(2 * c * g.n, dtype=torch.int32, device=g.device)
    host = torch.empty(2 * c * g.n, dtype=torch.int32, pin_memory=True)
    base = host.data_ptr()
    hv = host.numpy().view(np.uint32)
    err = []

    def _cb(_user, first, rows, ptr):
        try:
            off = (ptr - base) // 4
            r = sink(int(first), hv[off: off + rows * g.n].reshape(rows, g.n))
            return 1 if r is False else 0
        except BaseException as ex:  # noqa: BLE001 - surfaced after the C call returns
            err.append(ex)
            return 1

    cb = _ROW_SINK(_cb)
    st = lib().dawn_apsp_rows(g.handle, src.ctypes.data_as(ctypes.c_void_p), k, c, _dptr(dev),
                              base, cb, None, _stream(stream))
    if err:
        raise err[0]
    _check(st)


def apsp_shard(k: int, rank: int, world: int) -> np.ndarray:
    """Indices into the source list owned by `rank` (dawn_apsp_shard: MS_BATCH-source batches,
    batch b on rank b mod world)."""
    cnt = ctypes.c_int64(0)
    _check(lib().dawn_apsp_shard(k, rank, world, None, 0, ctypes.byref(cnt)))
    idx = np.empty(cnt.value, np.int64)
    _check(lib().dawn_apsp_shard(k, rank, world, idx.ctypes.data_as(ctypes.c_void_p), len(idx),
                                 ctypes.byref(cnt)))
    return idx


def apsp(g: Graph, sources, rank: int = 0, world: int = 1, group=None, gather: bool = True,
         stream=None):
    """dawn_apsp for this rank's shard, then (world > 1, gather=True) one NCCL all-gather of the
    32-byte records.  Returns int64[k, 4] records in source order (gathered) or this rank's
    shard records (gather=False)."""
    src = np.ascontiguousarray(np.asarray(sources, dtype=np.int64).reshape(-1))
    k = len(src)
    mine = apsp_shard(k, rank, world)
    cap = max(1, len(mine))
    rec = torch.zeros((cap, 4), dtype=torch.int64, device=g.device)
    nw = ctypes.c_int64(0)
    _check(lib().dawn_apsp(g.handle, src.ctypes.data_as(ctypes.c_void_p), k, rank, world,
                           _dptr(rec), cap, ctypes.byref(nw), _stream(stream)))
    if world == 1 or not gather:
        return rec[: nw.value]
    return gather_records(rec[: nw.value], k, world, group)


def gather_records(local: torch.Tensor, k: int, world: int, group=None) -> torch.Tensor:
    """Reassemble per-rank APSP shards (int64[*, 4] record rows) into source order with one
    all-gather (NCCL over NVLink on GPU tensors; gloo on CPU tensors).  The only collective of
    the APSP path."""
    import torch.distributed as dist
    maxcap = len(apsp_shard(k, 0, world))  # rank 0 always owns the largest shard
    buf = torch.zeros((maxcap, 4), dtype=torch.int64, device=local.device)
    buf[: local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    full = torch.empty((k, 4), dtype=torch.int64, device=local.device)
    for r in range(world):
        idx = apsp_shard(k, r, world)
        if len(idx):
            full[torch.from_numpy(idx).to(local.device)] = parts[r][: len(idx)]
    return full


def dist_u8(dist: torch.Tensor, out: torch.Tensor | None = None,
            flags: torch.Tensor | None = None, stream=None):
    """dawn_dist_u8: 1-byte copy of distance rows (255 = unreached, or a distance >= 255 that
    did not fit: then flags[0] bit 0 is set).  Returns (uint8 tensor like dist, int32 flags[1])."""
    assert dist.is_cuda and dist.dtype in (torch.int32, torch.uint32) and dist.is_contiguous()
    out = out if out is not None else torch.empty(dist.shape, dtype=torch.uint8, device=dist.device)
    flags = flags if flags is not None else torch.zeros(1, dtype=torch.int32, device=dist.device)
    _check(lib().dawn_dist_u8(_dptr(dist), dist.numel(), _dptr(out), _dptr(flags), _stream(stream)))
    return out, flags


def dist_u4(dist: torch.Tensor, out: torch.Tensor | None = None,
            flags: torch.Tensor | None = None, stream=None):
    """dawn_dist_u4: 4-bit copy of distance rows, two per byte (15 = unreached, or a distance
    >= 15 that did not fit: then flags[0] bit 0 is set).  Returns (uint8 tensor of
    ceil(numel / 2) bytes, int32 flags[1])."""
    assert dist.is_cuda and dist.dtype in (torch.int32, torch.uint32) and dist.is_contiguous()
    nb = (dist.numel() + 1) // 2
    out = out if out is not None else torch.empty(nb, dtype=torch.uint8, device=dist.device)
    assert out.numel() >= nb and out.dtype == torch.uint8
    flags = flags if flags is not None else torch.zeros(1, dtype=torch.int32, device=dist.device)
    _check(lib().dawn_dist_u4(_dptr(dist), dist.numel(), _dptr(out), _dptr(flags), _stream(stream)))
    return out, flags


def unpack_u4(packed: np.ndarray, count: int) -> np.ndarray:
    """Host-side inverse of dawn_dist_u4 (argument marshalling for the caller): uint32 distances
    with 15 read back as UNREACHED (valid when the call's flag stayed clear)."""
    b = np.asarray(packed, dtype=np.uint8)
    d = np.empty(2 * len(b), dtype=np.uint32)
    d[0::2] = b & 15
    d[1::2] = b >> 4
    d = d[:count]
    d[d == 15] = UNREACHED
    return d


def wsssp(g: Graph, source: int, weights: torch.Tensor, stats: bool = False,
          out: torch.Tensor | None = None, stream=None):
    """dawn_wsssp: weighted SSSP by (min,+) DAWN rounds (NEXT-4).  `weights`: uint32/int32 CUDA
    tensor [m] aligned with the CSR col array.  Returns int32 [n] (uint32 bits, UNREACHED = -1)."""
    assert weights.is_cuda and weights.dtype in (torch.int32, torch.uint32) and weights.numel() == g.m
    dist = out if out is not None else torch.empty(g.n, dtype=torch.int32, device=g.device)
    st = torch.zeros(4, dtype=torch.int64, device=g.device) if stats else None
    _check(lib().dawn_wsssp(g.handle, int(source), _dptr(weights), _dptr(dist), _dptr(st),
                            _stream(stream)))
    return (dist, st) if stats else dist


def wsssp_batch(g: Graph, sources: torch.Tensor, weights: torch.Tensor, stats: bool = False,
                out: torch.Tensor | None = None, stream=None, check: bool = False):
    """dawn_wsssp_batch: k weighted searches from a device source list on the batch lanes.
    Returns int32 [k, n] (and int64 [k, 4] statistics)."""
    assert sources.is_cuda and sources.dtype in (torch.int32, torch.uint32)
    assert weights.is_cuda and weights.dtype in (torch.int32, torch.uint32) and weights.numel() == g.m
    k = sources.numel()
    dist = out if out is not None else torch.empty((k, g.n), dtype=torch.int32, device=g.device)
    assert dist.shape == (k, g.n) and dist.dtype == torch.int32 and dist.is_contiguous()
    st = torch.zeros((k, 4), dtype=torch.int64, device=g.device) if stats else None
    _check(lib().dawn_wsssp_batch(g.handle, _dptr(sources), k, _dptr(weights), _dptr(dist),
                                  _dptr(st), _stream(stream)))
    if check:
        globals()["check"](g, stream)
    return (dist, st) if stats else dist


# ----------------------------------------------------------- partitioned SSSP (NEXT-3)
def part_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """dawn_part_range: the vertex ids [lo, hi) rank `rank` owns (host only)."""
    lo, hi = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(lib().dawn_part_range(n, world, rank, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def part_build(row_ptr, col, world: int, rank: int) -> dict:
    """dawn_part_build (host C++): rank's out-slice (out_rp, out_col: targets local), in-rows
    (in_rp, in_col: sources global) and own out-degrees, from the global host CSR."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cl = np.ascontiguousarray(col, dtype=np.int32)
    n, m = len(rp) - 1, len(cl)
    lo, hi = part_range(n, world, rank)
    mr = ctypes.c_int64(0)
    P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    _check(lib().dawn_part_build(n, m, P(rp), P(cl), world, rank, ctypes.byref(mr),
                                 None, None, None, None, None))
    out = {"n": n, "m": m, "lo": lo, "hi": hi, "m_r": mr.value,
           "out_rp": np.empty(n + 1, np.int64), "out_col": np.empty(max(1, mr.value), np.int32),
           "in_rp": np.empty(hi - lo + 1, np.int64), "in_col": np.empty(max(1, mr.value), np.int32),
           "deg": np.empty(max(1, hi - lo), np.uint32)}
    _check(lib().dawn_part_build(n, m, P(rp), P(cl), world, rank, ctypes.byref(mr),
                                 P(out["out_rp"]), P(out["out_col"]), P(out["in_rp"]),
                                 P(out["in_col"]), P(out["deg"])))
    out["out_col"] = out["out_col"][: mr.value]
    out["in_col"] = out["in_col"][: mr.value]
    out["deg"] = out["deg"][: hi - lo]
    return out


class PartGraph:
    """One rank's share of a vertex-partitioned graph on its device (dawn_part_load)."""

    def __init__(self, part: dict, world: int, rank: int, device=None, stream=None):
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dt)
        self.n, self.m, self.world, self.rank = part["n"], part["m"], world, rank
        self.lo, self.hi, self.m_r = part["lo"], part["hi"], part["m_r"]
        self.R = self.hi - self.lo
        self.out_rp = t(part["out_rp"], torch.int64)
        self.out_col = t(part["out_col"] if self.m_r else np.zeros(1, np.int32), torch.int32)
        self.in_rp = t(part["in_rp"], torch.int64)
        self.in_col = t(part["in_col"] if self.m_r else np.zeros(1, np.int32), torch.int32)
        self.deg = t(part["deg"].view(np.int32) if self.R else np.zeros(1, np.int32), torch.int32)
        nb = lib().dawn_part_workspace_bytes(self.n, self.m_r, world, rank)
        if nb == 0:
            raise DawnError(4, "unsupported partition size")
        self.workspace = torch.empty(nb, dtype=torch.uint8, device=dev)
        self.device = dev
        h = ctypes.c_void_p()
        with torch.cuda.device(dev):
            _check(lib().dawn_part_load(self.n, self.m, world, rank, self.m_r, _dptr(self.out_rp),
                                        _dptr(self.out_col), _dptr(self.in_rp), _dptr(self.in_col),
                                        _dptr(self.deg), _dptr(self.workspace), nb, _stream(stream),
                                        ctypes.byref(h)))
        self._h = h
        sp, rp, sw = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64(0)
        _check(lib().dawn_part_exchange(h, ctypes.byref(sp), ctypes.byref(rp), ctypes.byref(sw)))
        self.slice_words = sw.value
        off_s = sp.value - self.workspace.data_ptr()
        off_r = rp.value - self.workspace.data_ptr()
        # views of the workspace's exchange buffers (what the all-gather moves)
        self.send = self.workspace[off_s: off_s + 4 * sw.value].view(torch.int32)
        self.recv = self.workspace[off_r: off_r + 4 * sw.value * world].view(torch.int32)

    @property
    def handle(self):
        return self._h

    def xbuffer(self) -> torch.Tensor:
        """This rank's exchange buffer of the fused path (int32: two receive slots of
        world x slice_words words, then the 64-bit arrival counter), zero-initialised once."""
        if getattr(self, "_xbuf", None) is None:
            self._xbuf = torch.zeros(2 * self.world * self.slice_words + 2, dtype=torch.int32,
                                     device=self.device)
        return self._xbuf

    def set_peers(self, bufs: list):
        """dawn_part_fused_peers from every rank's exchange buffer (as mapped in this process)."""
        assert len(bufs) == self.world
        recv = (ctypes.c_void_p * self.world)(*[b.data_ptr() for b in bufs])
        flag = (ctypes.c_void_p * self.world)(
            *[b.data_ptr() + 4 * 2 * self.world * self.slice_words for b in bufs])
        _check(lib().dawn_part_fused_peers(self._h, self.world, recv, flag))
        self._peers = bufs  # keep the mappings alive

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.dawn_part_destroy(h)
            self._h = None


def part_fused_local(parts: list, source: int, variant="auto", stats: bool = False):
    """The fused exchange with all W ranks on ONE device (each rank's persistent kernel on its
    own stream and 1/W of the SMs; the slices go through device memory instead of NVLink): the
    same kernel and protocol as part_sssp_fused across processes.  Returns the global distance
    vector (int32 [n]) (and the per-rank statistics)."""
    W = len(parts)
    key = tuple(id(p) for p in parts)
    if getattr(parts[0], "_local_peers", None) != key:
        bufs = [p.xbuffer() for p in parts]
        for p in parts:
            p.set_peers(bufs)
            p._local_peers = key
    outs = [torch.empty(max(1, p.R), dtype=torch.int32, device=p.device) for p in parts]
    sts = [torch.zeros(4, dtype=torch.int64, device=p.device) for p in parts] if stats else None
    nsm = torch.cuda.get_device_properties(parts[0].device).multi_processor_count
    grid = max(1, 2 * nsm // W)
    cur = torch.cuda.current_stream()
    streams = [torch.cuda.Stream(device=parts[0].device) for _ in parts]
    for i, p in enumerate(parts):
        streams[i].wait_stream(cur)
        _check(lib().dawn_part_fused_sssp(p.handle, int(source), _VARIANTS[variant], _dptr(outs[i]),
                                          _dptr(sts[i]) if stats else None, grid,
                                          streams[i].cuda_stream))
    for st_ in streams:
        cur.wait_stream(st_)
    d = torch.cat([o[: p.R] for o, p in zip(outs, parts)])
    return (d, sts) if stats else d


def part_sssp_fused(pg: PartGraph, source: int, variant="auto", group=None, out=None,
                    stats: bool = False, stream=None):
    """Partitioned SSSP with the fused exchange across processes (one GPU per rank): the first
    call maps every rank's exchange buffer into this process (CUDA IPC through
    torch.multiprocessing's tensor sharing, handles exchanged with one all_gather_object), then
    each search is ONE persistent kernel per rank.  Every rank calls it with the same
    arguments; returns this rank's distance slice."""
    if getattr(pg, "_peers", None) is None:
        if pg.world == 1:
            pg.set_peers([pg.xbuffer()])
        else:
            import torch.distributed as dist
            from torch.multiprocessing.reductions import reduce_tensor
            mine = pg.xbuffer()
            objs = [None] * pg.world
            dist.all_gather_object(objs, reduce_tensor(mine), group=group)
            bufs = [mine if q == pg.rank else fn(*args) for q, (fn, args) in enumerate(objs)]
            pg.set_peers(bufs)
            dist.barrier(group=group)
    dist_t = out if out is not None else torch.empty(max(1, pg.R), dtype=torch.int32, device=pg.device)
    st = torch.zeros(4, dtype=torch.int64, device=pg.device) if stats else None
    _check(lib().dawn_part_fused_sssp(pg.handle, int(source), _VARIANTS[variant], _dptr(dist_t),
                                      _dptr(st), 0, _stream(stream)))
    d = dist_t[: pg.R]
    return (d, st) if stats else d


def part_exchange(pg: PartGraph, group=None):
    """recv <- concatenation over ranks of send: one all-gather (NCCL over NVLink for CUDA
    tensors; gloo for CPU tensors in the host tests); a device copy at world 1."""
    import torch.distributed as dist
    if pg.world == 1 and not (dist.is_available() and dist.is_initialized()):
        pg.recv.copy_(pg.send)
        return
    if pg.send.is_cuda:
        dist.all_gather_into_tensor(pg.recv, pg.send, group=group)
    else:
        parts = list(pg.recv.view(pg.world, -1).unbind(0))
        dist.all_gather(parts, pg.send, group=group)


def part_sssp(pg: PartGraph, source: int, variant="auto", group=None, out=None,
              stats: bool = False, check_every: int = 4, exchange=None, stream=None):
    """Partitioned SSSP on this rank (every rank calls it with the same arguments): returns the
    distances of the owned vertices [lo, hi) as int32 [hi - lo] (and the statistics)."""
    dist_t = out if out is not None else torch.empty(max(1, pg.R), dtype=torch.int32, device=pg.device)
    st = torch.zeros(4, dtype=torch.int64, device=pg.device) if stats else None
    s = _stream(stream)
    ex = exchange or (lambda: part_exchange(pg, group))
    _check(lib().dawn_part_begin(pg.handle, int(source), _VARIANTS[variant], _dptr(dist_t), s))
    steps = 0
    done = ctypes.c_int32(0)
    while True:
        ex()
        _check(lib().dawn_part_step(pg.handle, s))
        steps += 1
        if steps % check_every == 0:
            _check(lib().dawn_part_done(pg.handle, ctypes.byref(done), s))
            if done.value:
                break
    _check(lib().dawn_part_finish(pg.handle, _dptr(st), s))
    d = dist_t[: pg.R]
    return (d, st) if stats else d


def part_sssp_local(parts: list, source: int, variant="auto", stats: bool = False,
                    check_every: int = 4):
    """All W ranks' partitions on ONE device, the all-gather done by device copies: the same
    kernels and exchange layout as part_sssp under torch.distributed (used by the tests to
    check W > 1 on a single GPU).  Returns the global distance vector (int32 [n])."""
    W = len(parts)
    outs = [torch.empty(max(1, p.R), dtype=torch.int32, device=p.device) for p in parts]
    sts = [torch.zeros(4, dtype=torch.int64, device=p.device) for p in parts] if stats else None
    s = _stream(None)
    for i, p in enumerate(parts):
        _check(lib().dawn_part_begin(p.handle, int(source), _VARIANTS[variant], _dptr(outs[i]), s))
    steps = 0
    done = ctypes.c_int32(0)
    while True:
        full = torch.cat([p.send for p in parts])
        for p in parts:
            p.recv.copy_(full)
        for p in parts:
            _check(lib().dawn_part_step(p.handle, s))
        steps += 1
        if steps % check_every == 0:
            _check(lib().dawn_part_done(parts[0].handle, ctypes.byref(done), s))
            if done.value:
                break
    for i, p in enumerate(parts):
        _check(lib().dawn_part_finish(p.handle, _dptr(sts[i]) if stats else None, s))
    d = torch.cat([o[: p.R] for o, p in zip(outs, parts)])
    return (d, sts) if stats else d


def version() -> str:
    return lib().dawn_version().decode()

// dawn.cu — libdawn.so: the C ABI of include/dawn.h over the sm_100a kernels.
// Host side validates, lays out the caller's workspace and enqueues a fixed number of persistent
// kernels per call (one; k_narrow + k_sssp on cluster-start graphs), never per-level host work.
// No torch types cross this boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/dawn.h"
#include "layout.h"
#include "ms64_kernel.cuh"
#include "small_kernel.cuh"
#include "narrow_kernel.cuh"
#include "sssp_kernel.cuh"
#include "wcc_kernel.cuh"
#include "part_kernel.cuh"
#include "wsssp_kernel.cuh"

using namespace dawn;

namespace {

// Thread-local message buffer: formatting never allocates, so no exception can start here.
thread_local char g_err[512];

dawn_status fail(dawn_status s, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}
dawn_status cuda_fail(cudaError_t e, const char *where) {
  return fail(DAWN_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}
void clear_err() { g_err[0] = 0; }

constexpr int kNT = 512;  // threads per CTA of the persistent kernels
#ifndef DAWN_BATCH_CLAIM
#define DAWN_BATCH_CLAIM 2  // dynamic batch lanes: 2 = on for the 64-register kernel (n > 2^22)
#endif
// Graph-size thresholds of the kernel choice (measured on B200)
#ifndef DAWN_BATCH_TWO
#define DAWN_BATCH_TWO 1  // batch lanes use the 2-CTA/SM k_sssp on every graph
#endif
#ifndef DAWN_SSSP_ONE_MAX
#define DAWN_SSSP_ONE_MAX (1 << 22)
#endif
constexpr int64_t kSsspOneMaxN = DAWN_SSSP_ONE_MAX;  // k_sssp<kNT, 1> (1 CTA/SM, 128 regs) up to 2^22
constexpr int64_t kOneCtaMaxNM = 1 << 15;  // n + m this small: one CTA, barriers are __syncthreads
constexpr int kMsBlocksPerSm = 2;          // k_ms64 CTAs per SM (if they fit)
constexpr uint32_t kNarrowQcapMax = 1u << 20;
// dawn_sssp_batch lanes (concurrent searches) by default: measured on B200
constexpr int kDefaultMsLanes = DAWN_MS_LANES;  // multi-source lanes (B200 measurement)
#ifndef DAWN_WDELTA
#define DAWN_WDELTA 8  // near/far step of dawn_wsssp (weights 1..255 on Kronecker-24)
#endif
#ifndef DAWN_LANES_SMALL
#define DAWN_LANES_SMALL 16  // default batch lanes for n <= 2^22 (C2, 2-CTA/SM kernel: 8 -> 1,365, 12 -> 1,443, 16 -> 1,538, 24 -> 1,460, 32 -> 1,502 GTEPS)
#endif
#ifndef DAWN_LANES_BIG
#define DAWN_LANES_BIG 4    // ... and above (C4: 1 -> 1343, 2 -> 1590, 4 -> 1678 GTEPS)
#endif
int kDefaultLanes(int64_t n) { return n <= (int64_t(1) << 22) ? DAWN_LANES_SMALL : DAWN_LANES_BIG; }

// ---------------------------------------------------------------- graph residency kernels
__global__ void k_offsets32(const int64_t *__restrict__ in, uint32_t *__restrict__ out, int64_t n1) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n1;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)in[i];
}

// noin bit v = (in-degree(v) == 0); counts vertices with in-degree > 0.
__global__ void k_noin(const uint32_t *__restrict__ irp, uint32_t n, uint32_t nwords,
                       uint32_t *__restrict__ noin, uint32_t *n_hasin) {
  uint32_t local = 0;
  for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
       w += gridDim.x * blockDim.x) {
    uint32_t bits = 0;
    for (uint32_t b = 0; b < 32; ++b) {
      const uint32_t v = w * 32 + b;
      if (v < n && irp[v + 1] == irp[v]) bits |= 1u << b;
      if (v < n && irp[v + 1] != irp[v]) local++;
    }
    noin[w] = bits;
  }
  local = warp_sum(local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(n_hasin, local);
}

// CSR invariants: row_ptr[0] = 0, monotone, row_ptr[n] = m, cols in [0, n).
__global__ void k_validate(const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                           int64_t n, int64_t m, uint32_t *err) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t0 == 0 && (rp[0] != 0 || rp[n] != m)) atomicOr(err, 1u);
  for (int64_t i = t0; i < n; i += stride)
    if (rp[i + 1] < rp[i]) atomicOr(err, 2u);
  for (int64_t j = t0; j < m; j += stride)
    if (col[j] < 0 || col[j] >= n) atomicOr(err, 4u);
}

// ---- static heavy-row pieces (rows with degree > kHeavy, cut into kHPiece-edge pieces)
__device__ __forceinline__ uint32_t hpieces(const uint32_t *rp, uint32_t v) {
  const uint32_t d = rp[v + 1] - rp[v];
  return d > kHeavy ? (d + kHPiece - 1) / kHPiece : 0u;
}

// pass 1: per 2048-vertex block, the piece count (-> tmp[block]) and the heavy bitmap words
__global__ void k_hcount(const uint32_t *__restrict__ rp, uint32_t n, uint32_t *__restrict__ bits,
                         uint32_t *__restrict__ tmp) {
  __shared__ uint32_t sm[32];
  const uint32_t base = blockIdx.x * kScanBlock;
  uint32_t local = 0;
  for (uint32_t w = threadIdx.x; w < kScanBlock / 32; w += blockDim.x) {
    uint32_t b = 0;
    for (uint32_t i = 0; i < 32; ++i) {
      const uint32_t v = base + w * 32 + i;
      if (v < n) {
        const uint32_t c = hpieces(rp, v);
        if (c) b |= 1u << i;
        local += c;
      }
    }
    if (base / 32 + w < (n + 31) / 32) bits[base / 32 + w] = b;
  }
  local = warp_sum(local);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x / 32] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (uint32_t i = 0; i < blockDim.x / 32; ++i) t += sm[i];
    tmp[blockIdx.x] = t;
  }
}

// pass 2: one CTA: exclusive scan of the block counts; total -> *total
__global__ void k_hscan(uint32_t *tmp, uint32_t nblk, uint32_t *total) {
  if (threadIdx.x == 0) {
    uint32_t run = 0;
    for (uint32_t i = 0; i < nblk; ++i) {
      const uint32_t c = tmp[i];
      tmp[i] = run;
      run += c;
    }
    *total = run;
  }
}

// ---- static ascending list of vertices with an in-edge (the first pull level's unreached list)
__global__ void k_lcount(const uint32_t *__restrict__ irp, uint32_t n, uint32_t *__restrict__ tmp) {
  __shared__ uint32_t sm[32];
  const uint32_t base = blockIdx.x * kScanBlock;
  uint32_t c = 0;
  for (uint32_t i = threadIdx.x; i < kScanBlock; i += blockDim.x) {
    const uint32_t v = base + i;
    if (v < n && irp[v + 1] > irp[v]) ++c;
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x / 32] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (uint32_t i = 0; i < blockDim.x / 32; ++i) t += sm[i];
    tmp[blockIdx.x] = t;
  }
}

__global__ void k_lfill(const uint32_t *__restrict__ irp, uint32_t n, const uint32_t *__restrict__ tmp,
                        uint32_t *__restrict__ out) {
  __shared__ uint32_t sm[256];
  constexpr uint32_t kPer = kScanBlock / 256;  // blockDim.x == 256
  const uint32_t v0 = blockIdx.x * kScanBlock + threadIdx.x * kPer;
  uint32_t c = 0;
  for (uint32_t i = 0; i < kPer; ++i)
    if (v0 + i < n && irp[v0 + i + 1] > irp[v0 + i]) ++c;
  sm[threadIdx.x] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = tmp[blockIdx.x];
    for (uint32_t i = 0; i < blockDim.x; ++i) {
      const uint32_t x = sm[i];
      sm[i] = run;
      run += x;
    }
  }
  __syncthreads();
  uint32_t o = sm[threadIdx.x];
  for (uint32_t i = 0; i < kPer; ++i) {
    const uint32_t v = v0 + i;
    if (v < n && irp[v + 1] > irp[v]) out[o++] = v;
  }
}

// ---- pull-friendly in-rows: copy each CSC row and move its kTopK in-neighbours of largest
// out-degree to the front, in descending order (ties: earlier position).  Distances do not
// depend on adjacency order; a pull probe meets a hub of the frontier first.  Warp per row.
__global__ void k_topk_rows(const uint32_t *__restrict__ irp, const int32_t *__restrict__ icol,
                            const uint32_t *__restrict__ rp, uint32_t n, int32_t *__restrict__ out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t u = gw; u < n; u += nw) {
    const uint32_t s = irp[u], e = irp[u + 1];
    for (uint32_t j = s + lane; j < e; j += 32) out[j] = icol[j];
    __syncwarp();
    if (e - s < 2) continue;
    const uint32_t K = min(kTopK, e - s - 1);
    for (uint32_t i = 0; i < K; ++i) {
      uint32_t bd = 0, bp = 0xffffffffu;
      for (uint32_t j = s + i + lane; j < e; j += 32) {
        const uint32_t v = (uint32_t)out[j];
        const uint32_t d = rp[v + 1] - rp[v];
        if (bp == 0xffffffffu || d > bd) { bd = d; bp = j; }
      }
      for (int o = 16; o; o >>= 1) {
        const uint32_t od = __shfl_xor_sync(DAWN_FULL, bd, o), op = __shfl_xor_sync(DAWN_FULL, bp, o);
        if (op != 0xffffffffu && (bp == 0xffffffffu || od > bd || (od == bd && op < bp))) {
          bd = od;
          bp = op;
        }
      }
      if (lane == 0 && bp != s + i) {
        const int32_t t = out[s + i];
        out[s + i] = out[bp];
        out[bp] = t;
      }
      __syncwarp();
    }
  }
}

// top1[u] = the first in-neighbour of u's degree-ordered in-row (0xffffffff: none)
__global__ void k_top1(const uint32_t *__restrict__ irp, const int32_t *__restrict__ icol2,
                       uint32_t n, uint32_t *__restrict__ top1) {
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < n; u += gridDim.x * blockDim.x)
    top1[u] = irp[u + 1] > irp[u] ? (uint32_t)icol2[irp[u]] : 0xffffffffu;
}

// pass 3 (piece-major order): hc[c] = #heavy rows with exactly c pieces; maxc
__global__ void k_hhist(const uint32_t *__restrict__ rp, uint32_t n, uint32_t *hc, uint32_t *maxc) {
  uint32_t mx = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint32_t c = hpieces(rp, v);
    if (c) {
      atomicAdd(hc + c, 1u);
      mx = max(mx, c);
    }
  }
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(DAWN_FULL, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(maxc, mx);
}

// pass 4 (one thread): base[k] = #pieces with piece index < k  (rows with > k pieces: suffix
// sums of hc); cursor[k] = 0
__global__ void k_hbase(uint32_t *hc, uint32_t *base, uint32_t *cursor, const uint32_t *maxc) {
  if (threadIdx.x != 0) return;
  const uint32_t mx = *maxc;
  uint32_t rows = 0;  // rows with > k pieces, built from the top
  for (uint32_t c = mx; c >= 1; --c) {
    rows += hc[c];
    hc[c] = rows;      // now hc[c] = #rows with >= c pieces = #pieces of index c-1
  }
  uint32_t run = 0;
  for (uint32_t k = 0; k < mx; ++k) {
    base[k] = run;
    cursor[k] = 0;
    run += hc[k + 1];
  }
}

// pass 5: write every piece at base[k] + (arrival order within index k): all first pieces,
// then all second pieces, ...  A later piece of a row usually finds the row already settled
// by an earlier one (pull early exit survives the split).
__global__ void k_hfill(const uint32_t *__restrict__ rp, uint32_t n, const uint32_t *__restrict__ base,
                        uint32_t *cursor, uint32_t *__restrict__ hv, uint32_t *__restrict__ hs,
                        uint32_t *__restrict__ he) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint32_t s = rp[v], e = rp[v + 1];
    if (e - s <= kHeavy) continue;
    uint32_t k = 0;
    for (uint32_t a = s; a < e; a += kHPiece, ++k) {
      const uint32_t o = base[k] + atomicAdd(cursor + k, 1u);
      hv[o] = v;
      hs[o] = a;
      he[o] = min(e, a + kHPiece);
    }
  }
}

// ---- id locality of the graph: arcs (v, u) whose visited words have the same owner CTA in
// k_narrow (word mod 16), over the rows of the first 2^20 vertices (untimed, at load)
__global__ void k_locality(const uint32_t *__restrict__ rp, const int32_t *__restrict__ col,
                           uint32_t nv, unsigned long long *cnt) {
  unsigned long long same = 0, tot = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += gridDim.x * blockDim.x) {
    const uint32_t s = rp[v], e = min(rp[v + 1], rp[v] + 64u);
    for (uint32_t j = s; j < e; ++j) {
      same += (((uint32_t)col[j] >> 5) % kNarrowCluster) == ((v >> 5) % kNarrowCluster);
      ++tot;
    }
  }
  same = warp_sum(same);
  tot = warp_sum(tot);
  if ((threadIdx.x & 31) == 0 && tot) {
    atomicAdd(cnt, same);
    atomicAdd(cnt + 1, tot);
  }
}

// ---- k_narrow's augmented arcs: arc[j] = (col[j], row_ptr[col[j]], row_ptr[col[j] + 1], 0)
__global__ void k_arcs(const int32_t *__restrict__ col, const uint32_t *__restrict__ rp, int64_t m,
                       uint4 *__restrict__ arc) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m;
       j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = (uint32_t)col[j];
    arc[j] = make_uint4(v, rp[v], rp[v + 1], 0u);
  }
}

}  // namespace

struct dawn_graph_s {
  int64_t n, m;
  uint32_t flags;
  int device;
  int nsm;
  char *ws;
  Layout L;
  const int32_t *col, *icol;
  bool has_csc;
  float alpha = 2.f, beta = 96.f, ms_alpha = 2.f;
  int sssp_grid, ms_grid, wsssp_grid = 1;
  int sssp_grid2 = 1;     // grid of the 2-CTA/SM instantiation (batch lanes use it on any graph)
  bool sssp_one = false;  // the 1-CTA-per-SM instantiation of k_sssp (small graphs)
  bool trace;
  size_t small_cap;  // max dynamic smem for k_small (0 = disabled)
  uint32_t bmpush_e = 1u << 18, solo_e = 512, bmpush_grow = 4096;
  uint32_t n_hasin = 0;
  bool cluster_start = false;     // DAWN_PARAM_CLUSTER_START (default set at load)
  unsigned long long handover_m = 0;  // DAWN_PARAM_CLUSTER_HANDOVER_EDGES (set at load)
  bool batch_claim = false;            // DAWN_PARAM_BATCH_DYNAMIC (default set at load)
  bool narrow_owner = false;     // owner-computes queues (ids local: most arcs stay in a CTA)
  bool narrow_ok = false;        // the visited bitmap fits 16 CTAs and the cluster launches
  uint32_t narrow_wpc = 0, narrow_qcap = 0, narrow_grid = 0;
  uint32_t narrow_qcap_max = 0;  // load-time capacity (DAWN_PARAM_NARROW_QUEUE_CAP lowers qcap)
  size_t narrow_smem = 0;
  uint32_t seq = 0;
  bool lean = false;             // DAWN_GRAPH_LEAN: no ms64 words / icol2 / augmented arcs
  int lanes = 1;                 // DAWN_PARAM_BATCH_LANES (<= L.nlanes)
  int ms_lanes = 1;               // DAWN_PARAM_MS_LANES (<= L.ms_nlanes)
  uint32_t wdelta = DAWN_WDELTA;   // DAWN_PARAM_WEIGHT_DELTA (0: near/far off)
  double dense_max = 1099511627776.0;  // DAWN_PARAM_DENSE_MAX_ENTRIES (k*n of a dense output)
  // lane streams / fork-join events of dawn_sssp_batch (created at load, host resources only)
  cudaStream_t lane_st[kMaxLanes] = {};
  cudaEvent_t ev_fork = nullptr, ev_join[kMaxLanes] = {};
  ~dawn_graph_s() {
    for (int l = 0; l < kMaxLanes; ++l) {
      if (lane_st[l]) cudaStreamDestroy(lane_st[l]);
      if (ev_join[l]) cudaEventDestroy(ev_join[l]);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
  }
};

namespace {

template <class T>
T *at(dawn_graph g, size_t off) {
  return reinterpret_cast<T *>(g->ws + off);
}

int grid_for(const void *fn, int nsm) {
  int bps = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, kNT, 0);
  bps = std::max(1, std::min(bps, 2));
  return std::min<int>(nsm * bps, (int)kMaxBlocks);
}

dawn_status set_device(dawn_graph g) {
  cudaError_t e = cudaSetDevice(g->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  return DAWN_OK;
}

}  // namespace

// Every exported function runs its body inside this guard: a host allocation failure (the
// only exception the bodies can raise: std::vector) becomes DAWN_ERR_CAPACITY instead of
// crossing the C ABI.
#define DAWN_GUARD(body)                                                       \
  try {                                                                        \
    clear_err();                                                               \
    body                                                                       \
  } catch (...) {                                                              \
    return fail(DAWN_ERR_CAPACITY, "host allocation failed");                  \
  }

namespace {

dawn_status load_csr(int64_t n, int64_t m, const int64_t *row_ptr, const int32_t *col,
                     const int64_t *in_row_ptr, const int32_t *in_col, uint32_t flags,
                     void *workspace, size_t ws_bytes, void *stream, dawn_graph *out) {
  if (!out) return fail(DAWN_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (n < 1 || m < 0) return fail(DAWN_ERR_INVALID_ARGUMENT, "n must be >= 1 and m >= 0");
  if (n >= (int64_t(1) << 31) || m >= (int64_t(1) << 32))
    return fail(DAWN_ERR_CAPACITY, "n must be < 2^31 and m < 2^32 (32-bit offsets)");
  if (flags & ~uint32_t(DAWN_GRAPH_SYMMETRIC | DAWN_GRAPH_VALIDATE | DAWN_GRAPH_TRACE |
                        DAWN_GRAPH_LEAN))
    return fail(DAWN_ERR_INVALID_ARGUMENT, "unknown graph flag");
  if (!row_ptr || (!col && m > 0) || !workspace)
    return fail(DAWN_ERR_INVALID_ARGUMENT, "row_ptr/col/workspace is NULL");
  const bool sym = flags & DAWN_GRAPH_SYMMETRIC;
  const bool has_csc = sym || (in_row_ptr && (in_col || m == 0));
  if (!sym && ((in_row_ptr == nullptr) != (in_col == nullptr) && m > 0))
    return fail(DAWN_ERR_INVALID_ARGUMENT, "in_row_ptr and in_col must both be given or NULL");
  if (reinterpret_cast<uintptr_t>(workspace) & 255)
    return fail(DAWN_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  Layout L = make_layout(n, m, flags);
  if (ws_bytes < L.total)
    return fail(DAWN_ERR_WORKSPACE, "workspace too small: need %zu bytes, got %zu", L.total,
                ws_bytes);
  cudaPointerAttributes pa{};
  cudaError_t e = cudaPointerGetAttributes(&pa, workspace);
  if (e != cudaSuccess) return cuda_fail(e, "cudaPointerGetAttributes(workspace)");
  if (pa.type != cudaMemoryTypeDevice)
    return fail(DAWN_ERR_INVALID_ARGUMENT, "workspace is not device memory");
  auto *g = new (std::nothrow) dawn_graph_s;
  if (!g) return fail(DAWN_ERR_CAPACITY, "host allocation failed");
  g->n = n;
  g->m = m;
  g->flags = flags;
  g->device = pa.device;
  g->ws = static_cast<char *>(workspace);
  g->L = L;
  g->col = col;
  g->has_csc = has_csc;
  g->icol = sym ? col : in_col;
  g->trace = flags & DAWN_GRAPH_TRACE;
  g->lean = flags & DAWN_GRAPH_LEAN;
  if ((e = cudaSetDevice(g->device)) != cudaSuccess) { delete g; return cuda_fail(e, "cudaSetDevice"); }
  cudaDeviceGetAttribute(&g->nsm, cudaDevAttrMultiProcessorCount, g->device);
  // small graphs: k_sssp<kNT, 1> (one CTA per SM, 128 registers); big ones k_sssp<kNT, 2>
  g->sssp_one = n <= kSsspOneMaxN;
  // dynamic batch lanes: Kronecker-24 1,690 -> 1,718 GTEPS, Kronecker-20 1,463 -> 1,531
  g->batch_claim = DAWN_BATCH_CLAIM == 1 || (DAWN_BATCH_CLAIM == 2 && (!g->sssp_one || DAWN_BATCH_TWO));
  g->sssp_grid2 = grid_for((const void *)k_sssp<kNT, 2>, g->nsm);
  g->sssp_grid = g->sssp_one ? std::min<int>(g->nsm, (int)kMaxBlocks) : g->sssp_grid2;
  {
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, g->device);
    const size_t cap = (size_t)std::max(0, optin - 1024);
    g->small_cap = 0;
    if (cudaFuncSetAttribute((const void *)k_small<1024>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap) == cudaSuccess)
      g->small_cap = cap;
    cudaGetLastError();
    // k_narrow: visited slice of ceil(nwords / 16) words (multiple of 4) per CTA, the rest of
    // the shared memory holds the two frontier queues
    g->narrow_ok = false;
    if ((uint64_t)n <= kNarrowMaxN && m > 0) {
      const uint32_t nw = (uint32_t)((n + 31) / 32);
      const uint32_t wpc = ((nw + kNarrowCluster - 1) / kNarrowCluster + 3) & ~3u;
      const size_t fixed = narrow_smem_bytes(wpc, 0);
      uint32_t qcap = fixed < cap ? (uint32_t)((cap - fixed) / kNarrowEntryBytes) : 0u;
      qcap = std::min<uint32_t>(qcap, kNarrowQcapMax);
      const size_t bytes = narrow_smem_bytes(wpc, qcap);
      if (qcap >= 32 && bytes <= cap &&
          cudaFuncSetAttribute((const void *)k_narrow, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)bytes) == cudaSuccess &&
          cudaFuncSetAttribute((const void *)k_narrow,
                               cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = kNarrowCluster;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(kNarrowCluster * 16);
        cfg.blockDim = dim3(kNarrowThreads);
        cfg.dynamicSmemBytes = bytes;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, (const void *)k_narrow, &cfg) == cudaSuccess &&
            ncl >= 1) {
          g->narrow_ok = true;
          g->narrow_wpc = wpc;
          g->narrow_qcap = g->narrow_qcap_max = qcap;
          g->narrow_smem = bytes;
          g->narrow_grid = kNarrowCluster * (uint32_t)std::min(ncl, std::max(1, g->nsm / (int)kNarrowCluster));
        }
      }
    }
    cudaGetLastError();
  }
  g->wsssp_grid = grid_for((const void *)k_wsssp<kNT>, g->nsm);
  if (!g->lean) {
    cudaFuncSetAttribute((const void *)k_ms64<kMsNT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)ms_smem_bytes(kMsNT));
    int bps = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, (const void *)k_ms64<kMsNT>, kMsNT,
                                                  ms_smem_bytes(kMsNT));
    bps = std::max(1, std::min(bps, kMsBlocksPerSm));
    g->ms_grid = std::min<int>(g->nsm * bps, (int)kMaxBlocks);
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const uint32_t nwords = (uint32_t)((n + 31) / 32);
  const int blocks = std::max(1, std::min<int>(g->nsm * 4, (int)((n + 255) / 256)));
  for (int l = 0; l < L.nlanes; ++l) {
    cudaMemsetAsync(g->ws + L.lane[l].ctrl, 0, sizeof(Ctrl), st);
    cudaMemsetAsync(g->ws + L.lane[l].cand, 0, 4 * (size_t)nwords, st);  // zero between uses
  }
  for (int l = 0; l < L.ms_nlanes; ++l) cudaMemsetAsync(g->ws + L.ms[l].msctrl, 0, sizeof(MsCtrl), st);
  if (flags & DAWN_GRAPH_VALIDATE) {
    k_validate<<<blocks, 256, 0, st>>>(row_ptr, col, n, m, &at<Ctrl>(g, L.ctrl)->err);
    if (!sym && has_csc && m > 0)
      k_validate<<<blocks, 256, 0, st>>>(in_row_ptr, in_col, n, m, &at<Ctrl>(g, L.ctrl)->err);
    uint32_t err = 0;
    cudaMemcpyAsync(&err, &at<Ctrl>(g, L.ctrl)->err, 4, cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) { delete g; return cuda_fail(e, "validate"); }
    if (err) {
      delete g;
      return fail(DAWN_ERR_INVALID_GRAPH, "CSR invariant violated:%s%s%s",
                  (err & 1) ? " row_ptr[0]!=0 or row_ptr[n]!=m" : "",
                  (err & 2) ? " row_ptr not monotone" : "",
                  (err & 4) ? " column id out of range" : "");
    }
  }
  k_offsets32<<<blocks, 256, 0, st>>>(row_ptr, at<uint32_t>(g, L.rp), n + 1);
  const uint32_t *irp = at<uint32_t>(g, L.rp);
  if (!sym) {
    if (has_csc) {
      k_offsets32<<<blocks, 256, 0, st>>>(in_row_ptr, at<uint32_t>(g, L.irp), n + 1);
      irp = at<uint32_t>(g, L.irp);
    } else {
      // no CSC: treat every vertex as possibly reachable (noin = 0) — push only
      cudaMemsetAsync(g->ws + L.irp, 0, 4 * (size_t)(n + 1), st);
    }
  }
  if (sym || has_csc) {
    k_noin<<<blocks, 256, 0, st>>>(irp, (uint32_t)n, nwords, at<uint32_t>(g, L.noin),
                                   &at<Ctrl>(g, L.ctrl)->n_hasin);
  } else {
    cudaMemsetAsync(g->ws + L.noin, 0, 4 * (size_t)nwords, st);
    uint32_t nh = (uint32_t)n;
    cudaMemcpyAsync(&at<Ctrl>(g, L.ctrl)->n_hasin, &nh, 4, cudaMemcpyHostToDevice, st);
    cudaStreamSynchronize(st);
  }
  // static heavy-row pieces: out-rows (push side of the 64-source kernel) and in-rows (pull)
  {
    const uint32_t nblk = (uint32_t)((n + kScanBlock - 1) / kScanBlock);
    Ctrl *C = at<Ctrl>(g, L.ctrl);
    auto build_list = [&](const uint32_t *rows, const HeavyList &h, uint32_t *count) {
      k_hcount<<<nblk, 256, 0, st>>>(rows, (uint32_t)n, at<uint32_t>(g, h.bits),
                                     at<uint32_t>(g, L.scan_tmp));
      k_hscan<<<1, 32, 0, st>>>(at<uint32_t>(g, L.scan_tmp), nblk, count);
      const size_t cap = (size_t)m / kHPiece + 3;
      uint32_t *hc = at<uint32_t>(g, L.piece_tmp), *base = hc + cap, *cursor = base + cap,
               *maxc = cursor + cap;
      cudaMemsetAsync(hc, 0, 4 * cap, st);
      cudaMemsetAsync(maxc, 0, 4, st);
      k_hhist<<<blocks, 256, 0, st>>>(rows, (uint32_t)n, hc, maxc);
      k_hbase<<<1, 32, 0, st>>>(hc, base, cursor, maxc);
      k_hfill<<<blocks, 256, 0, st>>>(rows, (uint32_t)n, base, cursor, at<uint32_t>(g, h.v),
                                      at<uint32_t>(g, h.s), at<uint32_t>(g, h.e));
    };
    build_list(at<uint32_t>(g, L.rp), L.hout, &C->n_hp_out);
    if (L.own_irp) {
      if (has_csc) {
        build_list(at<uint32_t>(g, L.irp), L.hin, &C->n_hp_in);
      } else {
        cudaMemsetAsync(g->ws + L.hin.bits, 0, 4 * (size_t)nwords, st);
        cudaMemsetAsync(&C->n_hp_in, 0, 4, st);
      }
    } else {
      cudaMemcpyAsync(&C->n_hp_in, &C->n_hp_out, 4, cudaMemcpyDeviceToDevice, st);
    }
  }
  if ((sym || has_csc) && m > 0 && L.icol2) {  // degree-ordered in-rows for the pull probes
    const uint32_t *irp2 = sym ? at<uint32_t>(g, L.rp) : at<uint32_t>(g, L.irp);
    k_topk_rows<<<g->nsm * 8, 256, 0, st>>>(irp2, sym ? col : in_col, at<uint32_t>(g, L.rp),
                                            (uint32_t)n, at<int32_t>(g, L.icol2));
    g->icol = at<int32_t>(g, L.icol2);
    k_top1<<<g->nsm * 8, 256, 0, st>>>(irp2, at<int32_t>(g, L.icol2), (uint32_t)n,
                                       at<uint32_t>(g, L.top1));
  }
  if (sym || has_csc) {  // unreached-list seed for the pull sweep
    const uint32_t nblk = (uint32_t)((n + kScanBlock - 1) / kScanBlock);
    const uint32_t *irp2 = sym ? at<uint32_t>(g, L.rp) : at<uint32_t>(g, L.irp);
    k_lcount<<<nblk, 256, 0, st>>>(irp2, (uint32_t)n, at<uint32_t>(g, L.scan_tmp));
    k_hscan<<<1, 32, 0, st>>>(at<uint32_t>(g, L.scan_tmp), nblk, at<uint32_t>(g, L.useg));  // total -> scratch
    k_lfill<<<nblk, 256, 0, st>>>(irp2, (uint32_t)n, at<uint32_t>(g, L.scan_tmp),
                                  at<uint32_t>(g, L.hasin));
  }
  if (L.arc)
    k_arcs<<<g->nsm * 8, 256, 0, st>>>(col, at<uint32_t>(g, L.rp), m, at<uint4>(g, L.arc));
  unsigned long long loc[2] = {0, 0};
  if (g->narrow_ok) {
    unsigned long long *dcnt = at<unsigned long long>(g, L.useg);  // scratch (pull segments)
    cudaMemsetAsync(dcnt, 0, 16, st);
    k_locality<<<g->nsm * 4, 256, 0, st>>>(at<uint32_t>(g, L.rp), col,
                                             (uint32_t)std::min<int64_t>(n, 1 << 20), dcnt);
    cudaMemcpyAsync(loc, dcnt, 16, cudaMemcpyDeviceToHost, st);
  }
  uint32_t nh = 0;
  cudaMemcpyAsync(&nh, &at<Ctrl>(g, L.ctrl)->n_hasin, 4, cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) { delete g; return cuda_fail(e, "graph load"); }
  g->n_hasin = nh;
  // owner computes when at least half of the sampled arcs stay within a CTA (meshes, road
  // networks: ~97% on the 4096^2 grid); then the cluster keeps the whole search unless a queue
  // overflows.  Otherwise the cluster only runs the narrow first levels (frontier rows totalling
  // <= 1024 arcs) and hands the wide ones to the grid-wide kernel.
  g->narrow_owner = loc[1] > 0 && 2 * loc[0] >= loc[1];
  g->handover_m = g->narrow_owner ? ~0ull : 1024ull;
  // Other graphs start on the grid-wide kernel by default: their narrow first levels are a
  // few microseconds, less than the extra kernel boundary (measured on Kronecker-20: +6 us).
  g->cluster_start = g->narrow_owner;
  // the other lanes' control blocks get lane 0's load-time fields (n_hasin, heavy-piece counts)
  for (int l = 1; l < L.nlanes; ++l)
    cudaMemcpyAsync(g->ws + L.lane[l].ctrl, g->ws + L.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToDevice, st);
  if (L.nlanes > 1) {
    bool ok = cudaEventCreateWithFlags(&g->ev_fork, cudaEventDisableTiming) == cudaSuccess;
    for (int l = 1; l < L.nlanes && ok; ++l)
      ok = cudaStreamCreateWithFlags(&g->lane_st[l], cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&g->ev_join[l], cudaEventDisableTiming) == cudaSuccess;
    g->lanes = ok ? std::min(L.nlanes, kDefaultLanes(n)) : 1;
    g->ms_lanes = ok ? std::min(L.ms_nlanes, kDefaultMsLanes) : 1;
  }
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) { delete g; return cuda_fail(e, "graph load"); }
  if ((e = cudaGetLastError()) != cudaSuccess) { delete g; return cuda_fail(e, "graph load"); }
  *out = g;
  return DAWN_OK;
}

dawn_status set_param(dawn_graph g, dawn_param key, double value) {
  if (!g) return fail(DAWN_ERR_INVALID_ARGUMENT, "graph is NULL");
  if (!(value >= 0)) return fail(DAWN_ERR_INVALID_ARGUMENT, "value must be >= 0");
  switch (key) {
    case DAWN_PARAM_ALPHA: g->alpha = (float)value; break;
    case DAWN_PARAM_BETA: g->beta = (float)value; break;
    case DAWN_PARAM_MS_ALPHA: g->ms_alpha = (float)value; break;
    case DAWN_PARAM_BITMAP_PUSH_EDGES: g->bmpush_e = (uint32_t)std::min(value, 4294967295.0); break;
    case DAWN_PARAM_SOLO_EDGES: g->solo_e = (uint32_t)std::min(value, 4294967295.0); break;
    case DAWN_PARAM_BITMAP_PUSH_GROW_EDGES:
      g->bmpush_grow = (uint32_t)std::min(value, 4294967295.0);
      break;
    case DAWN_PARAM_CLUSTER_START: g->cluster_start = value != 0; break;
    case DAWN_PARAM_CLUSTER_HANDOVER_EDGES:
      g->handover_m = value >= 1.8e19 ? ~0ull : (unsigned long long)value;
      break;
    case DAWN_PARAM_BATCH_LANES:
      if (value < 1 || value > g->L.nlanes || (value > 1 && !g->ev_fork))
        return fail(DAWN_ERR_INVALID_ARGUMENT, "batch lanes must be in [1, %d]", g->L.nlanes);
      g->lanes = (int)value;
      break;
    case DAWN_PARAM_WEIGHT_DELTA: g->wdelta = (uint32_t)std::min(value, 4294967294.0); break;
    case DAWN_PARAM_BATCH_DYNAMIC: g->batch_claim = value != 0; break;
    case DAWN_PARAM_MS_LANES:
      if (value < 1 || value > g->L.ms_nlanes || (value > 1 && !g->ev_fork))
        return fail(DAWN_ERR_INVALID_ARGUMENT, "multi-source lanes must be in [1, %d]", g->L.ms_nlanes);
      g->ms_lanes = (int)value;
      break;
    case DAWN_PARAM_DENSE_MAX_ENTRIES:
      if (value < 1) return fail(DAWN_ERR_INVALID_ARGUMENT, "dense limit must be >= 1");
      g->dense_max = std::min(value, 1099511627776.0);
      break;
    case DAWN_PARAM_NARROW_QUEUE_CAP:
      if (value < 32) return fail(DAWN_ERR_INVALID_ARGUMENT, "queue capacity must be >= 32");
      g->narrow_qcap = (uint32_t)std::min<double>(value, g->narrow_qcap_max);
      break;
    default: return fail(DAWN_ERR_INVALID_ARGUMENT, "unknown parameter");
  }
  return DAWN_OK;
}

SsspParams sssp_params(dawn_graph g, uint32_t variant, uint32_t *dist, dawn_sssp_stats *stats,
                       int lane = 0) {
  const Layout &L = g->L;
  const LaneLayout &Q = L.lane[lane];
  SsspParams p{};
  p.n = (uint32_t)g->n;
  p.nwords = (uint32_t)((g->n + 31) / 32);
  p.m = (unsigned long long)g->m;
  p.rp = at<uint32_t>(g, L.rp);
  p.irp = at<uint32_t>(g, L.irp);
  p.col = g->col;
  p.icol = g->icol;
  p.noin = at<uint32_t>(g, L.noin);
  p.hin_v = at<uint32_t>(g, L.hin.v);
  p.hin_s = at<uint32_t>(g, L.hin.s);
  p.hin_e = at<uint32_t>(g, L.hin.e);
  p.hin_bits = at<uint32_t>(g, L.hin.bits);
  p.top1 = (DAWN_PULL_TOP1 && L.top1 && g->icol == at<int32_t>(g, L.icol2)) ? at<uint32_t>(g, L.top1)
                                                                           : nullptr;
  p.vis = at<uint32_t>(g, Q.vis);
  p.cand = at<uint32_t>(g, Q.cand);
  p.hasin = at<uint32_t>(g, L.hasin);
  p.ulist = at<uint32_t>(g, Q.ulist);
  p.useg = at<uint32_t>(g, Q.useg);
  p.n_hasin = g->n_hasin;
  for (int i = 0; i < 3; ++i) p.fb[i] = at<uint32_t>(g, Q.fb[i]);
  p.trace = (g->trace && lane == 0) ? at<TraceRec>(g, L.trace) : nullptr;
  for (int i = 0; i < 2; ++i) {
    p.Lv[i] = at<uint32_t>(g, Q.Lv[i]);
    p.Lsd[i] = at<uint2>(g, Q.Lsd[i]);
    p.Cf[i] = at<uint32_t>(g, Q.Cf[i]);
  }
  p.ctrl = at<Ctrl>(g, Q.ctrl);
  p.dist = dist;
  p.stats = stats;
  p.variant = variant;
  p.can_pull = g->has_csc ? 1u : 0u;
  p.sym = (g->flags & DAWN_GRAPH_SYMMETRIC) ? 1u : 0u;
  p.alpha = g->alpha;
  p.beta = g->beta;
  p.bmpush_e = g->bmpush_e;
  p.solo_e = g->solo_e;
  p.bmpush_grow = std::min(g->bmpush_grow, g->bmpush_e);
  p.seq = ++g->seq;
  return p;
}

dawn_status launch_sssp(dawn_graph g, SsspParams &p, cudaStream_t stream, int lanes = 1) {
  // batch lanes run the 2-CTA/SM (64-register) instantiation on every graph: twice the warps
  // per SM hide the latency of several concurrent searches (Kronecker-20 at 8 lanes: 1,030 ->
  // 1,349 GTEPS); one search on a graph up to 2^22 vertices keeps the 1-CTA/SM one
  const bool two = !g->sssp_one || (DAWN_BATCH_TWO && lanes > 1);
  int grid = std::max(1, (two ? g->sssp_grid2 : g->sssp_grid) / lanes);
  if (g->m + g->n <= kOneCtaMaxNM) grid = 1;  // tiny graphs: one CTA, barriers are __syncthreads
  void *args[] = {&p};
  const void *kfn = two ? (const void *)k_sssp<kNT, 2> : (const void *)k_sssp<kNT, 1>;
  cudaError_t e = cudaLaunchCooperativeKernel(kfn, dim3(grid), dim3(kNT), args, 0, stream);
  if (e != cudaSuccess) return cuda_fail(e, "k_sssp launch");
  return DAWN_OK;
}

dawn_status launch_narrow(dawn_graph g, const SsspParams &p, uint32_t source,
                          const uint32_t *src_dev, cudaStream_t stream) {
  const Layout &L = g->L;
  NarrowParams np{};
  np.n = p.n;
  np.nwords = p.nwords;
  np.wpc = g->narrow_wpc;
  np.qcap = g->narrow_qcap;
  np.rp = p.rp;
  np.arc = L.arc ? at<uint4>(g, L.arc) : nullptr;
  np.col = g->col;
  np.owner = g->narrow_owner ? 1u : 0u;
  np.handover_m = g->handover_m;
  np.noin = p.noin;
  np.vis = p.vis;
  np.dist = p.dist;
  np.fb0 = p.fb[0];
  np.fb1 = p.fb[1];
  np.ctrl = p.ctrl;
  np.stats = p.stats;
  np.source = source;
  np.src_dev = src_dev;
  np.vsrc = p.vsrc;
  np.vn = p.vn;
  np.max_reach_base = g->n_hasin;
  np.seq = p.seq;
  np.trace = p.trace;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kNarrowCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(g->narrow_grid);
  cfg.blockDim = dim3(kNarrowThreads);
  cfg.dynamicSmemBytes = g->narrow_smem;
  cfg.stream = stream;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_narrow, np);
  if (e != cudaSuccess) return cuda_fail(e, "k_narrow launch");
  return DAWN_OK;
}

dawn_status sssp_one(dawn_graph g, int64_t source, uint32_t variant, uint32_t *dist,
                     dawn_sssp_stats *stats, void *stream) {
  if (!g || !dist) return fail(DAWN_ERR_INVALID_ARGUMENT, "graph or dist is NULL");
  if (variant > DAWN_PULL) return fail(DAWN_ERR_INVALID_ARGUMENT, "unknown variant");
  if (source < 0 || source >= g->n)
    return fail(DAWN_ERR_BOUNDS, "source %lld not in [0, n)", (long long)source);
  if (variant == DAWN_PULL && !g->has_csc)
    return fail(DAWN_ERR_CONFIG, "PULL needs CSC (in-edges) on a directed graph");
  dawn_status s = set_device(g);
  if (s != DAWN_OK) return s;
  const Layout &L = g->L;
  const size_t small_bytes = small_smem_bytes(g->n, g->m);
  if (variant != DAWN_PULL && !g->trace && small_bytes <= g->small_cap) {
    // whole SSSP in one CTA's shared memory (tiny graphs, e.g. configs[0])
    SmallParams sp{(uint32_t)g->n, (uint32_t)g->m, at<uint32_t>(g, L.rp), g->col, dist, stats,
                   (uint32_t)source, nullptr, 0u, &at<Ctrl>(g, L.ctrl)->bad_src};
    k_small<1024><<<1, 1024, small_bytes, static_cast<cudaStream_t>(stream)>>>(sp);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "k_small launch");
    return DAWN_OK;
  }
  SsspParams p = sssp_params(g, variant, dist, stats);
  p.source = (uint32_t)source;
  if (variant != DAWN_PULL && g->narrow_ok && g->cluster_start) {
    // the search starts on one 16-CTA cluster (state in distributed shared memory); k_sssp
    // below resumes from its hand-over (wide frontier or full queue) or exits at once
    dawn_status sn = launch_narrow(g, p, (uint32_t)source, nullptr, static_cast<cudaStream_t>(stream));
    if (sn != DAWN_OK) return sn;
  }
  return launch_sssp(g, p, static_cast<cudaStream_t>(stream));
}

dawn_status sssp_batch(dawn_graph g, const uint32_t *sources, int64_t k, uint32_t variant,
                       uint32_t *dist, dawn_sssp_stats *stats, void *stream) {
  if (!g || k < 0 || (k > 0 && (!dist || !sources)))
    return fail(DAWN_ERR_INVALID_ARGUMENT, "bad arguments");
  if (variant > DAWN_PULL) return fail(DAWN_ERR_INVALID_ARGUMENT, "unknown variant");
  if (variant == DAWN_PULL && !g->has_csc)
    return fail(DAWN_ERR_CONFIG, "PULL needs CSC (in-edges) on a directed graph");
  if (k == 0) return DAWN_OK;
  if (k >= (int64_t(1) << 32)) return fail(DAWN_ERR_CAPACITY, "k too large");
  dawn_status s = set_device(g);
  if (s != DAWN_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t small_bytes = small_smem_bytes(g->n, g->m);
  if (variant != DAWN_PULL && !g->trace && small_bytes <= g->small_cap) {
    // tiny graphs: the searches are independent, so up to one CTA per SM, each loading the CSR
    // into its shared memory once and running searches blockIdx.x, blockIdx.x + grid, ...
    SmallParams sp{(uint32_t)g->n, (uint32_t)g->m, at<uint32_t>(g, g->L.rp), g->col, dist, stats,
                   0u, sources, (uint32_t)k, &at<Ctrl>(g, g->L.ctrl)->bad_src};
    const unsigned grid = (unsigned)std::min<int64_t>(k, g->nsm);
    k_small<1024><<<grid, 1024, small_bytes, st>>>(sp);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "k_small launch");
    return DAWN_OK;
  }
  if (variant != DAWN_PULL && g->narrow_ok && g->cluster_start) {
    // cluster-start graphs: per search, k_narrow then k_sssp (resume or exit), both reading the
    // source id from the device list; every launch validates the whole list first
    for (int64_t i = 0; i < k; ++i) {
      SsspParams p = sssp_params(g, variant, dist + (size_t)i * g->n, stats ? stats + i : nullptr);
      p.sources = sources + i;
      p.nsrc = 1;
      p.vsrc = sources;
      p.vn = (uint32_t)k;
      dawn_status sn = launch_narrow(g, p, 0u, sources + i, st);
      if (sn != DAWN_OK) return sn;
      sn = launch_sssp(g, p, st);
      if (sn != DAWN_OK) return sn;
    }
    return DAWN_OK;
  }
  const int lanes = (g->trace || k < 2) ? 1 : (int)std::min<int64_t>(g->lanes, k);
  if (lanes > 1) {
    // dynamic lanes: a shared claim counter (lane 0's control block) hands out the batch
    // indices, one per search, so no lane idles while another finishes a long share
    uint32_t *claim = g->batch_claim ? &at<Ctrl>(g, g->L.lane[0].ctrl)->claim : nullptr;
    if (claim) {
      cudaError_t ec = cudaMemsetAsync(claim, 0, 4, st);
      if (ec != cudaSuccess) return cuda_fail(ec, "batch claim reset");
    }
    // independent searches at once: lane l (its own per-search state, its own stream, grid/lanes
    // CTAs) runs the contiguous share [k*l/lanes, k*(l+1)/lanes) of the batch; every lane
    // validates the whole list first, so a bad id still means nothing is written
    cudaError_t e = cudaEventRecord(g->ev_fork, st);
    for (int l = 1; l < lanes && e == cudaSuccess; ++l) e = cudaStreamWaitEvent(g->lane_st[l], g->ev_fork, 0);
    if (e != cudaSuccess) return cuda_fail(e, "batch fork");
    for (int l = 0; l < lanes; ++l) {
      const int64_t b = claim ? 0 : k * l / lanes, c = claim ? k : k * (l + 1) / lanes - b;
      SsspParams p = sssp_params(g, variant, dist + (size_t)b * g->n, stats ? stats + b : nullptr, l);
      p.sources = sources + b;
      p.nsrc = (uint32_t)c;
      p.claim = claim;
      p.vsrc = sources;
      p.vn = (uint32_t)k;
      dawn_status sl = launch_sssp(g, p, l ? g->lane_st[l] : st, lanes);
      if (sl != DAWN_OK) return sl;
    }
    for (int l = 1; l < lanes && e == cudaSuccess; ++l) {
      e = cudaEventRecord(g->ev_join[l], g->lane_st[l]);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(st, g->ev_join[l], 0);
    }
    if (e != cudaSuccess) return cuda_fail(e, "batch join");
    return DAWN_OK;
  }
  SsspParams p = sssp_params(g, variant, dist, stats);
  p.sources = sources;
  p.nsrc = (uint32_t)k;
  p.vsrc = sources;
  p.vn = (uint32_t)k;
  return launch_sssp(g, p, st);
}

dawn_status graph_check(dawn_graph g, void *stream) {
  if (!g) return fail(DAWN_ERR_INVALID_ARGUMENT, "graph is NULL");
  dawn_status s = set_device(g);
  if (s != DAWN_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint32_t bad = 0;
  uint32_t *flag = &at<Ctrl>(g, g->L.ctrl)->bad_src;
  cudaError_t e = cudaMemcpyAsync(&bad, flag, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "dawn_graph_check");
  if (bad) {
    cudaMemsetAsync(flag, 0, 4, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "dawn_graph_check");
    return fail(DAWN_ERR_BOUNDS, "a dawn_sssp_batch source id was not in [0, n); nothing written");
  }
  return DAWN_OK;
}

// One k_ms64 launch of lane `l` over cnt sources (its own state; grid = its share of the SMs).
dawn_status launch_ms_lane(dawn_graph g, int l, const uint32_t *src, size_t cnt, size_t off,
                           uint32_t *dist, dawn_record *rec, int grid, cudaStream_t st) {
  const Layout &L = g->L;
  const MsLaneLayout &Q = L.ms[l];
  cudaError_t e = cudaMemcpyAsync(g->ws + Q.srcbuf, src, 4 * cnt, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "source upload");
  MsParams p{};
  p.n = (uint32_t)g->n;
  p.nwords = (uint32_t)((g->n + 31) / 32);
  p.m = (unsigned long long)g->m;
  p.rp = at<uint32_t>(g, L.rp);
  p.irp = at<uint32_t>(g, L.irp);
  p.col = g->col;
  p.icol = g->icol;
  p.hout_v = at<uint32_t>(g, L.hout.v);
  p.hout_s = at<uint32_t>(g, L.hout.s);
  p.hout_e = at<uint32_t>(g, L.hout.e);
  p.hout_bits = at<uint32_t>(g, L.hout.bits);
  p.hin_v = at<uint32_t>(g, L.hin.v);
  p.hin_s = at<uint32_t>(g, L.hin.s);
  p.hin_e = at<uint32_t>(g, L.hin.e);
  p.hin_bits = at<uint32_t>(g, L.hin.bits);
  p.sctrl = at<Ctrl>(g, L.ctrl);
  p.seen = at<unsigned long long>(g, Q.seen);
  p.F[0] = at<unsigned long long>(g, Q.F0);
  p.F[1] = at<unsigned long long>(g, Q.F1);
  p.nxt = at<unsigned long long>(g, Q.nxt);
  p.ctrl = at<MsCtrl>(g, Q.msctrl);
  p.sources = at<uint32_t>(g, Q.srcbuf);
  p.count = (uint32_t)cnt;
  p.rec = rec ? rec + off : nullptr;
  p.dist = dist ? dist + off * (size_t)g->n : nullptr;
  p.can_pull = g->has_csc ? 1u : 0u;
  p.sym = (g->flags & DAWN_GRAPH_SYMMETRIC) ? 1u : 0u;
  p.ms_alpha = g->ms_alpha;
  p.part = at<uint4>(g, Q.part);
  p.trace = (g->trace && l == 0) ? at<TraceRec>(g, L.trace) : nullptr;
  p.trace_n = &at<Ctrl>(g, L.ctrl)->trace_n;
  void *args[] = {&p};
  e = cudaLaunchCooperativeKernel((const void *)k_ms64<kMsNT>, dim3(grid), dim3(kMsNT), args,
                                  ms_smem_bytes(kMsNT), st);
  if (e != cudaSuccess) return cuda_fail(e, "k_ms64 launch");
  return DAWN_OK;
}

dawn_status launch_ms(dawn_graph g, const std::vector<uint32_t> &src, uint32_t *dist,
                      dawn_record *rec, cudaStream_t st) {
  const Layout &L = g->L;
  const size_t chunk = (L.srccap / kMsBatch) * kMsBatch;
  for (size_t off = 0; off < src.size(); off += chunk) {
    const size_t cnt = std::min(src.size() - off, chunk);
    const size_t nb = (cnt + kMsBatch - 1) / kMsBatch;
    int lanes = (g->trace || g->m + g->n <= kOneCtaMaxNM) ? 1 : (int)std::min<size_t>(g->ms_lanes, nb);
    if (lanes > 1 && !g->ev_fork) lanes = 1;
    if (lanes == 1) {
      int grid = g->ms_grid;
      if (g->m + g->n <= kOneCtaMaxNM) grid = 1;
      dawn_status s = launch_ms_lane(g, 0, src.data() + off, cnt, off, dist, rec, grid, st);
      if (s != DAWN_OK) return s;
      continue;
    }
    // independent batches at once: lane l runs the contiguous batch share
    // [nb*l/lanes, nb*(l+1)/lanes) on grid/lanes CTAs with its own state and stream
    cudaError_t e = cudaEventRecord(g->ev_fork, st);
    for (int l = 1; l < lanes && e == cudaSuccess; ++l) e = cudaStreamWaitEvent(g->lane_st[l], g->ev_fork, 0);
    if (e != cudaSuccess) return cuda_fail(e, "ms fork");
    for (int l = 0; l < lanes; ++l) {
      const size_t b0 = nb * l / lanes * kMsBatch, b1 = std::min(cnt, nb * (l + 1) / lanes * kMsBatch);
      dawn_status s = launch_ms_lane(g, l, src.data() + off + b0, b1 - b0, off + b0, dist, rec,
                                     std::max(1, g->ms_grid / lanes), l ? g->lane_st[l] : st);
      if (s != DAWN_OK) return s;
    }
    for (int l = 1; l < lanes && e == cudaSuccess; ++l) {
      e = cudaEventRecord(g->ev_join[l], g->lane_st[l]);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(st, g->ev_join[l], 0);
    }
    if (e != cudaSuccess) return cuda_fail(e, "ms join");
  }
  return DAWN_OK;
}

dawn_status msssp(dawn_graph g, const int64_t *sources, int64_t k, uint32_t *dist,
                  dawn_record *rec, void *stream) {
  if (!g || (!sources && k > 0) || k < 0) return fail(DAWN_ERR_INVALID_ARGUMENT, "bad arguments");
  if (g->lean) return fail(DAWN_ERR_CONFIG, "graph loaded with DAWN_GRAPH_LEAN (no multi-source words)");
  for (int64_t i = 0; i < k; ++i)
    if (sources[i] < 0 || sources[i] >= g->n)
      return fail(DAWN_ERR_BOUNDS, "sources[%lld] = %lld not in [0, n)", (long long)i,
                  (long long)sources[i]);
  if (dist && (double)k * (double)g->n >= g->dense_max)
    return fail(DAWN_ERR_CAPACITY, "k*n above the dense-output limit (use dawn_apsp_rows)");
  if (k == 0) return DAWN_OK;
  dawn_status s = set_device(g);
  if (s != DAWN_OK) return s;
  std::vector<uint32_t> src(sources, sources + k);
  return launch_ms(g, src, dist, rec, static_cast<cudaStream_t>(stream));
}

dawn_status graph_trace(dawn_graph g, dawn_trace_rec *host_out, int64_t cap, int64_t *count,
                        void *stream) {
  if (!g || !count || (cap > 0 && !host_out)) return fail(DAWN_ERR_INVALID_ARGUMENT, "bad arguments");
  if (!g->trace) return fail(DAWN_ERR_CONFIG, "graph loaded without DAWN_GRAPH_TRACE");
  dawn_status s = set_device(g);
  if (s != DAWN_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint32_t nrec = 0;
  cudaMemcpyAsync(&nrec, &at<Ctrl>(g, g->L.ctrl)->trace_n, 4, cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "trace");
  const int64_t k = std::min<int64_t>(cap, nrec);
  static_assert(sizeof(dawn_trace_rec) == sizeof(TraceRec), "trace record layout");
  if (k > 0) {
    e = cudaMemcpy(host_out, g->ws + g->L.trace, sizeof(TraceRec) * k, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "trace copy");
  }
  static_assert(DAWN_TRACE_CAP == kTraceCap, "dawn.h DAWN_TRACE_CAP");
  if (cap >= kTraceCap) {
    e = cudaMemcpy(host_out + (kTraceCap - 1), g->ws + g->L.trace + sizeof(TraceRec) * (kTraceCap - 1),
                   sizeof(TraceRec), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "trace copy");
  }
  *count = nrec;
  return DAWN_OK;
}

dawn_status apsp_shard(int64_t k, int32_t rank, int32_t world, int64_t *idx, int64_t cap,
                       int64_t *count) {
  if (k < 0 || world < 1 || rank < 0 || rank >= world || !count)
    return fail(DAWN_ERR_INVALID_ARGUMENT, "need k >= 0, 0 <= rank < world");
  int64_t c = 0;
  const int64_t B = kMsBatch;
  const int64_t nb = (k + B - 1) / B;
  for (int64_t b = rank; b < nb; b += world) {
    const int64_t e = std::min(k, (b + 1) * B);
    for (int64_t i = b * B; i < e; ++i) {
      if (idx && c < cap) idx[c] = i;
      ++c;
    }
  }
  *count = c;
  if (idx && c > cap) return fail(DAWN_ERR_CAPACITY, "idx capacity too small");
  return DAWN_OK;
}

dawn_status apsp(dawn_graph g, const int64_t *sources, int64_t k, int32_t rank, int32_t world,
                 dawn_record *rec, int64_t cap, int64_t *n_written, void *stream) {
  if (!g || !rec || !n_written || (!sources && k > 0) || k < 0)
    return fail(DAWN_ERR_INVALID_ARGUMENT, "bad arguments");
  if (world < 1 || rank < 0 || rank >= world)
    return fail(DAWN_ERR_INVALID_ARGUMENT, "need 0 <= rank < world");
  if (g->lean) return fail(DAWN_ERR_CONFIG, "graph loaded with DAWN_GRAPH_LEAN (no multi-source words)");
  for (int64_t i = 0; i < k; ++i)
    if (sources[i] < 0 || sources[i] >= g->n)
      return fail(DAWN_ERR_BOUNDS, "sources[%lld] not in [0, n)", (long long)i);
  std::vector<uint32_t> mine;
  const int64_t B = kMsBatch;
  const int64_t nb = (k + B - 1) / B;
  for (int64_t b = rank; b < nb; b += world)
    for (int64_t i = b * B; i < std::min(k, (b + 1) * B); ++i) mine.push_back((uint32_t)sources[i]);
  *n_written = (int64_t)mine.size();
  if ((int64_t)mine.size() > cap) return fail(DAWN_ERR_CAPACITY, "rec capacity too small");
  if (mine.empty()) return DAWN_OK;
  dawn_status s = set_device(g);
  if (s != DAWN_OK) return s;
  return launch_ms(g, mine, nullptr, rec, static_cast<cudaStream_t>(stream));
}

// Owns the host-side resources of one dawn_apsp_rows call (no device memory).
struct RowsRes {
  cudaStream_t copy = nullptr;
  cudaEvent_t done[2] = {}, landed[2] = {};
  ~RowsRes() {
    for (int i = 0; i < 2; ++i) {
      if (done[i]) cudaEventDestroy(done[i]);
      if (landed[i]) cudaEventDestroy(landed[i]);
    }
    if (copy) cudaStreamDestroy(copy);
  }
};

dawn_status apsp_rows(dawn_graph g, const int64_t *sources, int64_t k, int64_t chunk,
                      uint32_t *dev_stage, uint32_t *host_stage, dawn_row_sink sink, void *user,
                      void *stream) {
  if (!g || !sink || k < 0 || (k > 0 && (!sources || !dev_stage || !host_stage)) || chunk < 1)
    return fail(DAWN_ERR_INVALID_ARGUMENT, "bad arguments");
  if (g->lean) return fail(DAWN_ERR_CONFIG, "graph loaded with DAWN_GRAPH_LEAN (no multi-source words)");
  for (int64_t i = 0; i < k; ++i)
    if (sources[i] < 0 || sources[i] >= g->n)
      return fail(DAWN_ERR_BOUNDS, "sources[%lld] = %lld not in [0, n)", (long long)i,
                  (long long)sources[i]);
  if ((double)chunk * (double)g->n >= g->dense_max)
    return fail(DAWN_ERR_CAPACITY, "chunk*n above the dense-output limit");
  if (k == 0) return DAWN_OK;
  dawn_status s = set_device(g);
  if (s != DAWN_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  RowsRes R;
  cudaError_t e = cudaStreamCreateWithFlags(&R.copy, cudaStreamNonBlocking);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&R.done[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&R.landed[i], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) return cuda_fail(e, "dawn_apsp_rows resources");
  const size_t n = (size_t)g->n;
  const int64_t np = (k + chunk - 1) / chunk;
  std::vector<uint32_t> src;
  src.reserve((size_t)std::min(k, chunk));
  // piece p: compute into dev_stage[p % 2] on `stream`, D2H into host_stage[p % 2] on the copy
  // stream, sink(p) on this thread once it landed; piece p + 1 computes meanwhile
  for (int64_t p = 0; p <= np; ++p) {
    if (p < np) {
      const int64_t b = p * chunk, c = std::min(k, b + chunk) - b;
      const int slot = (int)(p & 1);
      uint32_t *d = dev_stage + (size_t)slot * (size_t)chunk * n;
      src.assign(sources + b, sources + b + c);
      // dev_stage[slot] is free once piece p - 2's copy has left it
      if (p >= 2 && (e = cudaStreamWaitEvent(st, R.landed[slot], 0)) != cudaSuccess)
        return cuda_fail(e, "dawn_apsp_rows");
      if ((s = launch_ms(g, src, d, nullptr, st)) != DAWN_OK) {
        cudaStreamSynchronize(R.copy);
        return s;
      }
      if ((e = cudaEventRecord(R.done[slot], st)) != cudaSuccess) return cuda_fail(e, "dawn_apsp_rows");
    }
    if (p >= 1) {  // hand piece p - 1 to the sink (host_stage[slot] was enqueued last iteration)
      const int slot = (int)((p - 1) & 1);
      if ((e = cudaEventSynchronize(R.landed[slot])) != cudaSuccess) return cuda_fail(e, "dawn_apsp_rows copy");
      const int64_t b = (p - 1) * chunk, c = std::min(k, b + chunk) - b;
      if (sink(user, b, c, host_stage + (size_t)slot * (size_t)chunk * n) != 0) {
        // nothing may still write the caller's buffers once we return
        cudaStreamSynchronize(st);
        cudaStreamSynchronize(R.copy);
        return fail(DAWN_ERR_INVALID_ARGUMENT, "the row sink aborted at row %lld", (long long)b);
      }
    }
    if (p < np) {  // host_stage[slot] is free: its previous piece (p - 2) went to the sink
      const int slot = (int)(p & 1);
      const int64_t b = p * chunk, c = std::min(k, b + chunk) - b;
      e = cudaStreamWaitEvent(R.copy, R.done[slot], 0);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(host_stage + (size_t)slot * (size_t)chunk * n,
                            dev_stage + (size_t)slot * (size_t)chunk * n, 4 * (size_t)c * n,
                            cudaMemcpyDeviceToHost, R.copy);
      if (e == cudaSuccess) e = cudaEventRecord(R.landed[slot], R.copy);
      if (e != cudaSuccess) return cuda_fail(e, "dawn_apsp_rows copy");
    }
  }
  // `stream` must not run past the rows' copies (the caller may reuse dev_stage)
  if ((e = cudaStreamWaitEvent(st, R.landed[(np - 1) & 1], 0)) != cudaSuccess)
    return cuda_fail(e, "dawn_apsp_rows");
  if ((e = cudaStreamSynchronize(R.copy)) != cudaSuccess) return cuda_fail(e, "dawn_apsp_rows");
  return DAWN_OK;
}

dawn_status largest_wcc(dawn_graph g, int64_t *sources_out, int64_t *k, uint64_t *arcs,
                        void *stream) {
  if (!g || !k) return fail(DAWN_ERR_INVALID_ARGUMENT, "graph or k is NULL");
  dawn_status s = set_device(g);
  if (s != DAWN_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Layout &L = g->L;
  const uint32_t n = (uint32_t)g->n;
  // frontier scratch of the handle (no search is in flight: one call per handle at a time)
  uint32_t *par = at<uint32_t>(g, L.Lv[0]), *cnt = at<uint32_t>(g, L.Lv[1]);
  uint32_t *arcc = at<uint32_t>(g, L.ulist), *list = reinterpret_cast<uint32_t *>(g->ws + L.Lsd[0]);
  Ctrl *C = at<Ctrl>(g, L.ctrl);
  const int blocks = std::max(1, std::min<int>(g->nsm * 8, (int)((n + 255) / 256)));
  const uint32_t nblk = (n + kScanBlock - 1) / kScanBlock;
  cudaMemsetAsync(cnt, 0, 4 * (size_t)n, st);
  cudaMemsetAsync(arcc, 0, 4 * (size_t)n, st);
  cudaMemsetAsync(&C->wcc_cnt, 0, 8, st);            // wcc_cnt, wcc_arcs
  cudaMemsetAsync(&C->wcc_root, 0xff, 4, st);
  k_wcc_init<<<blocks, 256, 0, st>>>(par, n);
  if (g->m > 0) {
    k_wcc_hook_light<<<blocks, 256, 0, st>>>(at<uint32_t>(g, L.rp), g->col, n, par);
    k_wcc_hook_pieces<<<g->nsm * 8, 256, 0, st>>>(at<uint32_t>(g, L.hout.v),
                                                    at<uint32_t>(g, L.hout.s),
                                                    at<uint32_t>(g, L.hout.e), &C->n_hp_out,
                                                    g->col, par);
  }
  uint32_t *lab = reinterpret_cast<uint32_t *>(g->ws + L.Lsd[1]);  // final component labels
  k_wcc_count<<<blocks, 256, 0, st>>>(at<uint32_t>(g, L.rp), n, par, lab, cnt, arcc);
  for (int pass = 0; pass < 3; ++pass)
    k_wcc_select<<<blocks, 256, 0, st>>>(lab, cnt, arcc, n, pass, C);
  k_wcc_bcount<<<nblk, 256, 0, st>>>(lab, n, C, at<uint32_t>(g, L.scan_tmp));
  k_hscan<<<1, 32, 0, st>>>(at<uint32_t>(g, L.scan_tmp), nblk, &C->wcc_k);
  k_wcc_bfill<<<nblk, 256, 0, st>>>(lab, n, C, at<uint32_t>(g, L.scan_tmp), list);
  uint32_t hdr[3] = {0, 0, 0};  // wcc_cnt, wcc_arcs, wcc_root
  cudaError_t e = cudaMemcpyAsync(hdr, &C->wcc_cnt, 12, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "dawn_largest_wcc");
  const uint32_t kk = hdr[0];
  if (sources_out && kk) {
    std::vector<uint32_t> tmp(kk);
    e = cudaMemcpy(tmp.data(), list, 4 * (size_t)kk, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "dawn_largest_wcc copy");
    for (uint32_t i = 0; i < kk; ++i) sources_out[i] = tmp[i];
  }
  *k = kk;
  if (arcs) *arcs = hdr[1];
  return DAWN_OK;
}

dawn_status ms_counters(dawn_graph g, uint64_t *host_out, void *stream) {
  if (!g || !host_out) return fail(DAWN_ERR_INVALID_ARGUMENT, "graph or host_out is NULL");
  dawn_status s = set_device(g);
  if (s != DAWN_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int i = 0; i < 4; ++i) host_out[i] = 0;
  for (int l = 0; l < g->L.ms_nlanes; ++l) {  // summed over the multi-source lanes
    MsCtrl *C = at<MsCtrl>(g, g->L.ms[l].msctrl);
    uint64_t part[4] = {0, 0, 0, 0};
    cudaError_t e = cudaMemcpyAsync(part, C->stat, sizeof(C->stat), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(C->stat, 0, sizeof(C->stat), st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "dawn_graph_ms_counters");
    for (int i = 0; i < 4; ++i) host_out[i] += part[i];
  }
  return DAWN_OK;
}

// ---------------------------------------------------------------- compact distance rows
// out[i] = d[i] for d < 255, 255 otherwise (UNREACHED, or a finite distance that does not fit:
// then bit 0 of *flags is set).  4 distances per thread, one flag atomic per CTA at most.
__global__ void k_dist_u8(const uint32_t *__restrict__ d, int64_t count, uint8_t *__restrict__ out,
                          uint32_t *flags) {
  const int64_t n4 = count / 4;
  bool over = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 x = __ldcs(reinterpret_cast<const uint4 *>(d) + i);
    const uint32_t a[4] = {x.x, x.y, x.z, x.w};
    uint32_t packed = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t v = a[k] < 255u ? a[k] : 255u;
      over |= a[k] >= 255u && a[k] != kUnreached;
      packed |= v << (8 * k);
    }
    reinterpret_cast<uint32_t *>(out)[i] = packed;
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = d[i];
    over |= v >= 255u && v != kUnreached;
    out[i] = (uint8_t)(v < 255u ? v : 255u);
  }
  if (__syncthreads_or(over) && threadIdx.x == 0) atomicOr(flags, 1u);
}

// 4-bit rows: thread i packs entries 8i .. 8i+7 (two 16-byte loads) into one 32-bit word
__global__ void k_dist_u4(const uint32_t *__restrict__ d, int64_t count, uint8_t *__restrict__ out,
                          uint32_t *flags) {
  const int64_t n8 = count / 8;
  bool over = false;
  auto nib = [&](uint32_t v) -> uint32_t {
    over |= v >= 15u && v != kUnreached;
    return v < 15u ? v : 15u;
  };
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 x = __ldcs(reinterpret_cast<const uint4 *>(d) + 2 * i);
    const uint4 y = __ldcs(reinterpret_cast<const uint4 *>(d) + 2 * i + 1);
    const uint32_t a[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
    uint32_t packed = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) packed |= nib(a[k]) << (4 * k);
    reinterpret_cast<uint32_t *>(out)[i] = packed;
  }
  // tail (< 8 entries): one thread per output byte
  const int64_t b0 = 4 * n8, nb = (count + 1) / 2;
  for (int64_t b = b0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t lo = nib(d[2 * b]);
    const uint32_t hi = (2 * b + 1 < count) ? nib(d[2 * b + 1]) : 15u;
    out[b] = (uint8_t)(lo | (hi << 4));
  }
  if (__syncthreads_or(over) && threadIdx.x == 0) atomicOr(flags, 1u);
}

dawn_status dist_u4(const uint32_t *dist, int64_t count, uint8_t *out, uint32_t *flags,
                    void *stream) {
  if (count < 0 || (count > 0 && (!dist || !out || !flags)))
    return fail(DAWN_ERR_INVALID_ARGUMENT, "bad arguments");
  if ((reinterpret_cast<uintptr_t>(dist) & 15) || (reinterpret_cast<uintptr_t>(out) & 3))
    return fail(DAWN_ERR_INVALID_ARGUMENT, "dist must be 16-byte and out 4-byte aligned");
  if (count == 0) return DAWN_OK;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(nsm * 8, (count / 8 + 255) / 256));
  k_dist_u4<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(dist, count, out, flags);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "k_dist_u4 launch");
  return DAWN_OK;
}

dawn_status dist_u8(const uint32_t *dist, int64_t count, uint8_t *out, uint32_t *flags,
                    void *stream) {
  if (count < 0 || (count > 0 && (!dist || !out || !flags)))
    return fail(DAWN_ERR_INVALID_ARGUMENT, "bad arguments");
  if ((reinterpret_cast<uintptr_t>(dist) & 15) || (reinterpret_cast<uintptr_t>(out) & 3))
    return fail(DAWN_ERR_INVALID_ARGUMENT, "dist must be 16-byte and out 4-byte aligned");
  if (count == 0) return DAWN_OK;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(nsm * 8, (count / 4 + 255) / 256));
  k_dist_u8<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(dist, count, out, flags);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "k_dist_u8 launch");
  return DAWN_OK;
}

// ---------------------------------------------------------------- weighted (min,+) (NEXT-4)
WParams wparams(dawn_graph g, int lane, const uint32_t *weights, uint32_t *dist,
                dawn_sssp_stats *stats) {
  const Layout &L = g->L;
  const LaneLayout &Q = L.lane[lane];
  WParams p{};
  p.n = (uint32_t)g->n;
  p.nwords = (uint32_t)((g->n + 31) / 32);
  p.rp = at<uint32_t>(g, L.rp);
  p.col = g->col;
  p.w = weights;
  p.hout_v = at<uint32_t>(g, L.hout.v);
  p.hout_s = at<uint32_t>(g, L.hout.s);
  p.hout_e = at<uint32_t>(g, L.hout.e);
  p.hout_bits = at<uint32_t>(g, L.hout.bits);
  for (int i = 0; i < 3; ++i) p.fb[i] = at<uint32_t>(g, Q.fb[i]);
  p.ctrl = at<Ctrl>(g, Q.ctrl);
  p.dist = dist;
  p.stats = stats;
  p.delta = g->wdelta == 0 ? kWInf : g->wdelta;
  p.bad_src = &at<Ctrl>(g, L.ctrl)->bad_src;
  return p;
}

dawn_status launch_wsssp(dawn_graph g, WParams &p, int grid, cudaStream_t st) {
  if (g->m + g->n <= kOneCtaMaxNM) grid = 1;
  void *args[] = {&p};
  cudaError_t e = cudaLaunchCooperativeKernel((const void *)k_wsssp<kNT>, dim3(grid), dim3(kNT), args,
                                              0, st);
  if (e != cudaSuccess) return cuda_fail(e, "k_wsssp launch");
  return DAWN_OK;
}

dawn_status wsssp(dawn_graph g, int64_t source, const uint32_t *weights, uint32_t *dist,
                  dawn_sssp_stats *stats, void *stream) {
  if (!g || !dist || (g->m > 0 && !weights)) return fail(DAWN_ERR_INVALID_ARGUMENT, "NULL argument");
  if (source < 0 || source >= g->n)
    return fail(DAWN_ERR_BOUNDS, "source %lld not in [0, n)", (long long)source);
  dawn_status s = set_device(g);
  if (s != DAWN_OK) return s;
  WParams p = wparams(g, 0, weights, dist, stats);
  p.source = (uint32_t)source;
  return launch_wsssp(g, p, g->wsssp_grid, static_cast<cudaStream_t>(stream));
}

// k weighted searches back to back in ONE persistent launch (a grid barrier between searches).
// Batch lanes (concurrent launches on SM shares, as dawn_sssp_batch) were measured slower here:
// a (min,+) round scans the whole frontier bitmap and every heavy piece, work that grows with
// the graph rather than the frontier, so a lane's share of the SMs just takes longer (C4 weighted
// 43.3 GTEPS sequential vs 37.8 on 4 lanes).
dawn_status wsssp_batch(dawn_graph g, const uint32_t *sources, int64_t k, const uint32_t *weights,
                        uint32_t *dist, dawn_sssp_stats *stats, void *stream) {
  if (!g || k < 0 || (k > 0 && (!dist || !sources)) || (g->m > 0 && !weights))
    return fail(DAWN_ERR_INVALID_ARGUMENT, "bad arguments");
  if (k == 0) return DAWN_OK;
  if (k >= (int64_t(1) << 32)) return fail(DAWN_ERR_CAPACITY, "k too large");
  dawn_status s = set_device(g);
  if (s != DAWN_OK) return s;
  WParams p = wparams(g, 0, weights, dist, stats);
  p.sources = sources;
  p.nsrc = (uint32_t)k;
  p.vsrc = sources;
  p.vn = (uint32_t)k;
  return launch_wsssp(g, p, g->wsssp_grid, static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- partitioned SSSP (NEXT-3)
int64_t part_block(int64_t n, int32_t world) {  // Rmax: ceil(n / world) rounded up to 32
  const int64_t q = (n + world - 1) / world;
  return (q + 31) / 32 * 32;
}

dawn_status part_range(int64_t n, int32_t world, int32_t rank, int64_t *lo, int64_t *hi) {
  if (n < 1 || world < 1 || rank < 0 || rank >= world || !lo || !hi)
    return fail(DAWN_ERR_INVALID_ARGUMENT, "need n >= 1, 0 <= rank < world, lo/hi");
  const int64_t B = part_block(n, world);
  *lo = std::min<int64_t>(n, (int64_t)rank * B);
  *hi = std::min<int64_t>(n, *lo + B);
  return DAWN_OK;
}

dawn_status part_build(int64_t n, int64_t m, const int64_t *row_ptr, const int32_t *col,
                       int32_t world, int32_t rank, int64_t *m_r, int64_t *out_rp,
                       int32_t *out_col, int64_t *in_rp, int32_t *in_col, uint32_t *own_deg) {
  int64_t lo = 0, hi = 0;
  dawn_status s = part_range(n, world, rank, &lo, &hi);
  if (s != DAWN_OK) return s;
  if (m < 0 || !row_ptr || (m > 0 && !col) || !m_r)
    return fail(DAWN_ERR_INVALID_ARGUMENT, "bad arguments");
  if (row_ptr[0] != 0 || row_ptr[n] != m)
    return fail(DAWN_ERR_INVALID_GRAPH, "row_ptr[0] must be 0 and row_ptr[n] = m");
  const int64_t R = hi - lo;
  // pass 1: arcs into the owned range, per source (out-slice) and per target (in-rows)
  int64_t cnt = 0;
  for (int64_t v = 0; v < n; ++v) {
    if (row_ptr[v + 1] < row_ptr[v]) return fail(DAWN_ERR_INVALID_GRAPH, "row_ptr not monotone");
    for (int64_t j = row_ptr[v]; j < row_ptr[v + 1]; ++j) {
      const int64_t u = col[j];
      if (u < 0 || u >= n) return fail(DAWN_ERR_INVALID_GRAPH, "col[%lld] out of range", (long long)j);
      cnt += (u >= lo && u < hi);
    }
  }
  *m_r = cnt;
  if (!out_rp && !out_col && !in_rp && !in_col && !own_deg) return DAWN_OK;  // count only
  if (!out_rp || !in_rp || !own_deg || (cnt > 0 && (!out_col || !in_col)))
    return fail(DAWN_ERR_INVALID_ARGUMENT, "outputs must all be given (or all NULL to count)");
  if (cnt >= (int64_t(1) << 32)) return fail(DAWN_ERR_CAPACITY, "partition holds >= 2^32 arcs");
  // out-slice: rows in global source order, targets local (row order of the input kept)
  int64_t o = 0;
  for (int64_t v = 0; v < n; ++v) {
    out_rp[v] = o;
    for (int64_t j = row_ptr[v]; j < row_ptr[v + 1]; ++j) {
      const int64_t u = col[j];
      if (u >= lo && u < hi) out_col[o++] = (int32_t)(u - lo);
    }
  }
  out_rp[n] = o;
  // in-rows: counting sort of the same arcs by target (sources ascending within a row)
  for (int64_t t = 0; t <= R; ++t) in_rp[t] = 0;
  for (int64_t j = 0; j < cnt; ++j) in_rp[out_col[j] + 1]++;
  for (int64_t t = 0; t < R; ++t) in_rp[t + 1] += in_rp[t];
  std::vector<int64_t> cur(in_rp, in_rp + R + 1);
  for (int64_t v = 0; v < n; ++v)
    for (int64_t j = out_rp[v]; j < out_rp[v + 1]; ++j) in_col[cur[out_col[j]]++] = (int32_t)v;
  for (int64_t t = 0; t < R; ++t) {
    const int64_t d = row_ptr[lo + t + 1] - row_ptr[lo + t];
    own_deg[t] = (uint32_t)std::min<int64_t>(d, 0xffffffffll);
  }
  return DAWN_OK;
}

struct PartLayout {
  size_t rp, irp, hout_bits, hout_v, hout_s, hout_e, hin_bits, hin_v, hin_s, hin_e;
  size_t scan_tmp, piece_tmp, vis, cand, lev, send, recv, ctrl, icol2, hasin, ulist, useg, hlist;
  size_t top1, hlist2;
  size_t total;
  uint64_t capHP;
};

PartLayout part_layout(int64_t n, int64_t m_r, int32_t world, int64_t R, int64_t Rmax) {
  PartLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = align_up(o + (bytes ? bytes : 1));
    return at;
  };
  const size_t S = kPartHdr + (size_t)Rmax / 32;
  L.capHP = (uint64_t)m_r / kHPiece + (uint64_t)m_r / kHeavy + 1;
  L.rp = take(4 * (size_t)(n + 1));
  L.irp = take(4 * (size_t)(R + 1));
  L.hout_bits = take(4 * (size_t)((n + 31) / 32));
  L.hout_v = take(4 * L.capHP);
  L.hout_s = take(4 * L.capHP);
  L.hout_e = take(4 * L.capHP);
  L.hin_bits = take(4 * (size_t)((R + 31) / 32 + 1));
  L.hin_v = take(4 * L.capHP);
  L.hin_s = take(4 * L.capHP);
  L.hin_e = take(4 * L.capHP);
  L.scan_tmp = take(4 * ((size_t)std::max(n, R) / kScanBlock + 2));
  L.piece_tmp = take(4 * (3 * ((size_t)m_r / kHPiece + 3) + 1));
  L.vis = take(4 * (size_t)((R + 31) / 32 + 1));
  L.cand = take(4 * (size_t)((R + 31) / 32 + 1));
  L.icol2 = take(4 * (size_t)m_r);  // in-rows with their highest-degree sources first
  L.hasin = take(4 * (size_t)R + 4);  // owned vertices with an in-edge (the first pull's list)
  L.ulist = take(4 * (size_t)R + 4);  // unreached survivors, per-warp segments
  L.useg = take(4 * (size_t)kMaxBlocks * 32);
  L.lev = take((size_t)R + 8);
  L.send = take(4 * S);
  L.recv = take(4 * S * (size_t)world);
  L.ctrl = take(sizeof(PartCtrl));
  L.hlist = take(4 * (size_t)kPartHList);  // heavy frontier vertices of a fused push level
  L.top1 = take(4 * (size_t)R + 4);  // first entry of every degree-ordered in-row (as k_sssp)
  L.hlist2 = take(4 * (size_t)R + 4);  // fused pull: heavy vertices the light pass left
  L.total = o;
  return L;
}

}  // namespace

struct dawn_part_s {
  int64_t n = 0, m = 0, lo = 0, R = 0, Rmax = 0, m_r = 0;
  int32_t world = 1, rank = 0;
  int device = 0, nsm = 0, grid = 0;
  char *ws = nullptr;
  PartLayout L{};
  const int32_t *col = nullptr, *icol = nullptr;
  const uint32_t *deg = nullptr;
  uint32_t *dist = nullptr;
  uint32_t steps = 0, src_local = 0xffffffffu, variant = 0;
  uint32_t n_has = 0;
  float alpha = 2.f, beta = 96.f;
  int fused_grid = 0;                   // full-device cooperative grid of k_part_fused
  bool have_peers = false;
  uint32_t *peer_recv[kPartMaxW] = {};
  unsigned long long *peer_flag[kPartMaxW] = {};
};

namespace {

PartParams part_params(dawn_part p) {
  PartParams q{};
  q.n = (uint32_t)p->n;
  q.R = (uint32_t)p->R;
  q.Rmax = (uint32_t)p->Rmax;
  q.lo = (uint32_t)p->lo;
  q.world = (uint32_t)p->world;
  q.S = (uint32_t)(kPartHdr + p->Rmax / 32);
  q.nwg = (uint32_t)((p->n + 31) / 32);
  q.src_local = p->src_local;
  q.rank = (uint32_t)p->rank;
  auto u32 = [&](size_t off) { return reinterpret_cast<uint32_t *>(p->ws + off); };
  q.rp = u32(p->L.rp);
  q.col = p->col;
  q.irp = u32(p->L.irp);
  q.icol = p->icol;
  q.deg = p->deg;
  q.hout_v = u32(p->L.hout_v);
  q.hout_s = u32(p->L.hout_s);
  q.hout_e = u32(p->L.hout_e);
  q.hout_bits = u32(p->L.hout_bits);
  q.hin_v = u32(p->L.hin_v);
  q.hin_s = u32(p->L.hin_s);
  q.hin_e = u32(p->L.hin_e);
  q.hin_bits = u32(p->L.hin_bits);
  q.vis = u32(p->L.vis);
  q.cand = u32(p->L.cand);
  q.hasin = u32(p->L.hasin);
  q.ulist = u32(p->L.ulist);
  q.useg = u32(p->L.useg);
  q.hlist = u32(p->L.hlist);
  q.hlist2 = u32(p->L.hlist2);
  q.top1 = (DAWN_PULL_TOP1 && p->m_r > 0) ? u32(p->L.top1) : nullptr;
  q.n_has = p->n_has;
  q.lev = reinterpret_cast<uint8_t *>(p->ws + p->L.lev);
  q.dist = p->dist;
  q.recv = u32(p->L.recv);
  q.send = u32(p->L.send);
  q.ctrl = reinterpret_cast<PartCtrl *>(p->ws + p->L.ctrl);
  q.variant = p->variant;
  q.can_pull = 1;
  q.alpha = p->alpha;
  q.beta = p->beta;
  q.m_total = (unsigned long long)p->m;
  return q;
}

dawn_status part_load(int64_t n, int64_t m, int32_t world, int32_t rank, int64_t m_r,
                      const int64_t *out_rp, const int32_t *out_col, const int64_t *in_rp,
                      const int32_t *in_col, const uint32_t *own_deg, void *workspace,
                      size_t ws_bytes, void *stream, dawn_part *out) {
  if (!out) return fail(DAWN_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  int64_t lo = 0, hi = 0;
  dawn_status s = part_range(n, world, rank, &lo, &hi);
  if (s != DAWN_OK) return s;
  if (n >= (int64_t(1) << 31) || m < 0 || m >= (int64_t(1) << 32) || m_r < 0 || m_r > m)
    return fail(DAWN_ERR_CAPACITY, "n < 2^31 and m_r <= m < 2^32 required");
  const int64_t R = hi - lo;
  if (!out_rp || !in_rp || (R > 0 && !own_deg) || (m_r > 0 && (!out_col || !in_col)) || !workspace)
    return fail(DAWN_ERR_INVALID_ARGUMENT, "NULL array");
  if (reinterpret_cast<uintptr_t>(workspace) & 255)
    return fail(DAWN_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  const int64_t Rmax = part_block(n, world);
  PartLayout L = part_layout(n, m_r, world, R, Rmax);
  if (ws_bytes < L.total)
    return fail(DAWN_ERR_WORKSPACE, "workspace too small: need %zu bytes, got %zu", L.total, ws_bytes);
  cudaPointerAttributes pa{};
  cudaError_t e = cudaPointerGetAttributes(&pa, workspace);
  if (e != cudaSuccess) return cuda_fail(e, "cudaPointerGetAttributes(workspace)");
  if (pa.type != cudaMemoryTypeDevice) return fail(DAWN_ERR_INVALID_ARGUMENT, "workspace is not device memory");
  if ((e = cudaSetDevice(pa.device)) != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  auto *p = new (std::nothrow) dawn_part_s;
  if (!p) return fail(DAWN_ERR_CAPACITY, "host allocation failed");
  p->n = n;
  p->m = m;
  p->lo = lo;
  p->R = R;
  p->Rmax = Rmax;
  p->m_r = m_r;
  p->world = world;
  p->rank = rank;
  p->device = pa.device;
  p->ws = static_cast<char *>(workspace);
  p->L = L;
  p->col = out_col;
  p->icol = m_r ? reinterpret_cast<int32_t *>(p->ws + L.icol2) : in_col;
  p->deg = own_deg;
  cudaDeviceGetAttribute(&p->nsm, cudaDevAttrMultiProcessorCount, pa.device);
  int bps = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_part_level<kNT>, kNT, 0);
  p->grid = std::max(1, p->nsm * std::max(1, std::min(bps, 2)));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int blocks = std::max(1, std::min<int>(p->nsm * 8, (int)((n + 255) / 256)));
  auto u32 = [&](size_t off) { return reinterpret_cast<uint32_t *>(p->ws + off); };
  k_offsets32<<<blocks, 256, 0, st>>>(out_rp, u32(L.rp), n + 1);
  k_offsets32<<<blocks, 256, 0, st>>>(in_rp, u32(L.irp), R + 1);
  PartCtrl *C = reinterpret_cast<PartCtrl *>(p->ws + L.ctrl);
  cudaMemsetAsync(C, 0, sizeof(PartCtrl), st);
  cudaMemsetAsync(p->ws + L.cand, 0, 4 * (size_t)((R + 31) / 32 + 1), st);
  {
    int fb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fb, k_part_fused<kNT>, kNT, 0);
    p->fused_grid = std::max(1, p->nsm * std::max(1, std::min(fb, 2)));
  }
  // static heavy pieces of the out-slice rows (over n sources) and of the in-rows (over R)
  auto build_list = [&](const uint32_t *rows, uint32_t nrows, size_t bits, size_t hv, size_t hs,
                        size_t he, uint32_t *count) {
    const uint32_t nblk = (uint32_t)((nrows + kScanBlock - 1) / kScanBlock);
    if (nrows == 0 || m_r == 0) {
      cudaMemsetAsync(p->ws + bits, 0, 4 * (size_t)((nrows + 31) / 32 + 1), st);
      cudaMemsetAsync(count, 0, 4, st);
      return;
    }
    k_hcount<<<nblk, 256, 0, st>>>(rows, nrows, u32(bits), u32(L.scan_tmp));
    k_hscan<<<1, 32, 0, st>>>(u32(L.scan_tmp), nblk, count);
    const size_t cap = (size_t)m_r / kHPiece + 3;
    uint32_t *hc = u32(L.piece_tmp), *base = hc + cap, *cursor = base + cap, *maxc = cursor + cap;
    cudaMemsetAsync(hc, 0, 4 * cap, st);
    cudaMemsetAsync(maxc, 0, 4, st);
    const int hb = std::max(1, std::min<int>(p->nsm * 8, (int)((nrows + 255) / 256)));
    k_hhist<<<hb, 256, 0, st>>>(rows, nrows, hc, maxc);
    k_hbase<<<1, 32, 0, st>>>(hc, base, cursor, maxc);
    k_hfill<<<hb, 256, 0, st>>>(rows, nrows, base, cursor, u32(hv), u32(hs), u32(he));
  };
  // pull probes meet hubs first: each in-row with its 8 sources of largest out-slice degree (a
  // proxy of the global out-degree: labels are random, so a vertex sends ~1/W of its arcs
  // to every range) moved to the front, as k_sssp's degree-ordered in-rows
  if (m_r > 0 && R > 0) {
    k_topk_rows<<<p->nsm * 8, 256, 0, st>>>(u32(L.irp), in_col, u32(L.rp), (uint32_t)R,
                                            reinterpret_cast<int32_t *>(p->ws + L.icol2));
    k_top1<<<p->nsm * 8, 256, 0, st>>>(u32(L.irp), reinterpret_cast<int32_t *>(p->ws + L.icol2),
                                       (uint32_t)R, u32(L.top1));
  }
  if (R > 0) {  // static ascending list of the owned vertices with an in-edge
    const uint32_t nblk = (uint32_t)((R + kScanBlock - 1) / kScanBlock);
    k_lcount<<<nblk, 256, 0, st>>>(u32(L.irp), (uint32_t)R, u32(L.scan_tmp));
    k_hscan<<<1, 32, 0, st>>>(u32(L.scan_tmp), nblk, u32(L.useg));  // total -> useg[0]
    k_lfill<<<nblk, 256, 0, st>>>(u32(L.irp), (uint32_t)R, u32(L.scan_tmp), u32(L.hasin));
    cudaMemcpyAsync(&p->n_has, u32(L.useg), 4, cudaMemcpyDeviceToHost, st);
  }
  build_list(u32(L.rp), (uint32_t)n, L.hout_bits, L.hout_v, L.hout_s, L.hout_e, &C->n_hp[0]);
  build_list(u32(L.irp), (uint32_t)R, L.hin_bits, L.hin_v, L.hin_s, L.hin_e, &C->n_hp[1]);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) {
    delete p;
    return cuda_fail(e, "dawn_part_load");
  }
  *out = p;
  return DAWN_OK;
}

dawn_status part_exchange(dawn_part p, uint32_t **send, uint32_t **recv, int64_t *slice_words) {
  if (!p || !send || !recv || !slice_words) return fail(DAWN_ERR_INVALID_ARGUMENT, "NULL argument");
  *send = reinterpret_cast<uint32_t *>(p->ws + p->L.send);
  *recv = reinterpret_cast<uint32_t *>(p->ws + p->L.recv);
  *slice_words = (int64_t)(kPartHdr + p->Rmax / 32);
  return DAWN_OK;
}

dawn_status part_begin(dawn_part p, int64_t source, uint32_t variant, uint32_t *dist, void *stream) {
  if (!p || (p->R > 0 && !dist)) return fail(DAWN_ERR_INVALID_ARGUMENT, "part or dist is NULL");
  if (variant > DAWN_PULL) return fail(DAWN_ERR_INVALID_ARGUMENT, "unknown variant");
  if (source < 0 || source >= p->n)
    return fail(DAWN_ERR_BOUNDS, "source %lld not in [0, n)", (long long)source);
  cudaError_t e = cudaSetDevice(p->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  p->dist = dist;
  p->variant = variant;
  p->steps = 0;
  p->src_local = (source >= p->lo && source < p->lo + p->R) ? (uint32_t)(source - p->lo) : 0xffffffffu;
  PartParams q = part_params(p);
  e = cudaMemsetAsync(q.send, 0, 4 * (size_t)q.S, st);
  if (e != cudaSuccess) return cuda_fail(e, "dawn_part_begin");
  const int blocks = std::max(1, std::min<int>(p->nsm * 4, (int)((p->R / 32 + 255) / 256)));
  k_part_begin<<<blocks, 256, 0, st>>>(q);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_part_begin launch");
  return DAWN_OK;
}

dawn_status part_step(dawn_part p, void *stream) {
  if (!p) return fail(DAWN_ERR_INVALID_ARGUMENT, "part is NULL");
  cudaError_t e = cudaSetDevice(p->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PartParams q = part_params(p);
  // the slice of F_{L+1} is built from zero (the previous one was already gathered)
  if ((e = cudaMemsetAsync(q.send, 0, 4 * (size_t)q.S, st)) != cudaSuccess) return cuda_fail(e, "dawn_part_step");
  k_part_level<kNT><<<p->grid, kNT, 0, st>>>(q, p->steps);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_part_level launch");
  p->steps++;
  return DAWN_OK;
}

dawn_status part_done(dawn_part p, int32_t *done, void *stream) {
  if (!p || !done) return fail(DAWN_ERR_INVALID_ARGUMENT, "NULL argument");
  cudaError_t e = cudaSetDevice(p->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PartCtrl *C = reinterpret_cast<PartCtrl *>(p->ws + p->L.ctrl);
  uint32_t d = 0;
  e = cudaMemcpyAsync(&d, &C->st[p->steps & 1].done, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "dawn_part_done");
  *done = (int32_t)d;
  return DAWN_OK;
}

dawn_status part_fused_peers(dawn_part p, int32_t world, void *const *peer_recv,
                             void *const *peer_flag) {
  if (!p || !peer_recv || !peer_flag) return fail(DAWN_ERR_INVALID_ARGUMENT, "NULL argument");
  if (world != p->world || world > kPartMaxW)
    return fail(DAWN_ERR_INVALID_ARGUMENT, "world must equal the partition's (<= %d)", kPartMaxW);
  cudaError_t e = cudaSetDevice(p->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  for (int q = 0; q < world; ++q) {
    if (!peer_recv[q] || !peer_flag[q]) return fail(DAWN_ERR_INVALID_ARGUMENT, "NULL peer pointer");
    // a buffer on another device (a CUDA-IPC mapping of a peer's buffer) needs peer access
    cudaPointerAttributes pa{};
    if ((e = cudaPointerGetAttributes(&pa, peer_recv[q])) != cudaSuccess)
      return cuda_fail(e, "cudaPointerGetAttributes(peer buffer)");
    if (pa.type == cudaMemoryTypeDevice && pa.device != p->device) {
      int can = 0;
      cudaDeviceCanAccessPeer(&can, p->device, pa.device);
      if (!can) return fail(DAWN_ERR_CONFIG, "device %d cannot access peer device %d", p->device, pa.device);
      e = cudaDeviceEnablePeerAccess(pa.device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        return cuda_fail(e, "cudaDeviceEnablePeerAccess");
      }
    }
    p->peer_recv[q] = static_cast<uint32_t *>(peer_recv[q]);
    p->peer_flag[q] = static_cast<unsigned long long *>(peer_flag[q]);
  }
  p->have_peers = true;
  return DAWN_OK;
}

dawn_status part_fused_sssp(dawn_part p, int64_t source, uint32_t variant, uint32_t *dist,
                            dawn_sssp_stats *stats, int32_t grid, void *stream) {
  if (!p || (p->R > 0 && !dist)) return fail(DAWN_ERR_INVALID_ARGUMENT, "part or dist is NULL");
  if (!p->have_peers) return fail(DAWN_ERR_CONFIG, "dawn_part_fused_peers was not called");
  if (variant > DAWN_PULL) return fail(DAWN_ERR_INVALID_ARGUMENT, "unknown variant");
  if (source < 0 || source >= p->n)
    return fail(DAWN_ERR_BOUNDS, "source %lld not in [0, n)", (long long)source);
  if (grid < 0 || grid > p->fused_grid)
    return fail(DAWN_ERR_INVALID_ARGUMENT, "grid must be in [0, %d]", p->fused_grid);
  cudaError_t e = cudaSetDevice(p->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  p->dist = dist;
  p->variant = variant;
  p->src_local = (source >= p->lo && source < p->lo + p->R) ? (uint32_t)(source - p->lo) : 0xffffffffu;
  PartParams q = part_params(p);
  PartPeers peers{};
  for (int r = 0; r < p->world; ++r) {
    peers.recv[r] = p->peer_recv[r];
    peers.flag[r] = p->peer_flag[r];
  }
  void *args[] = {&q, &peers, &stats};
  e = cudaLaunchCooperativeKernel((const void *)k_part_fused<kNT>, dim3(grid ? grid : p->fused_grid),
                                  dim3(kNT), args, 0, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "k_part_fused launch");
  return DAWN_OK;
}

dawn_status part_finish(dawn_part p, dawn_sssp_stats *stats, void *stream) {
  if (!p) return fail(DAWN_ERR_INVALID_ARGUMENT, "part is NULL");
  cudaError_t e = cudaSetDevice(p->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PartParams q = part_params(p);
  const int blocks = std::max(1, std::min<int>(p->nsm * 8, (int)((p->R + 255) / 256)));
  k_part_finish<<<blocks, 256, 0, st>>>(q, p->steps & 1, stats);
  if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "k_part_finish launch");
  return DAWN_OK;
}

}  // namespace

extern "C" {

const char *dawn_last_error(void) { return g_err; }
const char *dawn_version(void) { return "dawn-b200 0.4 sm_100a"; }

size_t dawn_workspace_bytes(int64_t n, int64_t m, uint32_t flags) {
  try {
    if (n < 1 || n >= (int64_t(1) << 31) || m < 0 || m >= (int64_t(1) << 32)) return 0;
    return make_layout(n, m, flags).total;
  } catch (...) {
    return 0;
  }
}

dawn_status dawn_graph_load_csr(int64_t n, int64_t m, const int64_t *row_ptr, const int32_t *col,
                                const int64_t *in_row_ptr, const int32_t *in_col, uint32_t flags,
                                void *workspace, size_t ws_bytes, void *stream, dawn_graph *out) {
  DAWN_GUARD(return load_csr(n, m, row_ptr, col, in_row_ptr, in_col, flags, workspace, ws_bytes,
                             stream, out);)
}

dawn_status dawn_graph_destroy(dawn_graph g) {
  delete g;
  return DAWN_OK;
}

dawn_status dawn_graph_get_param(dawn_graph g, dawn_param key, double *value) {
  DAWN_GUARD(
    if (!g || !value) return fail(DAWN_ERR_INVALID_ARGUMENT, "graph or value is NULL");
    switch (key) {
      case DAWN_PARAM_ALPHA: *value = g->alpha; break;
      case DAWN_PARAM_BETA: *value = g->beta; break;
      case DAWN_PARAM_MS_ALPHA: *value = g->ms_alpha; break;
      case DAWN_PARAM_BITMAP_PUSH_EDGES: *value = g->bmpush_e; break;
      case DAWN_PARAM_SOLO_EDGES: *value = g->solo_e; break;
      case DAWN_PARAM_CLUSTER_START: *value = g->cluster_start; break;
      case DAWN_PARAM_CLUSTER_HANDOVER_EDGES: *value = (double)g->handover_m; break;
      case DAWN_PARAM_BITMAP_PUSH_GROW_EDGES: *value = g->bmpush_grow; break;
      case DAWN_PARAM_NARROW_QUEUE_CAP: *value = g->narrow_qcap; break;
      case DAWN_PARAM_BATCH_LANES: *value = g->lanes; break;
      case DAWN_PARAM_DENSE_MAX_ENTRIES: *value = g->dense_max; break;
      case DAWN_PARAM_MS_LANES: *value = g->ms_lanes; break;
      case DAWN_PARAM_WEIGHT_DELTA: *value = g->wdelta; break;
      case DAWN_PARAM_BATCH_DYNAMIC: *value = g->batch_claim ? 1.0 : 0.0; break;
      default: return fail(DAWN_ERR_INVALID_ARGUMENT, "unknown parameter");
    }
    return DAWN_OK;)
}

dawn_status dawn_graph_set_param(dawn_graph g, dawn_param key, double value) {
  DAWN_GUARD(return set_param(g, key, value);)
}

dawn_status dawn_sssp(dawn_graph g, int64_t source, uint32_t variant, uint32_t *dist,
                      dawn_sssp_stats *stats, void *stream) {
  DAWN_GUARD(return sssp_one(g, source, variant, dist, stats, stream);)
}

dawn_status dawn_sssp_batch(dawn_graph g, const uint32_t *sources, int64_t k, uint32_t variant,
                            uint32_t *dist, dawn_sssp_stats *stats, void *stream) {
  DAWN_GUARD(return sssp_batch(g, sources, k, variant, dist, stats, stream);)
}

dawn_status dawn_graph_check(dawn_graph g, void *stream) {
  DAWN_GUARD(return graph_check(g, stream);)
}

dawn_status dawn_msssp(dawn_graph g, const int64_t *sources, int64_t k, uint32_t *dist,
                       dawn_record *rec, void *stream) {
  DAWN_GUARD(return msssp(g, sources, k, dist, rec, stream);)
}

dawn_status dawn_graph_trace(dawn_graph g, dawn_trace_rec *host_out, int64_t cap, int64_t *count,
                             void *stream) {
  DAWN_GUARD(return graph_trace(g, host_out, cap, count, stream);)
}

dawn_status dawn_apsp_shard(int64_t k, int32_t rank, int32_t world, int64_t *idx, int64_t cap,
                            int64_t *count) {
  DAWN_GUARD(return apsp_shard(k, rank, world, idx, cap, count);)
}

dawn_status dawn_apsp(dawn_graph g, const int64_t *sources, int64_t k, int32_t rank, int32_t world,
                      dawn_record *rec, int64_t cap, int64_t *n_written, void *stream) {
  DAWN_GUARD(return apsp(g, sources, k, rank, world, rec, cap, n_written, stream);)
}

dawn_status dawn_apsp_rows(dawn_graph g, const int64_t *sources, int64_t k, int64_t chunk,
                           uint32_t *dev_stage, uint32_t *host_stage, dawn_row_sink sink,
                           void *user, void *stream) {
  DAWN_GUARD(return apsp_rows(g, sources, k, chunk, dev_stage, host_stage, sink, user, stream);)
}

dawn_status dawn_largest_wcc(dawn_graph g, int64_t *sources_out, int64_t *k, uint64_t *arcs,
                             void *stream) {
  DAWN_GUARD(return largest_wcc(g, sources_out, k, arcs, stream);)
}

dawn_status dawn_graph_ms_counters(dawn_graph g, uint64_t *host_out, void *stream) {
  DAWN_GUARD(return ms_counters(g, host_out, stream);)
}

dawn_status dawn_dist_u8(const uint32_t *dist, int64_t count, uint8_t *out, uint32_t *flags,
                         void *stream) {
  DAWN_GUARD(return dist_u8(dist, count, out, flags, stream);)
}

dawn_status dawn_dist_u4(const uint32_t *dist, int64_t count, uint8_t *out, uint32_t *flags,
                         void *stream) {
  DAWN_GUARD(return dist_u4(dist, count, out, flags, stream);)
}

dawn_status dawn_wsssp(dawn_graph g, int64_t source, const uint32_t *weights, uint32_t *dist,
                       dawn_sssp_stats *stats, void *stream) {
  DAWN_GUARD(return wsssp(g, source, weights, dist, stats, stream);)
}

dawn_status dawn_wsssp_batch(dawn_graph g, const uint32_t *sources, int64_t k,
                             const uint32_t *weights, uint32_t *dist, dawn_sssp_stats *stats,
                             void *stream) {
  DAWN_GUARD(return wsssp_batch(g, sources, k, weights, dist, stats, stream);)
}

dawn_status dawn_part_range(int64_t n, int32_t world, int32_t rank, int64_t *lo, int64_t *hi) {
  DAWN_GUARD(return part_range(n, world, rank, lo, hi);)
}

dawn_status dawn_part_build(int64_t n, int64_t m, const int64_t *row_ptr, const int32_t *col,
                            int32_t world, int32_t rank, int64_t *m_r, int64_t *out_rp,
                            int32_t *out_col, int64_t *in_rp, int32_t *in_col, uint32_t *own_deg) {
  DAWN_GUARD(return part_build(n, m, row_ptr, col, world, rank, m_r, out_rp, out_col, in_rp, in_col,
                               own_deg);)
}

size_t dawn_part_workspace_bytes(int64_t n, int64_t m_r, int32_t world, int32_t rank) {
  try {
    int64_t lo = 0, hi = 0;
    if (n < 1 || n >= (int64_t(1) << 31) || m_r < 0 || m_r >= (int64_t(1) << 32) ||
        part_range(n, world, rank, &lo, &hi) != DAWN_OK)
      return 0;
    return part_layout(n, m_r, world, hi - lo, part_block(n, world)).total;
  } catch (...) {
    return 0;
  }
}

dawn_status dawn_part_load(int64_t n, int64_t m, int32_t world, int32_t rank, int64_t m_r,
                           const int64_t *out_rp, const int32_t *out_col, const int64_t *in_rp,
                           const int32_t *in_col, const uint32_t *own_deg, void *workspace,
                           size_t ws_bytes, void *stream, dawn_part *out) {
  DAWN_GUARD(return part_load(n, m, world, rank, m_r, out_rp, out_col, in_rp, in_col, own_deg,
                              workspace, ws_bytes, stream, out);)
}

dawn_status dawn_part_destroy(dawn_part p) {
  delete p;
  return DAWN_OK;
}

dawn_status dawn_part_exchange(dawn_part p, uint32_t **send, uint32_t **recv, int64_t *slice_words) {
  DAWN_GUARD(return part_exchange(p, send, recv, slice_words);)
}

dawn_status dawn_part_begin(dawn_part p, int64_t source, uint32_t variant, uint32_t *dist_own,
                            void *stream) {
  DAWN_GUARD(return part_begin(p, source, variant, dist_own, stream);)
}

dawn_status dawn_part_step(dawn_part p, void *stream) { DAWN_GUARD(return part_step(p, stream);) }

dawn_status dawn_part_done(dawn_part p, int32_t *done, void *stream) {
  DAWN_GUARD(return part_done(p, done, stream);)
}

dawn_status dawn_part_fused_peers(dawn_part p, int32_t world, void *const *peer_recv,
                                  void *const *peer_flag) {
  DAWN_GUARD(return part_fused_peers(p, world, peer_recv, peer_flag);)
}

dawn_status dawn_part_fused_sssp(dawn_part p, int64_t source, uint32_t variant, uint32_t *dist_own,
                                 dawn_sssp_stats *stats, int32_t grid, void *stream) {
  DAWN_GUARD(return part_fused_sssp(p, source, variant, dist_own, stats, grid, stream);)
}

dawn_status dawn_part_finish(dawn_part p, dawn_sssp_stats *stats, void *stream) {
  DAWN_GUARD(return part_finish(p, stats, stream);)
}

}  // extern "C"

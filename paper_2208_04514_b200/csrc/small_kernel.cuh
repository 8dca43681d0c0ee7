// small_kernel.cuh — single-CTA DAWN for graphs whose CSR fits in shared memory (SURVEY §2.5
// M8; BASELINE configs[0]: ER n = 1000, m = 8000).  The whole SSSP — CSR, distances, visited
// bitmap and both frontier queues — lives in shared memory, so a level costs one pass over the
// frontier plus one __syncthreads instead of a grid barrier and DRAM round trips.  Each level
// is the SOVM step (Algorithm 2): frontier rows are expanded, a target is
// claimed by a shared-memory atomic test-and-set on the visited bitmap (A2 line 6 filter,
// reading Q1), gets distance L+1 and joins the next queue.
#pragma once
#include "layout.h"

namespace dawn {

struct SmallParams {
  uint32_t n, m;
  const uint32_t *rp;
  const int32_t *col;
  uint32_t *dist;             // [nsrc or 1][n]
  dawn_sssp_stats *stats;     // [nsrc or 1] or NULL
  uint32_t source;
  const uint32_t *sources;    // batch mode (dawn_sssp_batch): nsrc device source ids
  uint32_t nsrc;
  uint32_t *bad_src;          // sticky flag: a batch source id was >= n (nothing written)
};

// Shared-memory bytes k_small needs for (n, m).
inline size_t small_smem_bytes(int64_t n, int64_t m) {
  return 4 * (size_t)(n + 1) + 4 * (size_t)m + 4 * (size_t)n + 8 * (size_t)n +
         4 * (size_t)((n + 31) / 32) + 64;
}

template <int NT>
__global__ void __launch_bounds__(NT) k_small(SmallParams p) {
  extern __shared__ uint32_t sm[];
  const uint32_t n = p.n, m = p.m, nw = (n + 31) / 32;
  uint32_t *rp = sm;              // n + 1
  uint32_t *col = rp + n + 1;     // m
  uint32_t *dist = col + m;       // n
  uint32_t *qa = dist + n;        // n
  uint32_t *qb = qa + n;          // n
  uint32_t *vis = qb + n;         // nw
  __shared__ uint32_t nq_cnt[3];  // level L appends to nq_cnt[L % 3]
  __shared__ unsigned long long m_acc;
  const uint32_t tid = threadIdx.x, lane = lane_id();
  if (p.nsrc) {  // the whole device source list is checked before anything is written
    bool bad = false;
    for (uint32_t i = tid; i < p.nsrc; i += NT) bad |= ld_nc(p.sources + i) >= n;
    if (__syncthreads_or(bad)) {
      if (blockIdx.x == 0 && tid == 0) atomicOr(p.bad_src, 1u);
      return;
    }
  }
  // CSR -> shared memory, 4 independent loads in flight per thread
  {
    constexpr int U = 4;
    for (uint32_t i0 = tid; i0 <= n; i0 += NT * U) {
      uint32_t v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = (i0 + u * NT <= n) ? ld_nc(p.rp + i0 + u * NT) : 0u;
#pragma unroll
      for (int u = 0; u < U; ++u) if (i0 + u * NT <= n) rp[i0 + u * NT] = v[u];
    }
    for (uint32_t i0 = tid; i0 < m; i0 += NT * U) {
      uint32_t v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = (i0 + u * NT < m) ? (uint32_t)ld_nc(p.col + i0 + u * NT) : 0u;
#pragma unroll
      for (int u = 0; u < U; ++u) if (i0 + u * NT < m) col[i0 + u * NT] = v[u];
    }
  }
  // the CSR stays in shared memory for every search of a batch; batch searches are independent,
  // so CTA b takes searches b, b + gridDim.x, ...
  const uint32_t nsrc = p.nsrc ? p.nsrc : 1u;
  for (uint32_t si = blockIdx.x; si < nsrc; si += gridDim.x) {
  for (uint32_t i = tid; i < n; i += NT) dist[i] = kUnreached;
  for (uint32_t i = tid; i < nw; i += NT) vis[i] = 0;
  __syncthreads();
  const uint32_t s = p.nsrc ? p.sources[si] : p.source;
  if (tid == 0) {
    dist[s] = 0;
    vis[s >> 5] = 1u << (s & 31);
    qa[0] = s;
    m_acc = rp[s + 1] - rp[s];
    nq_cnt[0] = nq_cnt[1] = nq_cnt[2] = 0;
  }
  uint32_t nq = 1, L = 0, reached = 0, levels = 0, ecc = 0;
  uint32_t *cur = qa, *nxt = qb;
  __syncthreads();
  // kLpv lanes per frontier vertex (4 vertices per warp round), one arc per lane per step
  constexpr uint32_t kLpv = 8;
  for (;;) {
    uint32_t *cnt = &nq_cnt[L % 3];
    if (tid == 0) nq_cnt[(L + 1) % 3] = 0;  // last read two barriers ago
    uint32_t my_m = 0;
    for (uint32_t base = (tid / 32) * (32 / kLpv); base < nq; base += (NT / 32) * (32 / kLpv)) {
      const uint32_t i = base + lane / kLpv;
      const uint32_t v = i < nq ? cur[i] : 0u;
      const uint32_t e0 = i < nq ? rp[v] : 0u, e1 = i < nq ? rp[v + 1] : 0u;
      for (uint32_t e = e0 + lane % kLpv; __any_sync(DAWN_FULL, e < e1); e += kLpv) {
        bool put = false;
        uint32_t u = 0;
        if (e < e1) {
          u = col[e];
          const uint32_t bit = 1u << (u & 31);
          if (!(vis[u >> 5] & bit)) put = !(atomicOr(&vis[u >> 5], bit) & bit);
        }
        const uint32_t b = __ballot_sync(DAWN_FULL, put);
        if (b) {
          uint32_t base2 = 0;
          if (lane == 0) base2 = atomicAdd(cnt, (uint32_t)__popc(b));
          base2 = __shfl_sync(DAWN_FULL, base2, 0);
          if (put) {
            dist[u] = L + 1;
            nxt[base2 + __popc(b & lanemask_lt())] = u;
            my_m += rp[u + 1] - rp[u];
          }
        }
      }
    }
    my_m = __reduce_add_sync(DAWN_FULL, my_m);
    if (lane == 0 && my_m) atomicAdd(&m_acc, (unsigned long long)my_m);
    __syncthreads();
    ++levels;
    const uint32_t k = *cnt;
    if (k == 0) break;
    reached += k;
    ecc = L + 1;
    nq = k;
    uint32_t *t = cur;
    cur = nxt;
    nxt = t;
    ++L;
  }
  uint32_t *drow = p.dist + (size_t)si * n;
  for (uint32_t i = tid; i < n; i += NT) drow[i] = dist[i];
  if (p.stats && tid == 0) {
    dawn_sssp_stats st;
    st.levels = ecc;
    st.reached = reached;
    st.edges_reach = m_acc;
    st.edges_examined = m_acc;
    st.push_levels = levels;
    st.pull_levels = 0;
    p.stats[si] = st;
  }
  __syncthreads();  // the next search re-initialises dist / vis / counters
  }  // sources
}

}  // namespace dawn

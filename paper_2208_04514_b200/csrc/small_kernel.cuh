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
  uint32_t *dist;
  dawn_sssp_stats *stats;
  uint32_t source;
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
  __shared__ uint32_t nq_next;
  __shared__ unsigned long long m_acc;
  const uint32_t tid = threadIdx.x;
  for (uint32_t i = tid; i <= n; i += NT) rp[i] = ld_nc(p.rp + i);
  for (uint32_t i = tid; i < m; i += NT) col[i] = (uint32_t)ld_nc(p.col + i);
  for (uint32_t i = tid; i < n; i += NT) dist[i] = kUnreached;
  for (uint32_t i = tid; i < nw; i += NT) vis[i] = 0;
  __syncthreads();
  const uint32_t s = p.source;
  if (tid == 0) {
    dist[s] = 0;
    vis[s >> 5] = 1u << (s & 31);
    qa[0] = s;
    m_acc = rp[s + 1] - rp[s];
  }
  uint32_t nq = 1, L = 0, reached = 0, levels = 0, ecc = 0;
  uint32_t *cur = qa, *nxt = qb;
  __syncthreads();
  for (;;) {
    if (tid == 0) nq_next = 0;
    __syncthreads();
    unsigned long long my_m = 0;
    // thread per frontier vertex (rows are short at this size; no hub splitting needed)
    for (uint32_t i = tid; i < nq; i += NT) {
      const uint32_t v = cur[i];
      for (uint32_t e = rp[v]; e < rp[v + 1]; ++e) {
        const uint32_t u = col[e];
        const uint32_t bit = 1u << (u & 31);
        if (vis[u >> 5] & bit) continue;
        if (atomicOr(&vis[u >> 5], bit) & bit) continue;
        dist[u] = L + 1;
        nxt[atomicAdd(&nq_next, 1u)] = u;
        my_m += rp[u + 1] - rp[u];
      }
    }
    my_m = warp_sum(my_m);
    if (lane_id() == 0 && my_m) atomicAdd(&m_acc, my_m);
    __syncthreads();
    ++levels;
    const uint32_t k = nq_next;
    if (k == 0) break;
    reached += k;
    ecc = L + 1;
    nq = k;
    uint32_t *t = cur;
    cur = nxt;
    nxt = t;
    ++L;
    __syncthreads();
  }
  for (uint32_t i = tid; i < n; i += NT) p.dist[i] = dist[i];
  if (p.stats && tid == 0) {
    dawn_sssp_stats st;
    st.levels = ecc;
    st.reached = reached;
    st.edges_reach = m_acc;
    st.edges_examined = m_acc;
    st.push_levels = levels;
    st.pull_levels = 0;
    *p.stats = st;
  }
}

}  // namespace dawn

// ms64_kernel.cuh — bit-parallel multi-source DAWN (BASELINE.json north_star: "packs 64
// sources per vertex word so one adjacency pass serves 64 BFS trees").
//
// Vertex words (uint64): seen[v] (bit k: source k has reached v), F[v] (bit k: v is in source
// k's level-L frontier), nxt[v] (push scratch).  One level generalises Eq. 9 (PAPER.md
// L260-264) to 64 right-hand sides over the (OR, AND) semiring:
//   PUSH  for v with F[v] != 0, for u in N+(v): nxt[u] |= F[v] & ~seen[u]          (SOVM)
//         then per vertex: new = nxt & ~seen; seen |= new; F' = new
//   PULL  for u with U = ~seen[u] & active != 0: acc = OR of F[v] over N-(u), stopping as soon
//         as acc covers U (Eq. 4 early exit per bit set); new = acc & U              (BOVM)
// Per-source records (ecc, reached, sum_dist, hash) are accumulated without per-event atomics:
// a warp's 32 new-words are bit-transposed with 64 ballots so lane j owns sources j, j+32.
#pragma once
#include "layout.h"

namespace dawn {

struct MsParams {
  uint32_t n, nwords;
  unsigned long long m;
  const uint32_t *rp, *irp;
  const int32_t *col, *icol;
  unsigned long long *seen, *F[2], *nxt;
  MsCtrl *ctrl;
  const uint32_t *sources;   // device, this launch's source list
  uint32_t count;            // number of sources in the list (batches of 64)
  dawn_record *rec;          // device [count] or null
  uint32_t *dist;            // device [count][n] or null
  uint32_t can_pull, sym;
  float ms_alpha;
  uint4 *part;               // per-CTA partial records [gridDim.x][64]: cnt, ecc, sum, hash
};

struct MsState {
  uint32_t L, dir, cur, stop;
  unsigned long long n_active, m_active;
};

__device__ __forceinline__ void ms_record_group(const MsParams &p, unsigned long long nw,
                                                uint32_t u, uint32_t L1, uint32_t batch_base,
                                                unsigned long long *hs, uint32_t &cnt0,
                                                uint32_t &cnt1, uint32_t &ecc0, uint32_t &ecc1,
                                                unsigned long long &h0,
                                                unsigned long long &h1) {
  // nw: this lane's vertex u new-bits (0 if none).  Warp-collective.
  if (!__any_sync(DAWN_FULL, nw != 0)) return;
  const uint32_t lane = lane_id();
  hs[lane] = nw ? rec_hash(u, L1) : 0ull;
  __syncwarp();
  uint32_t m0 = 0, m1 = 0;
#pragma unroll 8
  for (int k = 0; k < 32; ++k) {
    const uint32_t b0 = __ballot_sync(DAWN_FULL, (nw >> k) & 1ull);
    const uint32_t b1 = __ballot_sync(DAWN_FULL, (nw >> (k + 32)) & 1ull);
    if (lane == (uint32_t)k) { m0 = b0; m1 = b1; }
  }
  if (m0) { cnt0 += __popc(m0); ecc0 = L1; }
  if (m1) { cnt1 += __popc(m1); ecc1 = L1; }
  while (m0) { h0 += hs[__ffs(m0) - 1]; m0 &= m0 - 1; }
  while (m1) { h1 += hs[__ffs(m1) - 1]; m1 &= m1 - 1; }
  if (p.dist) {
    const uint32_t base_u = u - lane;
    for (int k = 0; k < 64; ++k) {
      const uint32_t b = __ballot_sync(DAWN_FULL, (nw >> k) & 1ull);
      if (b && ((b >> lane) & 1u))
        p.dist[(size_t)(batch_base + k) * p.n + base_u + lane] = L1;
    }
  }
  __syncwarp();
}

template <int NT>
__global__ void __launch_bounds__(NT) k_ms64(MsParams p) {
  __shared__ MsState st;
  __shared__ unsigned long long hsm[NT];  // per-warp 32-entry hash stash
  __shared__ unsigned long long red[4];
  const uint32_t nblocks = gridDim.x;
  const uint32_t lane = lane_id();
  const uint32_t gwarp = blockIdx.x * (NT / 32) + threadIdx.x / 32;
  const uint32_t nwarps = nblocks * (NT / 32);
  const uint32_t gtid = blockIdx.x * NT + threadIdx.x;
  const uint32_t nthreads = nblocks * NT;
  unsigned long long *hs = hsm + (threadIdx.x & ~31u);
  MsCtrl *C = p.ctrl;
  const uint32_t nbatches = (p.count + 63) / 64;
  const uint32_t ngroups = (p.n + 31) / 32;

  for (uint32_t bt = 0; bt < nbatches; ++bt) {
    const uint32_t bbase = bt * 64;
    const uint32_t bk = min(64u, p.count - bbase);
    const unsigned long long active = bk == 64 ? ~0ull : ((1ull << bk) - 1);
    // ---- init
    for (uint32_t v = gtid; v < p.n; v += nthreads) {
      p.seen[v] = 0;
      p.F[0][v] = 0;
      p.nxt[v] = 0;
    }
    if (p.dist) {
      const size_t tot = (size_t)bk * p.n;
      uint32_t *d0 = p.dist + (size_t)bbase * p.n;
      for (size_t i = gtid; i < tot; i += nthreads) d0[i] = kUnreached;
    }
    if (blockIdx.x == 0 && threadIdx.x < 12) (&C->cnt[0][0])[threadIdx.x] = 0;
    grid_sync(&C->bar, nblocks);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long na = 0, ma = 0;
      for (uint32_t k = 0; k < bk; ++k) {
        const uint32_t s = p.sources[bbase + k];
        if (p.F[0][s] == 0) { na++; ma += p.rp[s + 1] - p.rp[s]; }
        p.seen[s] |= 1ull << k;
        p.F[0][s] |= 1ull << k;
        if (p.dist) p.dist[(size_t)(bbase + k) * p.n + s] = 0;
      }
      C->cnt[0][0] = na;
      C->cnt[0][1] = ma;
    }
    if (threadIdx.x == 0) st = MsState{0, kPush, 0, 0, 0, 0};
    grid_sync(&C->bar, nblocks);

    uint32_t cnt0 = 0, cnt1 = 0, ecc0 = 0, ecc1 = 0;
    unsigned long long h0 = 0, h1 = 0, sd0 = 0, sd1 = 0;
    for (;;) {
      if (threadIdx.x == 0) {
        st.n_active = ld_cg(&C->cnt[st.L % 3][0]);
        st.m_active = ld_cg(&C->cnt[st.L % 3][1]);
        if (blockIdx.x == 0) {
          C->cnt[(st.L + 2) % 3][0] = 0;
          C->cnt[(st.L + 2) % 3][1] = 0;
        }
        st.stop = (st.n_active == 0) || (st.L + 1 >= p.n);
        st.dir = (p.can_pull && (double)st.m_active * p.ms_alpha > (double)p.m) ? kPull : kPush;
      }
      __syncthreads();
      if (st.stop) break;
      const uint32_t L1 = st.L + 1;
      const unsigned long long *Fc = p.F[st.cur];
      unsigned long long *Fn = p.F[st.cur ^ 1];
      uint32_t na = 0;
      unsigned long long ma = 0;
      uint32_t lc0 = 0, lc1 = 0;  // this level's per-source counts (for sum_dist)
      if (st.dir == kPush) {
        // phase A: expand active rows (32 vertices per warp item, edges dealt by shfl search)
        for (uint32_t g = gwarp; g < ngroups; g += nwarps) {
          const uint32_t v = g * 32 + lane;
          unsigned long long fv = 0;
          uint32_t s = 0, d = 0;
          if (v < p.n) {
            fv = Fc[v];
            if (fv) { s = ld_nc(p.rp + v); d = ld_nc(p.rp + v + 1) - s; }
          }
          const uint32_t incl = warp_incl_scan(d);
          const uint32_t total = __shfl_sync(DAWN_FULL, incl, 31);
          const uint32_t excl = incl - d;
          for (uint32_t base = 0; base < total; base += 32) {
            const uint32_t t = base + lane;
            uint32_t k = 0;
#pragma unroll
            for (uint32_t step = 16; step; step >>= 1) {
              const uint32_t e = __shfl_sync(DAWN_FULL, excl, k + step);
              if (e <= t) k += step;
            }
            const uint32_t ek = __shfl_sync(DAWN_FULL, excl, k);
            const uint32_t sk = __shfl_sync(DAWN_FULL, s, k);
            const unsigned long long fk = __shfl_sync(DAWN_FULL, fv, k);
            if (t < total) {
              const uint32_t u = (uint32_t)ld_nc(p.col + sk + (t - ek));
              const unsigned long long x = fk & ~p.seen[u];
              if (x) red_or64(p.nxt + u, x);
            }
          }
        }
        grid_sync(&C->bar, nblocks);
        // phase B: vertex pass
        for (uint32_t g = gwarp; g < ngroups; g += nwarps) {
          const uint32_t u = g * 32 + lane;
          unsigned long long nw = 0;
          if (u < p.n) {
            const unsigned long long nx = ld_cg(p.nxt + u);
            if (nx) {
              const unsigned long long sn = p.seen[u];
              nw = nx & ~sn;
              p.nxt[u] = 0;
              if (nw) {
                p.seen[u] = sn | nw;
                na += 1;
                ma += ld_nc(p.rp + u + 1) - ld_nc(p.rp + u);
              }
            }
            Fn[u] = nw;
          }
          const uint32_t c0 = cnt0, c1 = cnt1;
          ms_record_group(p, nw, u, L1, bbase, hs, cnt0, cnt1, ecc0, ecc1, h0, h1);
          lc0 += cnt0 - c0;
          lc1 += cnt1 - c1;
        }
      } else {
        for (uint32_t g = gwarp; g < ngroups; g += nwarps) {
          const uint32_t u = g * 32 + lane;
          unsigned long long nw = 0;
          if (u < p.n) {
            const unsigned long long sn = p.seen[u];
            const unsigned long long U = ~sn & active;
            if (U) {
              unsigned long long acc = 0;
              const uint32_t s = ld_nc(p.irp + u), e = ld_nc(p.irp + u + 1);
              for (uint32_t j = s; j < e; ++j) {
                acc |= Fc[(uint32_t)ld_nc(p.icol + j)];
                if ((acc & U) == U) break;
              }
              nw = acc & U;
              if (nw) {
                p.seen[u] = sn | nw;
                na += 1;
                ma += p.sym ? (e - s) : (ld_nc(p.rp + u + 1) - ld_nc(p.rp + u));
              }
            }
            Fn[u] = nw;
          }
          const uint32_t c0 = cnt0, c1 = cnt1;
          ms_record_group(p, nw, u, L1, bbase, hs, cnt0, cnt1, ecc0, ecc1, h0, h1);
          lc0 += cnt0 - c0;
          lc1 += cnt1 - c1;
        }
      }
      sd0 += (unsigned long long)lc0 * L1;
      sd1 += (unsigned long long)lc1 * L1;
      // frontier counters for the direction choice / stop test
      na = warp_sum(na);
      ma = warp_sum(ma);
      if (threadIdx.x == 0) { red[0] = 0; red[1] = 0; }
      __syncthreads();
      if (lane == 0 && na) { atomicAdd(&red[0], (unsigned long long)na); atomicAdd(&red[1], ma); }
      __syncthreads();
      if (threadIdx.x == 0 && red[0]) {
        atomicAdd(&C->cnt[(st.L + 1) % 3][0], red[0]);
        atomicAdd(&C->cnt[(st.L + 1) % 3][1], red[1]);
      }
      grid_sync(&C->bar, nblocks);
      if (threadIdx.x == 0) { st.cur ^= 1; st.L++; }
      __syncthreads();
    }
    // ---- records: lane j of every warp holds sources j and j+32 of this batch
    if (p.rec) {
      __shared__ unsigned long long bsum[64], bhash[64];
      __shared__ uint32_t bcnt[64], becc[64];
      if (threadIdx.x < 64) { bsum[threadIdx.x] = 0; bhash[threadIdx.x] = 0; bcnt[threadIdx.x] = 0; becc[threadIdx.x] = 0; }
      __syncthreads();
      if (cnt0) {
        atomicAdd(&bcnt[lane], cnt0);
        atomicMax(&becc[lane], ecc0);
        atomicAdd(&bsum[lane], sd0);
        atomicAdd(&bhash[lane], h0);
      }
      if (cnt1) {
        atomicAdd(&bcnt[lane + 32], cnt1);
        atomicMax(&becc[lane + 32], ecc1);
        atomicAdd(&bsum[lane + 32], sd1);
        atomicAdd(&bhash[lane + 32], h1);
      }
      __syncthreads();
      if (threadIdx.x < 64) {
        const uint32_t k = threadIdx.x;
        p.part[blockIdx.x * 64 + k] = make_uint4(bcnt[k], becc[k], 0, 0);
        p.part[(nblocks + blockIdx.x) * 64 + k] =
            make_uint4((uint32_t)bsum[k], (uint32_t)(bsum[k] >> 32), (uint32_t)bhash[k],
                       (uint32_t)(bhash[k] >> 32));
      }
      grid_sync(&C->bar, nblocks);
      if (blockIdx.x == 0 && threadIdx.x < bk) {
        const uint32_t k = threadIdx.x;
        const uint32_t s = p.sources[bbase + k];
        uint32_t c = 0, e = 0;
        unsigned long long sm = 0, hh = 0;
        for (uint32_t b = 0; b < nblocks; ++b) {
          const uint4 x = __ldcg(p.part + b * 64 + k);
          const uint4 y = __ldcg(p.part + (nblocks + b) * 64 + k);
          c += x.x;
          e = max(e, x.y);
          sm += ((unsigned long long)y.y << 32) | y.x;
          hh += ((unsigned long long)y.w << 32) | y.z;
        }
        dawn_record r;
        r.source = s;
        r.ecc = e;
        r.reached = c;
        r.pad = 0;
        r.sum_dist = sm;
        r.hash = hh + rec_hash(s, 0);
        p.rec[bbase + k] = r;
      }
    }
    grid_sync(&C->bar, nblocks);
  }
}

}  // namespace dawn

// ms64_kernel.cuh — bit-parallel multi-source DAWN (BASELINE.json north_star: "packs 64
// sources per vertex word so one adjacency pass serves 64 BFS trees").
//
// Vertex words (uint64): seen[v] (bit k: source k has reached v), F[v] (bit k: v is in source
// k's level-L frontier), nxt[v] (scratch).  One level generalises Eq. 9
// to 64 right-hand sides over the (OR, AND) semiring:
//   PUSH  for v with F[v] != 0, for u in N+(v): nxt[u] |= F[v] & ~seen[u]          (SOVM)
//         then per vertex: new = nxt & ~seen; seen |= new; F' = new
//   PULL  for u with U = ~seen[u] & active != 0: acc = OR of F[v] over N-(u), stopping as soon
//         as acc covers U (Eq. 4 early exit, per bit set); new = acc & U             (BOVM)
// Rows of degree > kHeavy are split into static kHPiece-edge pieces scanned by whole warps
// (partial ORs meet in nxt[u]); lighter rows are handled per lane / per 32-vertex warp group.
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
  const uint32_t *hout_v, *hout_s, *hout_e, *hout_bits;  // static heavy out-row pieces
  const uint32_t *hin_v, *hin_s, *hin_e, *hin_bits;      // static heavy in-row pieces
  unsigned long long *seen, *F[2], *nxt;
  MsCtrl *ctrl;
  Ctrl *sctrl;               // n_hp_out / n_hp_in
  const uint32_t *sources;   // device, this launch's source list
  uint32_t count;            // number of sources in the list (batches of 64)
  dawn_record *rec;          // device [count] or null
  uint32_t *dist;            // device [count][n] or null
  uint32_t can_pull, sym;
  float ms_alpha;
  uint4 *part;               // per-CTA partial records [2][gridDim.x][64]
};

struct MsState {
  uint32_t L, dir, cur, stop, n_hp_out, n_hp_in;
  unsigned long long n_active, m_active, m_uns;
};

struct MsAcc {  // per-lane record accumulators: sources `lane` and `lane + 32`
  uint32_t cnt0, cnt1, ecc0, ecc1, lc0, lc1;
  unsigned long long h0, h1;
};

__device__ __forceinline__ unsigned long long warp_or64(unsigned long long x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x |= __shfl_xor_sync(DAWN_FULL, x, o);
  return x;
}

// Warp-collective: fold this lane's vertex u new-bits nw (0 if none) into the per-source
// accumulators (bit-transposed with ballots) and, if requested, the dense distance rows.
__device__ __forceinline__ void ms_record_group(const MsParams &p, unsigned long long nw,
                                                uint32_t u, uint32_t L1, uint32_t batch_base,
                                                unsigned long long *hs, MsAcc &a) {
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
  if (m0) { a.lc0 += __popc(m0); a.ecc0 = L1; }
  if (m1) { a.lc1 += __popc(m1); a.ecc1 = L1; }
  while (m0) { a.h0 += hs[__ffs(m0) - 1]; m0 &= m0 - 1; }
  while (m1) { a.h1 += hs[__ffs(m1) - 1]; m1 &= m1 - 1; }
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
  unsigned long long bar_target = 0;

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
    grid_sync(&C->bar, nblocks, bar_target);
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
    if (threadIdx.x == 0) {
      st = MsState{0, kPush, 0, 0, ld_cg(&p.sctrl->n_hp_out), ld_cg(&p.sctrl->n_hp_in), 0, 0,
                   p.m};
    }
    grid_sync(&C->bar, nblocks, bar_target);

    MsAcc a{};
    unsigned long long sd0 = 0, sd1 = 0;
    for (;;) {
      if (threadIdx.x == 0) {
        st.n_active = ld_cg(&C->cnt[st.L % 3][0]);
        st.m_active = ld_cg(&C->cnt[st.L % 3][1]);
        st.m_uns -= ld_cg(&C->cnt[st.L % 3][2]);
        if (blockIdx.x == 0) {
          C->cnt[(st.L + 2) % 3][0] = 0;
          C->cnt[(st.L + 2) % 3][1] = 0;
          C->cnt[(st.L + 2) % 3][2] = 0;
        }
        st.stop = (st.n_active == 0) || (st.L + 1 >= p.n);
        st.dir = (p.can_pull && (double)st.m_active * p.ms_alpha > (double)st.m_uns) ? kPull
                                                                                     : kPush;
      }
      __syncthreads();
      if (st.stop) break;
      const uint32_t L1 = st.L + 1;
      const unsigned long long *Fc = p.F[st.cur];
      unsigned long long *Fn = p.F[st.cur ^ 1];
      uint32_t na = 0;
      unsigned long long ma = 0, mfull = 0;
      a.lc0 = a.lc1 = 0;
      if (st.dir == kPush) {
        // phase A1: light active rows, 32 vertices per warp item, edges dealt by shfl search
        for (uint32_t g = gwarp; g < ngroups; g += nwarps) {
          const uint32_t v = g * 32 + lane;
          const uint32_t hw = ld_nc(p.hout_bits + g);
          unsigned long long fv = 0;
          uint32_t s = 0, d = 0;
          if (v < p.n && !((hw >> lane) & 1u)) {
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
        // phase A2: heavy active rows by static pieces
        for (uint32_t pc = gwarp; pc < st.n_hp_out; pc += nwarps) {
          const uint32_t v = ld_nc(p.hout_v + pc);
          const unsigned long long fv = Fc[v];
          if (!fv) continue;
          const uint32_t s = ld_nc(p.hout_s + pc), e = ld_nc(p.hout_e + pc);
          for (uint32_t j = s + lane; j < e; j += 32) {
            const uint32_t u = (uint32_t)ld_nc(p.col + j);
            const unsigned long long x = fv & ~p.seen[u];
            if (x) red_or64(p.nxt + u, x);
          }
        }
        grid_sync(&C->bar, nblocks, bar_target);
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
                const uint32_t dg = ld_nc(p.rp + u + 1) - ld_nc(p.rp + u);
                na += 1;
                ma += dg;
                if (((sn | nw) & active) == active)
                  mfull += p.sym ? dg : (ld_nc(p.irp + u + 1) - ld_nc(p.irp + u));
              }
            }
            Fn[u] = nw;
          }
          ms_record_group(p, nw, u, L1, bbase, hs, a);
        }
      } else {
        // pass 1a: light in-rows, one lane per vertex, early exit once U is covered
        for (uint32_t g = gwarp; g < ngroups; g += nwarps) {
          const uint32_t u = g * 32 + lane;
          const uint32_t hw = ld_nc(p.hin_bits + g);
          unsigned long long nw = 0;
          if (u < p.n && !((hw >> lane) & 1u)) {
            const unsigned long long sn = p.seen[u];
            const unsigned long long U = ~sn & active;
            if (U) {
              unsigned long long acc = 0;
              const uint32_t s = ld_nc(p.irp + u), e = ld_nc(p.irp + u + 1);
              for (uint32_t j = s; j < e; j += 4) {
                const uint32_t v0 = (uint32_t)ld_nc(p.icol + j);
                const uint32_t v1 = j + 1 < e ? (uint32_t)ld_nc(p.icol + j + 1) : v0;
                const uint32_t v2 = j + 2 < e ? (uint32_t)ld_nc(p.icol + j + 2) : v0;
                const uint32_t v3 = j + 3 < e ? (uint32_t)ld_nc(p.icol + j + 3) : v0;
                acc |= Fc[v0] | Fc[v1] | Fc[v2] | Fc[v3];
                if ((acc & U) == U) break;
              }
              nw = acc & U;
              if (nw) {
                p.seen[u] = sn | nw;
                na += 1;
                const uint32_t din = e - s;
                ma += p.sym ? din : (ld_nc(p.rp + u + 1) - ld_nc(p.rp + u));
                if (nw == U) mfull += din;
              }
            }
            Fn[u] = nw;
          }
          ms_record_group(p, nw, u, L1, bbase, hs, a);
        }
        // pass 1b: heavy in-rows by static pieces; partial ORs meet in nxt[u]
        for (uint32_t pc = gwarp; pc < st.n_hp_in; pc += nwarps) {
          const uint32_t u = ld_nc(p.hin_v + pc);
          // bits already found by earlier pieces of this row (pieces are stored piece-major:
          // all first pieces, then all second pieces, ...) need not be looked for again
          const unsigned long long U = ~p.seen[u] & active & ~ld_cg(p.nxt + u);
          if (!U) continue;
          const uint32_t s = ld_nc(p.hin_s + pc), e = ld_nc(p.hin_e + pc);
          unsigned long long acc = 0;
          for (uint32_t j = s; j < e; j += 32) {
            const unsigned long long f = (j + lane < e) ? Fc[(uint32_t)ld_nc(p.icol + j + lane)] : 0ull;
            acc |= warp_or64(f);
            if ((acc & U) == U) break;
          }
          if (lane == 0 && (acc & U)) red_or64(p.nxt + u, acc & U);
        }
        grid_sync(&C->bar, nblocks, bar_target);
        // pass 2: finalise heavy vertices
        for (uint32_t g = gwarp; g < ngroups; g += nwarps) {
          const uint32_t hw = ld_nc(p.hin_bits + g);
          if (!hw) continue;
          const uint32_t u = g * 32 + lane;
          unsigned long long nw = 0;
          if ((hw >> lane) & 1u) {
            const unsigned long long nx = ld_cg(p.nxt + u);
            if (nx) {
              const unsigned long long sn = p.seen[u];
              nw = nx & ~sn;
              p.nxt[u] = 0;
              if (nw) {
                p.seen[u] = sn | nw;
                const uint32_t din = ld_nc(p.irp + u + 1) - ld_nc(p.irp + u);
                na += 1;
                ma += p.sym ? din : (ld_nc(p.rp + u + 1) - ld_nc(p.rp + u));
                if (((sn | nw) & active) == active) mfull += din;
              }
            }
            Fn[u] = nw;
          }
          ms_record_group(p, nw, u, L1, bbase, hs, a);
        }
      }
      a.cnt0 += a.lc0;
      a.cnt1 += a.lc1;
      sd0 += (unsigned long long)a.lc0 * L1;
      sd1 += (unsigned long long)a.lc1 * L1;
      // frontier counters for the direction choice / stop test
      na = warp_sum(na);
      ma = warp_sum(ma);
      mfull = warp_sum(mfull);
      if (threadIdx.x == 0) { red[0] = 0; red[1] = 0; red[2] = 0; }
      __syncthreads();
      if (lane == 0 && (na | mfull)) {
        atomicAdd(&red[0], (unsigned long long)na);
        atomicAdd(&red[1], ma);
        atomicAdd(&red[2], mfull);
      }
      __syncthreads();
      if (threadIdx.x == 0 && (red[0] | red[2])) {
        atomicAdd(&C->cnt[(st.L + 1) % 3][0], red[0]);
        atomicAdd(&C->cnt[(st.L + 1) % 3][1], red[1]);
        atomicAdd(&C->cnt[(st.L + 1) % 3][2], red[2]);
      }
      grid_sync(&C->bar, nblocks, bar_target);
      if (threadIdx.x == 0) { st.cur ^= 1; st.L++; }
      __syncthreads();
    }
    // ---- records: lane j of every warp holds sources j and j+32 of this batch
    if (p.rec) {
      __shared__ unsigned long long bsum[64], bhash[64];
      __shared__ uint32_t bcnt[64], becc[64];
      if (threadIdx.x < 64) {
        bsum[threadIdx.x] = 0;
        bhash[threadIdx.x] = 0;
        bcnt[threadIdx.x] = 0;
        becc[threadIdx.x] = 0;
      }
      __syncthreads();
      if (a.cnt0) {
        atomicAdd(&bcnt[lane], a.cnt0);
        atomicMax(&becc[lane], a.ecc0);
        atomicAdd(&bsum[lane], sd0);
        atomicAdd(&bhash[lane], a.h0);
      }
      if (a.cnt1) {
        atomicAdd(&bcnt[lane + 32], a.cnt1);
        atomicMax(&becc[lane + 32], a.ecc1);
        atomicAdd(&bsum[lane + 32], sd1);
        atomicAdd(&bhash[lane + 32], a.h1);
      }
      __syncthreads();
      if (threadIdx.x < 64) {
        const uint32_t k = threadIdx.x;
        p.part[blockIdx.x * 64 + k] = make_uint4(bcnt[k], becc[k], 0, 0);
        p.part[(nblocks + blockIdx.x) * 64 + k] =
            make_uint4((uint32_t)bsum[k], (uint32_t)(bsum[k] >> 32), (uint32_t)bhash[k],
                       (uint32_t)(bhash[k] >> 32));
      }
      grid_sync(&C->bar, nblocks, bar_target);
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
  }
  grid_exit(&C->bar, nblocks);
}

}  // namespace dawn

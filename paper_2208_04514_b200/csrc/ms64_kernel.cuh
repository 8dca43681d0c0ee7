// ms64_kernel.cuh — bit-parallel multi-source DAWN (BASELINE.json north_star: "packs 64
// sources per vertex word so one adjacency pass serves 64 BFS trees").
//
// A vertex holds W 64-bit words (kMsW = 4: 256 sources per pass, 32 bytes = one L2 sector,
// so a gather of F[v] costs the same sector whether it carries 64 or 256 sources):
//   seen[v] (bit k: source k has reached v), F[v] (bit k: v is in source k's level-L
//   frontier), nxt[v] (scratch).  One level generalises Eq. 9 to 64·W
//   right-hand sides over the (OR, AND) semiring:
//   PUSH  for v with F[v] != 0, for u in N+(v): nxt[u] |= F[v] & ~seen[u]          (SOVM)
//         then per vertex: new = nxt & ~seen; seen |= new; F' = new
//   PULL  for u with U = ~seen[u] & active != 0: acc = OR of F[v] over N-(u), stopping as soon
//         as acc covers U (Eq. 4 early exit, per bit set); new = acc & U             (BOVM)
// Rows of degree > kHeavy are split into static kHPiece-edge pieces (stored piece-major)
// scanned by whole warps; partial ORs meet in nxt[u].  Per-source records (ecc, reached,
// sum_dist, hash) are accumulated without per-event global atomics: a warp's 32 new-words are
// bit-transposed with ballots (lane j gets the 32-vertex mask of source 32i + j) and folded
// into per-CTA shared-memory accumulators.
#pragma once
#include "layout.h"

#ifndef DAWN_MS_PUSH_U
#define DAWN_MS_PUSH_U 4  // 32-arc rounds batched per warp iteration (push phases, heavy pulls)
#endif
#ifndef DAWN_MS_PULL_U
#define DAWN_MS_PULL_U 4  // in-neighbour gathers per lane per round trip in the light pull pass
#endif


namespace dawn {

template <int W>
struct alignas(8 * W) Word {
  unsigned long long w[W];
};

template <int W>
__device__ __forceinline__ Word<W> wload(const unsigned long long *p, uint32_t v) {
  Word<W> r;
  if constexpr (W % 2 == 0) {
    const ulonglong2 *q = reinterpret_cast<const ulonglong2 *>(p + (size_t)v * W);
#pragma unroll
    for (int i = 0; i < W / 2; ++i) {
      const ulonglong2 x = q[i];
      r.w[2 * i] = x.x;
      r.w[2 * i + 1] = x.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) r.w[i] = p[(size_t)v * W + i];
  }
  return r;
}
template <int W>
__device__ __forceinline__ Word<W> wload_cg(const unsigned long long *p, uint32_t v) {
  Word<W> r;
#pragma unroll
  for (int i = 0; i < W; ++i) r.w[i] = ld_cg(p + (size_t)v * W + i);
  return r;
}
template <int W>
__device__ __forceinline__ void wstore(unsigned long long *p, uint32_t v, const Word<W> &x) {
  if constexpr (W % 2 == 0) {
    ulonglong2 *q = reinterpret_cast<ulonglong2 *>(p + (size_t)v * W);
#pragma unroll
    for (int i = 0; i < W / 2; ++i) q[i] = make_ulonglong2(x.w[2 * i], x.w[2 * i + 1]);
  } else {
#pragma unroll
    for (int i = 0; i < W; ++i) p[(size_t)v * W + i] = x.w[i];
  }
}
template <int W>
__device__ __forceinline__ bool wany(const Word<W> &x) {
  unsigned long long o = 0;
#pragma unroll
  for (int i = 0; i < W; ++i) o |= x.w[i];
  return o != 0;
}
template <int W>
__device__ __forceinline__ Word<W> wzero() {
  Word<W> r;
#pragma unroll
  for (int i = 0; i < W; ++i) r.w[i] = 0;
  return r;
}

struct MsParams {
  uint32_t n, nwords;
  unsigned long long m;
  const uint32_t *rp, *irp;
  const int32_t *col, *icol;
  const uint32_t *hout_v, *hout_s, *hout_e, *hout_bits;  // static heavy out-row pieces
  const uint32_t *hin_v, *hin_s, *hin_e, *hin_bits;      // static heavy in-row pieces
  unsigned long long *seen, *F[2], *nxt;                 // [n][kMsW] words
  MsCtrl *ctrl;
  Ctrl *sctrl;               // n_hp_out / n_hp_in
  const uint32_t *sources;   // device, this launch's source list
  uint32_t count;            // number of sources in the list (batches of kMsBatch)
  dawn_record *rec;          // device [count] or null
  uint32_t *dist;            // device [count][n] or null
  uint32_t can_pull, sym;
  float ms_alpha;
  uint4 *part;               // per-CTA partial records [2][gridDim.x][kMsBatch]
  TraceRec *trace;           // per-level trace of the first batch (DAWN_GRAPH_TRACE) or null
  uint32_t *trace_n;
};

struct MsState {
  uint32_t L, dir, cur, stop, n_hp_out, n_hp_in;
  unsigned long long n_active, m_active, m_uns;
};

// Per-warp record accumulators of the current batch (dynamic shared memory, one slice per warp):
// lane j of a warp owns sources 32i + j (i < 2W) of its slice, so the updates need no atomics;
// the CTA folds its slices once per batch.
struct MsWarpAcc {
  unsigned long long sum[kMsBatch], hash[kMsBatch];
  uint32_t cnt[kMsBatch], ecc[kMsBatch];
  unsigned long long tab[8][16];  // subset sums of the group's hash terms, per 4-lane block
};
inline size_t ms_smem_bytes(int nt) { return sizeof(MsWarpAcc) * (size_t)(nt / 32); }


// Warp-collective: fold this lane's vertex u new-bits nw into the per-CTA accumulators and, if
// requested, the dense distance rows.  Lane j receives, for source block i, the 32-vertex
// mask of source 32i + j (one ballot per source).
// Lane j gets column j of the 32x32 bit matrix whose row k is lane k's x (butterfly transpose:
// five shfl_xor stages instead of 32 ballots).
__device__ __forceinline__ uint32_t transpose32(uint32_t x) {
  const uint32_t lane = lane_id();
  uint32_t m = 0x0000FFFFu;
#pragma unroll
  for (uint32_t s = 16; s > 0; s >>= 1) {
    const uint32_t y = __shfl_xor_sync(DAWN_FULL, x, s);
    x = (lane & s) ? ((x & ~m) | ((y & ~m) >> s)) : ((x & m) | ((y & m) << s));
    m ^= m << (s >> 1);
  }
  return x;
}

// Warp-collective: fold this lane's vertex u new-bits nw into the warp's record slice and, if
// requested, the dense distance rows.  Lane j receives, for source block i, the 32-vertex
// mask of source 32i + j (a bit-matrix transpose of the warp's new-words).
template <int W>
__device__ __forceinline__ void ms_record_group(const MsParams &p, const Word<W> &nw, uint32_t u,
                                                uint32_t L1, uint32_t batch_base,
                                                unsigned long long *hs, MsWarpAcc &wa) {
  const bool mine = wany<W>(nw);
  if (!__any_sync(DAWN_FULL, mine)) return;
  const uint32_t lane = lane_id();
  // tab[b][m] = sum of the hash terms of lanes 4b + i for the bits i of m: a source's hash
  // contribution over a 32-vertex mask is then 8 table reads instead of popc(mask) dependent ones
  {
    // lane l builds entries m = 4 (l & 3) .. + 3 of block b = l >> 2 from the block's four hash
    // terms, fetched by shuffles
    const unsigned long long mh = mine ? rec_hash(u, L1) : 0ull;
    const uint32_t b = lane >> 2, q = lane & 3;
    unsigned long long h4[4];
#pragma unroll
    for (uint32_t i = 0; i < 4; ++i) h4[i] = __shfl_sync(DAWN_FULL, mh, 4 * b + i);
#pragma unroll
    for (uint32_t r = 0; r < 4; ++r) {
      const uint32_t m = 4 * q + r;
      unsigned long long v = 0;
#pragma unroll
      for (uint32_t i = 0; i < 4; ++i)
        if ((m >> i) & 1u) v += h4[i];
      wa.tab[b][m] = v;
    }
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 2 * W; ++i) {
    const unsigned long long word = nw.w[i >> 1];
    const uint32_t half = (uint32_t)(word >> ((i & 1) * 32));
    if (!__any_sync(DAWN_FULL, half != 0)) continue;
    uint32_t mk = transpose32(half);
    if (mk) {
      const uint32_t src = 32 * i + lane;
      const uint32_t c = __popc(mk);
      unsigned long long h = 0;
#pragma unroll
      for (uint32_t b = 0; b < 8; ++b) h += wa.tab[b][(mk >> (4 * b)) & 15u];
      wa.cnt[src] += c;
      wa.ecc[src] = L1;  // levels only grow
      wa.sum[src] += (unsigned long long)c * L1;
      wa.hash[src] += h;
      if (p.dist) {
        // lane j owns source src: its row gets L1 at the vertices of mk
        uint32_t *row = p.dist + (size_t)(batch_base + src) * p.n + (u - lane);
        while (mk) {
          row[__ffs(mk) - 1] = L1;
          mk &= mk - 1;
        }
      }
    }
  }
  __syncwarp();
}

#ifndef DAWN_MS_MINB
#define DAWN_MS_MINB 1
#endif
template <int NT>
__global__ void __launch_bounds__(NT, DAWN_MS_MINB) k_ms64(MsParams p) {
  constexpr int W = kMsW;
  __shared__ MsState st;
  __shared__ unsigned long long hsm[NT];  // per-warp 32-entry hash stash
  __shared__ unsigned long long red[4];
  extern __shared__ __align__(16) unsigned char ms_dyn[];
  MsWarpAcc &wacc = reinterpret_cast<MsWarpAcc *>(ms_dyn)[threadIdx.x / 32];
  const uint32_t nblocks = gridDim.x;
  const uint32_t lane = lane_id();
  const uint32_t gwarp = blockIdx.x * (NT / 32) + threadIdx.x / 32;
  const uint32_t nwarps = nblocks * (NT / 32);
  const uint32_t gtid = blockIdx.x * NT + threadIdx.x;
  const uint32_t nthreads = nblocks * NT;
  unsigned long long *hs = hsm + (threadIdx.x & ~31u);
  MsCtrl *C = p.ctrl;
  const uint32_t nbatches = (p.count + kMsBatch - 1) / kMsBatch;
  const uint32_t ngroups = (p.n + 31) / 32;
  unsigned long long bar_target = 0;
  unsigned long long c_arcs = 0, c_reds = 0;  // executed-schedule counters (MsCtrl::stat)

  for (uint32_t bt = 0; bt < nbatches; ++bt) {
    const uint32_t bbase = bt * kMsBatch;
    const uint32_t bk = min(kMsBatch, p.count - bbase);
    Word<W> active;
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const int lo = 64 * i;
      active.w[i] = (int)bk >= lo + 64 ? ~0ull : ((int)bk <= lo ? 0ull : ((1ull << (bk - lo)) - 1));
    }
    // ---- init
    // nxt is all-zero at the end of every batch (each level's vertex pass clears what it
    // consumed), so only the launch's first batch clears it
    for (size_t x = gtid; x < (size_t)p.n * W; x += nthreads) {
      p.seen[x] = 0;
      p.F[0][x] = 0;
      if (bt == 0) p.nxt[x] = 0;
    }
    if (p.dist) {
      const size_t tot = (size_t)bk * p.n;
      uint32_t *d0 = p.dist + (size_t)bbase * p.n;
      for (size_t i = gtid; i < tot; i += nthreads) d0[i] = kUnreached;
    }
    for (uint32_t i = lane; i < kMsBatch; i += 32) {
      wacc.sum[i] = 0;
      wacc.hash[i] = 0;
      wacc.cnt[i] = 0;
      wacc.ecc[i] = 0;
    }
    if (blockIdx.x == 0 && threadIdx.x < 12) (&C->cnt[0][0])[threadIdx.x] = 0;
    grid_sync(&C->bar, nblocks, bar_target);
    if (blockIdx.x == 0) {
      // batch sources in parallel (one thread per source): set bit k of s's seen / frontier
      // words; the level-0 frontier counters count each distinct vertex once (a repeated source
      // is counted by its first occurrence only).  A serial loop here had held every other CTA
      // at the next barrier for ~200 us per batch.
      uint32_t *ssrc = reinterpret_cast<uint32_t *>(hsm);  // hsm is free outside the levels
      for (uint32_t k = threadIdx.x; k < bk; k += NT) ssrc[k] = p.sources[bbase + k];
      __syncthreads();
      unsigned long long na = 0, ma = 0;
      for (uint32_t k = threadIdx.x; k < bk; k += NT) {
        const uint32_t s = ssrc[k];
        bool fresh = true;
        for (uint32_t j = 0; j < k && fresh; ++j) fresh = ssrc[j] != s;
        if (fresh) { na += 1; ma += p.rp[s + 1] - p.rp[s]; }
        atomicOr(p.seen + (size_t)s * W + k / 64, 1ull << (k % 64));
        atomicOr(p.F[0] + (size_t)s * W + k / 64, 1ull << (k % 64));
        if (p.dist) p.dist[(size_t)(bbase + k) * p.n + s] = 0;
      }
      na = warp_sum(na);
      ma = warp_sum(ma);
      if (lane == 0 && na) {
        atomicAdd(&C->cnt[0][0], na);
        atomicAdd(&C->cnt[0][1], ma);
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      st = MsState{0, kPush, 0, 0, ld_cg(&p.sctrl->n_hp_out), ld_cg(&p.sctrl->n_hp_in), 0, 0,
                   p.m};
    }
    grid_sync(&C->bar, nblocks, bar_target);

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
        if (p.trace && bt == 0 && blockIdx.x == 0 && st.L < kTraceCap) {
          TraceRec r{};
          unsigned long long t;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          r.t_ns = t;
          r.level = st.L;
          r.dir = st.stop ? 2u : st.dir;
          r.nf = (uint32_t)st.n_active;
          r.mf = st.m_active;
          p.trace[st.L] = r;
          *p.trace_n = st.L + 1;
        }
      }
      __syncthreads();
      if (st.stop) break;
      const bool trc = p.trace && bt == 0 && st.L < kTraceCap;  // per-phase slowest-warp cycles
      long long tA = trc ? clock64() : 0, tB = 0, tC = 0, trec = 0, tL = 0;
      const uint32_t L1 = st.L + 1;
      const unsigned long long *Fc = p.F[st.cur];
      unsigned long long *Fn = p.F[st.cur ^ 1];
      uint32_t na = 0;
      unsigned long long ma = 0, mfull = 0;
      if (st.dir == kPush) {
        // phase A1: light active rows, 32 vertices per warp item, edges dealt by shfl search
        for (uint32_t g = gwarp; g < ngroups; g += nwarps) {
          const uint32_t v = g * 32 + lane;
          const uint32_t hw = ld_nc(p.hout_bits + g);
          Word<W> fv = wzero<W>();
          uint32_t s = 0, d = 0;
          if (v < p.n && !((hw >> lane) & 1u)) {
            fv = wload<W>(Fc, v);
            if (wany<W>(fv)) { s = ld_nc(p.rp + v); d = ld_nc(p.rp + v + 1) - s; }
          }
          const uint32_t incl = warp_incl_scan(d);
          const uint32_t total = __shfl_sync(DAWN_FULL, incl, 31);
          const uint32_t excl = incl - d;
          // kPU rounds of 32 arcs per iteration: every target and seen-word load of the batch is
          // issued before the first red.or (the asm memory clobber would otherwise serialise
          // the rounds into load -> gather -> red chains)
          constexpr uint32_t kPU = DAWN_MS_PUSH_U;
          for (uint32_t base = 0; base < total; base += 32 * kPU) {
            uint32_t u[kPU];
            Word<W> fk[kPU];
#pragma unroll
            for (uint32_t r = 0; r < kPU; ++r) {
              const uint32_t t = base + 32 * r + lane;
              uint32_t k = 0;
#pragma unroll
              for (uint32_t step = 16; step; step >>= 1) {
                const uint32_t e = __shfl_sync(DAWN_FULL, excl, k + step);
                if (e <= t) k += step;
              }
              const uint32_t ek = __shfl_sync(DAWN_FULL, excl, k);
              const uint32_t sk = __shfl_sync(DAWN_FULL, s, k);
#pragma unroll
              for (int i = 0; i < W; ++i) fk[r].w[i] = __shfl_sync(DAWN_FULL, fv.w[i], k);
              u[r] = (t < total) ? (uint32_t)ld_nc(p.col + sk + (t - ek)) : 0xffffffffu;
            }
            Word<W> su[kPU];
#pragma unroll
            for (uint32_t r = 0; r < kPU; ++r)
              su[r] = (u[r] != 0xffffffffu) ? wload<W>(p.seen, u[r]) : wzero<W>();
#pragma unroll
            for (uint32_t r = 0; r < kPU; ++r) {
              if (u[r] == 0xffffffffu) continue;
              ++c_arcs;
#pragma unroll
              for (int i = 0; i < W; ++i) {
                const unsigned long long x = fk[r].w[i] & ~su[r].w[i];
                if (x) { red_or64(p.nxt + (size_t)u[r] * W + i, x); ++c_reds; }
              }
            }
          }
        }
        if (trc) tL = clock64();
        // phase A2: heavy active rows by static pieces.  Warp w takes pieces w + k * nwarps (the
        // live ones of a level spread over all warps) and tests 32 of them at once (lane k: is the
        // piece's vertex in the frontier?) before expanding the live ones — a per-piece test was
        // two dependent round trips, ~20 per warp per level even when nothing was live
        const uint32_t hend = st.n_hp_out;
        for (uint32_t pb = gwarp; pb < hend; pb += 32 * nwarps) {
          const uint32_t pcl = pb + lane * nwarps;
          uint32_t vl = 0;
          bool live = false;
          if (pcl < hend) {
            vl = ld_nc(p.hout_v + pcl);
            live = wany<W>(wload<W>(Fc, vl));
          }
          uint32_t lm = __ballot_sync(DAWN_FULL, live);
          while (lm) {
          const uint32_t kk = __ffs(lm) - 1;
          lm &= lm - 1;
          const uint32_t pc = pb + kk * nwarps;
          const uint32_t v = __shfl_sync(DAWN_FULL, vl, kk);
          const Word<W> fv = wload<W>(Fc, v);
          const uint32_t s = ld_nc(p.hout_s + pc), e = ld_nc(p.hout_e + pc);
          constexpr uint32_t kPU = DAWN_MS_PUSH_U;  // rounds batched as in phase A1
          for (uint32_t j0 = s + lane; j0 < e; j0 += 32 * kPU) {
            uint32_t u[kPU];
#pragma unroll
            for (uint32_t r = 0; r < kPU; ++r)
              u[r] = (j0 + 32 * r < e) ? (uint32_t)ld_nc(p.col + j0 + 32 * r) : 0xffffffffu;
            Word<W> su[kPU];
#pragma unroll
            for (uint32_t r = 0; r < kPU; ++r)
              su[r] = (u[r] != 0xffffffffu) ? wload<W>(p.seen, u[r]) : wzero<W>();
#pragma unroll
            for (uint32_t r = 0; r < kPU; ++r) {
              if (u[r] == 0xffffffffu) continue;
              ++c_arcs;
#pragma unroll
              for (int i = 0; i < W; ++i) {
                const unsigned long long x = fv.w[i] & ~su[r].w[i];
                if (x) { red_or64(p.nxt + (size_t)u[r] * W + i, x); ++c_reds; }
              }
            }
          }
          }
        }
        if (trc) tB = clock64();
        grid_sync(&C->bar, nblocks, bar_target);
        if (trc) tC = clock64();
        // phase B: vertex pass
        for (uint32_t g = gwarp; g < ngroups; g += nwarps) {
          const uint32_t u = g * 32 + lane;
          Word<W> nw = wzero<W>();
          if (u < p.n) {
            const Word<W> nx = wload_cg<W>(p.nxt, u);
            if (wany<W>(nx)) {
              const Word<W> sn = wload<W>(p.seen, u);
              bool full = true;
#pragma unroll
              for (int i = 0; i < W; ++i) {
                nw.w[i] = nx.w[i] & ~sn.w[i];
                full = full && ((sn.w[i] | nw.w[i]) & active.w[i]) == active.w[i];
              }
              wstore<W>(p.nxt, u, wzero<W>());
              if (wany<W>(nw)) {
                Word<W> sv;
#pragma unroll
                for (int i = 0; i < W; ++i) sv.w[i] = sn.w[i] | nw.w[i];
                wstore<W>(p.seen, u, sv);
                const uint32_t dg = ld_nc(p.rp + u + 1) - ld_nc(p.rp + u);
                na += 1;
                ma += dg;
                if (full) mfull += p.sym ? dg : (ld_nc(p.irp + u + 1) - ld_nc(p.irp + u));
              }
            }
            wstore<W>(Fn, u, nw);
          }
          {
            const long long tr0 = trc ? clock64() : 0;
            ms_record_group<W>(p, nw, u, L1, bbase, hs, wacc);
            if (trc) trec += clock64() - tr0;
          }
        }
      } else {
        // pass 1a: light in-rows, one lane per vertex, early exit once U is covered
        for (uint32_t g = gwarp; g < ngroups; g += nwarps) {
          const uint32_t u = g * 32 + lane;
          const uint32_t hw = ld_nc(p.hin_bits + g);
          Word<W> nw = wzero<W>();
          if (u < p.n && !((hw >> lane) & 1u)) {
            const Word<W> sn = wload<W>(p.seen, u);
            Word<W> U;
#pragma unroll
            for (int i = 0; i < W; ++i) U.w[i] = ~sn.w[i] & active.w[i];
            if (wany<W>(U)) {
              Word<W> a = wzero<W>();
              const uint32_t s = ld_nc(p.irp + u), e = ld_nc(p.irp + u + 1);
              constexpr uint32_t PU = DAWN_MS_PULL_U;  // in-neighbour gathers in flight per lane
              for (uint32_t j = s; j < e; j += PU) {
                uint32_t vv[PU];
#pragma unroll
                for (uint32_t x = 0; x < PU; ++x)
                  vv[x] = (x == 0 || j + x < e) ? (uint32_t)ld_nc(p.icol + j + x) : 0xffffffffu;
#pragma unroll
                for (uint32_t x = 0; x < PU; ++x) {
                  if (vv[x] == 0xffffffffu) continue;
                  ++c_arcs;
                  const Word<W> f = wload<W>(Fc, vv[x]);
#pragma unroll
                  for (int i = 0; i < W; ++i) a.w[i] |= f.w[i];
                }
                bool cov = true;
#pragma unroll
                for (int i = 0; i < W; ++i) cov = cov && (a.w[i] & U.w[i]) == U.w[i];
                if (cov) break;
              }
              bool full = true;
#pragma unroll
              for (int i = 0; i < W; ++i) {
                nw.w[i] = a.w[i] & U.w[i];
                full = full && nw.w[i] == U.w[i];
              }
              if (wany<W>(nw)) {
                Word<W> sv;
#pragma unroll
                for (int i = 0; i < W; ++i) sv.w[i] = sn.w[i] | nw.w[i];
                wstore<W>(p.seen, u, sv);
                na += 1;
                const uint32_t din = e - s;
                ma += p.sym ? din : (ld_nc(p.rp + u + 1) - ld_nc(p.rp + u));
                if (full) mfull += din;
              }
            }
            wstore<W>(Fn, u, nw);
          }
          {
            const long long tr0 = trc ? clock64() : 0;
            ms_record_group<W>(p, nw, u, L1, bbase, hs, wacc);
            if (trc) trec += clock64() - tr0;
          }
        }
        if (trc) tL = clock64();
        // pass 1b: heavy in-rows by static pieces; partial ORs meet in nxt[u]
        // (pieces w + k * nwarps, 32 tested at once, as in phase A2)
        const uint32_t iend = st.n_hp_in;
        for (uint32_t pb = gwarp; pb < iend; pb += 32 * nwarps) {
          const uint32_t pcl = pb + lane * nwarps;
          uint32_t ul = 0;
          bool live = false;
          if (pcl < iend) {
            ul = ld_nc(p.hin_v + pcl);
            const Word<W> sn = wload<W>(p.seen, ul), have = wload_cg<W>(p.nxt, ul);
#pragma unroll
            for (int i = 0; i < W; ++i) live = live || (~sn.w[i] & active.w[i] & ~have.w[i]) != 0;
          }
          uint32_t lm = __ballot_sync(DAWN_FULL, live);
          while (lm) {
          const uint32_t kk = __ffs(lm) - 1;
          lm &= lm - 1;
          const uint32_t pc = pb + kk * nwarps;
          const uint32_t u = __shfl_sync(DAWN_FULL, ul, kk);
          // bits already found by earlier pieces of this row (pieces are stored piece-major:
          // all first pieces, then all second pieces, ...) need not be looked for again
          const Word<W> sn = wload<W>(p.seen, u), have = wload_cg<W>(p.nxt, u);
          Word<W> U;
#pragma unroll
          for (int i = 0; i < W; ++i) U.w[i] = ~sn.w[i] & active.w[i] & ~have.w[i];
          if (!wany<W>(U)) continue;
          const uint32_t s = ld_nc(p.hin_s + pc), e = ld_nc(p.hin_e + pc);
          Word<W> a = wzero<W>();
          constexpr uint32_t kHU = DAWN_MS_PUSH_U;  // 32 * kHU in-edges per round trip
          for (uint32_t j = s; j < e; j += 32 * kHU) {
            Word<W> f = wzero<W>();
            {
              uint32_t vv[kHU];
#pragma unroll
              for (uint32_t r = 0; r < kHU; ++r)
                vv[r] = (j + 32 * r + lane < e) ? (uint32_t)ld_nc(p.icol + j + 32 * r + lane)
                                                : 0xffffffffu;
#pragma unroll
              for (uint32_t r = 0; r < kHU; ++r) {
                if (vv[r] == 0xffffffffu) continue;
                ++c_arcs;
                const Word<W> g = wload<W>(Fc, vv[r]);
#pragma unroll
                for (int i = 0; i < W; ++i) f.w[i] |= g.w[i];
              }
            }
            bool cov = true;
#pragma unroll
            for (int i = 0; i < W; ++i) {
              unsigned long long x = f.w[i];
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) x |= __shfl_xor_sync(DAWN_FULL, x, o);
              a.w[i] |= x;
              cov = cov && (a.w[i] & U.w[i]) == U.w[i];
            }
            if (cov) break;
          }
#pragma unroll
          for (int i = 0; i < W; ++i) {
            const unsigned long long x = a.w[i] & U.w[i];
            if (lane == (uint32_t)i && x) { red_or64(p.nxt + (size_t)u * W + i, x); ++c_reds; }
          }
          }
        }
        if (trc) tB = clock64();
        grid_sync(&C->bar, nblocks, bar_target);
        if (trc) tC = clock64();
        // pass 2: finalise heavy vertices
        for (uint32_t g = gwarp; g < ngroups; g += nwarps) {
          const uint32_t hw = ld_nc(p.hin_bits + g);
          if (!hw) continue;
          const uint32_t u = g * 32 + lane;
          Word<W> nw = wzero<W>();
          if ((hw >> lane) & 1u) {
            const Word<W> nx = wload_cg<W>(p.nxt, u);
            if (wany<W>(nx)) {
              const Word<W> sn = wload<W>(p.seen, u);
              bool full = true;
#pragma unroll
              for (int i = 0; i < W; ++i) {
                nw.w[i] = nx.w[i] & ~sn.w[i];
                full = full && ((sn.w[i] | nw.w[i]) & active.w[i]) == active.w[i];
              }
              wstore<W>(p.nxt, u, wzero<W>());
              if (wany<W>(nw)) {
                Word<W> sv;
#pragma unroll
                for (int i = 0; i < W; ++i) sv.w[i] = sn.w[i] | nw.w[i];
                wstore<W>(p.seen, u, sv);
                const uint32_t din = ld_nc(p.irp + u + 1) - ld_nc(p.irp + u);
                na += 1;
                ma += p.sym ? din : (ld_nc(p.rp + u + 1) - ld_nc(p.rp + u));
                if (full) mfull += din;
              }
            }
            wstore<W>(Fn, u, nw);
          }
          {
            const long long tr0 = trc ? clock64() : 0;
            ms_record_group<W>(p, nw, u, L1, bbase, hs, wacc);
            if (trc) trec += clock64() - tr0;
          }
        }
      }
      if (trc && lane == 0) {
        const long long tD = clock64();
        atomicMax(&p.trace[st.L].cyc[0], (unsigned long long)(tB - tA));
        // pass-A balance: t_first = sum over warps of pass A cycles, t_last = slowest light pass
        atomicAdd(&p.trace[st.L].t_first, (unsigned long long)(tB - tA));
        atomicMax(&p.trace[st.L].t_last, (unsigned long long)(tL - tA));
        atomicMax(&p.trace[st.L].cyc[1], (unsigned long long)(tC - tB));
        atomicMax(&p.trace[st.L].cyc[2], (unsigned long long)(tD - tC));
        atomicMax(&p.trace[st.L].cyc[3], (unsigned long long)trec);
      }
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
      if (threadIdx.x == 0) {
        if (blockIdx.x == 0) atomicAdd(&C->stat[0], 1ull);
        st.cur ^= 1;
        st.L++;
      }
      __syncthreads();
    }
    // ---- records: per-CTA partials, reduced by CTA 0 after a barrier
    if (p.rec) {
      __syncthreads();  // every warp's slice is final
      const MsWarpAcc *slices = reinterpret_cast<const MsWarpAcc *>(ms_dyn);
      for (uint32_t k = threadIdx.x; k < kMsBatch; k += NT) {
        uint32_t c = 0, e = 0;
        unsigned long long sm = 0, hh = 0;
        for (uint32_t w = 0; w < NT / 32; ++w) {
          c += slices[w].cnt[k];
          e = max(e, slices[w].ecc[k]);
          sm += slices[w].sum[k];
          hh += slices[w].hash[k];
        }
        p.part[blockIdx.x * kMsBatch + k] = make_uint4(c, e, 0, 0);
        p.part[(nblocks + blockIdx.x) * kMsBatch + k] =
            make_uint4((uint32_t)sm, (uint32_t)(sm >> 32), (uint32_t)hh, (uint32_t)(hh >> 32));
      }
      grid_sync(&C->bar, nblocks, bar_target);
      // one warp per source over the whole grid, lanes split the CTA partials (one CTA doing
      // all 256 sources serially over 148 partials each held the grid ~20 us per batch)
      for (uint32_t k = gwarp; k < bk; k += nwarps) {
        uint32_t c = 0, e = 0;
        unsigned long long sm = 0, hh = 0;
        for (uint32_t b = lane; b < nblocks; b += 32) {
          const uint4 x = __ldcg(p.part + b * kMsBatch + k);
          const uint4 y = __ldcg(p.part + (nblocks + b) * kMsBatch + k);
          c += x.x;
          e = max(e, x.y);
          sm += ((unsigned long long)y.y << 32) | y.x;
          hh += ((unsigned long long)y.w << 32) | y.z;
        }
        c = warp_sum(c);
        sm = warp_sum(sm);
        hh = warp_sum(hh);
#pragma unroll
        for (int o = 16; o; o >>= 1) e = max(e, __shfl_xor_sync(DAWN_FULL, e, o));
        if (lane == 0) {
          const uint32_t s = p.sources[bbase + k];
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
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&C->stat[3], 1ull);
  }
  c_arcs = warp_sum(c_arcs);
  c_reds = warp_sum(c_reds);
  if (lane == 0 && (c_arcs | c_reds)) {
    atomicAdd(&C->stat[1], c_arcs);
    atomicAdd(&C->stat[2], c_reds);
  }
  grid_exit(&C->bar, nblocks);
}

}  // namespace dawn

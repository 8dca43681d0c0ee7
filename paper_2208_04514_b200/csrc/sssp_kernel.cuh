// sssp_kernel.cuh — single-source DAWN as ONE persistent cooperative kernel (sm_100a).
//
// One launch = init + every level + statistics.  Each level is either
//   PUSH (SOVM, Algorithm 2; Eq. 9): the frontier queue's CSR rows
//        are expanded; a target u is claimed by an atomic test-and-set on the `vis` bitmap
//        (the "distance[col[j]] = 0" filter of line 6, reading Q1), dist[u] = L+1, and u is
//        appended to the next queue through a per-warp shared-memory stage (ballot + popc),
//        flushed 32 entries per global atomic;
//   PULL (BOVM, Algorithm 1; Eq. 4): every unreached vertex scans
//        its CSC row until the first in-neighbour in the level-L frontier bitmap (early exit).
//        Rows of in-degree <= kHeavy: one lane each, 4 probes per round trip; longer rows: a
//        static list of kHPiece-edge pieces scanned by whole warps (32 probes per round trip,
//        early exit across pieces through the `vis` bit).  The frontier bitmap read is a
//        level-start snapshot; the next one is a separate buffer (reading Q2).
// The direction is chosen on the device from the frontier's measured size (n_f, m_f) against
// the unexplored edges (Beamer's rule, cited by the paper at L123), and the frontier-empty
// test (PAPER.md L174-179 conditions 1-2) is evaluated after each grid barrier: no host
// round trip per level.
#pragma once
#include "layout.h"

namespace dawn {

#ifndef DAWN_TRACE_MAX
#define DAWN_TRACE_MAX 0  // experiment: trace per-phase max over warps instead of the sum
#endif
#define DIST_ST(i, v) (st.drow[i] = (v))

struct SsspParams {
  uint32_t n, nwords;
  unsigned long long m;
  const uint32_t *rp, *irp;
  const int32_t *col, *icol;
  const uint32_t *noin;
  const uint32_t *hin_v, *hin_s, *hin_e, *hin_bits;  // static heavy in-row pieces
  const uint32_t *hasin;  // static ascending list of vertices with an in-edge (n_hasin)
  const uint32_t *top1;   // [n]: first entry of each degree-ordered in-row, or null
  uint32_t *ulist, *useg;  // unreached list (per-warp segments) and segment counts
  uint32_t n_hasin;
  uint32_t *vis, *cand, *fb[3];  // cand: candidate bitmap of bitmap-push levels (zero between uses)
  uint32_t *Lv[2];   // frontier queue: vertex
  uint2 *Lsd[2];     //                 (row start, edge offset within the frontier)
  uint32_t *Cf[2];   //                 chunk c -> entry holding edge c*kChunk
  Ctrl *ctrl;
  TraceRec *trace;
  uint32_t *dist;
  dawn_sssp_stats *stats;
  uint32_t source, variant, can_pull, sym;
  float alpha, beta;
  uint32_t bmpush_e, solo_e;  // DAWN_PARAM_BITMAP_PUSH_EDGES / DAWN_PARAM_SOLO_EDGES
  uint32_t bmpush_grow;       // bitmap push threshold while the frontier grows
  uint32_t seq;               // call number (k_narrow hand-over)
  // batch mode (dawn_sssp_batch): nsrc > 0 sources from the device array `sources`, searched one
  // after the other in this launch; source i writes dist + i * n and stats[i]
  const uint32_t *sources;
  uint32_t nsrc;
  // device source list validated before any write (dawn_sssp_batch; vn = 0: host-validated)
  const uint32_t *vsrc;
  uint32_t vn;
  // dynamic batch lanes: every lane takes the next unclaimed index of the whole batch from this
  // shared counter (one atomic per search, one ahead) instead of a fixed contiguous share, so
  // lanes finish together; sources / dist / stats then address the whole batch (nsrc = k)
  uint32_t *claim;
};

// Every CTA checks the whole device source list of a dawn_sssp_batch call before it writes
// anything (identical inputs -> the same decision in every CTA, no communication).  A bad id
// sets the handle's sticky flag (dawn_graph_check reports DAWN_ERR_BOUNDS) and the kernel
// exits with every output untouched (validation before work).
template <int NT>
__device__ __forceinline__ bool sources_invalid(const uint32_t *vsrc, uint32_t vn, uint32_t n,
                                                uint32_t *flag) {
  bool bad = false;
  for (uint32_t i = threadIdx.x; i < vn; i += NT) bad |= ld_nc(vsrc + i) >= n;
  bad = __syncthreads_or(bad);
  if (bad && blockIdx.x == 0 && threadIdx.x == 0) atomicOr(flag, 1u);
  return bad;
}

struct __align__(16) LevelState {
  uint32_t L, nf, prev_nf, dir, rep, q, b, stop, ecc, solo, bm, deep, ul;
  uint32_t push_levels, pull_levels, reached;
  uint32_t qn, n_hp;            // queue entries of frontier L; static heavy pieces
  uint32_t qe;                  // queue edges of frontier L
  uint32_t big;                 // frontier L (bitmap form) has a row of > kDirectRow arcs
  uint32_t novis;               // candidate push without the visited-word read (see push_item)
  unsigned long long mf, explored, push_edges, pad;
  uint32_t *drow;               // this search's distance row
};
static_assert(sizeof(LevelState) % 16 == 0, "LevelState is copied as uint4");

struct WarpStage {
  uint32_t u[64], rs[64], d[64];
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Per-warp phase cycle accounting (trace builds only): lane 0 adds its warp's cycles to a
// per-CTA shared accumulator; trace_done folds it into the level's record (4 atomics per CTA).
__device__ unsigned long long *phase_smem() {
  __shared__ unsigned long long acc[4];
  return acc;
}
__device__ __forceinline__ void phase_add(const SsspParams &p, uint32_t L, int ph,
                                          long long &t0) {
  if (p.trace) {
    const long long t = clock64();
#if DAWN_TRACE_MAX  // per-phase maximum over the warps (stragglers) instead of the sum
    if (lane_id() == 0 && L < kTraceCap) atomicMax(phase_smem() + ph, (unsigned long long)(t - t0));
#else
    if (lane_id() == 0 && L < kTraceCap) atomicAdd(phase_smem() + ph, (unsigned long long)(t - t0));
#endif
    t0 = t;
  }
}

// Flush the first k (<= 32) staged entries to queue q: one 64-bit atomic reserves k slots AND
// their edge range; entry i gets (row start, exclusive edge offset) and the chunk map Cf gets
// the entry for every chunk boundary inside its row.  Warp-collective.
// Write the first k staged entries at the packed queue position `old` = (slot << 32) | edge
// offset, reserved by the caller.  Warp-collective.
__device__ __forceinline__ void stage_write(const SsspParams &p, int q, WarpStage &stg,
                                            uint32_t k, unsigned long long old) {
  const uint32_t lane = lane_id();
  const uint32_t d = lane < k ? stg.d[lane] : 0u;
  const uint32_t incl = warp_incl_scan(d);
  const uint32_t i = (uint32_t)(old >> 32) + lane;
  const uint32_t o = (uint32_t)old + incl - d;
  if (lane < k) {
    p.Lv[q][i] = stg.u[lane];
    p.Lsd[q][i] = make_uint2(stg.rs[lane], o);
  }
  // chunk map: entry i owns chunks [ceil(o/C), ceil((o+d)/C)).  Rows with many chunks (hubs:
  // 12K chunks for a 400K-arc row) are filled by the whole warp with coalesced stores, one row
  // at a time; short rows lane-serially in parallel.
  const uint32_t c0 = (o + kChunk - 1) / kChunk;
  const uint32_t nc = (lane < k) ? (o + d + kChunk - 1) / kChunk - c0 : 0u;
  const bool big = nc > 8;
  if (!big)
    for (uint32_t x = 0; x < nc; ++x) p.Cf[q][c0 + x] = i;
  uint32_t bm = __ballot_sync(DAWN_FULL, big);
  while (bm) {
    const uint32_t kk = __ffs(bm) - 1;
    bm &= bm - 1;
    const uint32_t cb = __shfl_sync(DAWN_FULL, c0, kk), nb = __shfl_sync(DAWN_FULL, nc, kk);
    const uint32_t ik = __shfl_sync(DAWN_FULL, i, kk);
    for (uint32_t x = lane; x < nb; x += 32) p.Cf[q][cb + x] = ik;
  }
  __syncwarp();
}

__device__ __forceinline__ void stage_emit(const SsspParams &p, Slot *s, int q, WarpStage &stg,
                                           uint32_t k) {
  const uint32_t lane = lane_id();
  const uint32_t D = warp_sum(lane < k ? stg.d[lane] : 0u);
  unsigned long long old = 0;
  if (lane == 0) old = atomicAdd(&s->qpack, ((unsigned long long)k << 32) | D);
  stage_write(p, q, stg, k, __shfl_sync(DAWN_FULL, old, 0));
}

// End-of-level flush of every warp's leftover stage (< 32 entries) with ONE atomic per CTA
// (a per-warp atomic here serialised ~4.7K same-address atomics: 7.6 us per level).
// CTA-collective: every thread of the CTA must call it.
__device__ __forceinline__ void cta_flush(const SsspParams &p, Slot *s, int q, WarpStage &stg,
                                          uint32_t cnt, unsigned long long *sm) {
  const uint32_t lane = lane_id(), w = threadIdx.x / 32, nw = blockDim.x / 32;
  const uint32_t D = warp_sum(lane < cnt ? stg.d[lane] : 0u);
  if (lane == 0) sm[w] = ((unsigned long long)cnt << 32) | D;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long run = 0;
    for (uint32_t i = 0; i < nw; ++i) {
      const unsigned long long x = sm[i];
      sm[i] = run;
      run += x;
    }
    sm[nw] = run ? atomicAdd(&s->qpack, run) : 0ull;
  }
  __syncthreads();
  if (cnt) stage_write(p, q, stg, cnt, sm[nw] + sm[w]);
  __syncthreads();
}

// Warp-collective append of discovered vertices (has: lane discovered u, row start rs,
// out-degree d) through the warp's shared-memory stage; 32 entries per global atomic.
// Vertices with out-degree 0 are not enqueued ("skipping ... reachable nodes
// with an out-degree of 0").
__device__ __forceinline__ void enqueue_frontier(const SsspParams &p, Slot *s, int q, bool has,
                                                 uint32_t u, uint32_t rs, uint32_t d,
                                                 WarpStage &stg, uint32_t &cnt) {
  const uint32_t lane = lane_id();
  const bool put = has && d > 0;
  const uint32_t mk = __ballot_sync(DAWN_FULL, put);
  if (!mk) return;
  if (put) {
    const uint32_t pos = cnt + __popc(mk & lanemask_lt());
    stg.u[pos] = u;
    stg.rs[pos] = rs;
    stg.d[pos] = d;
  }
  cnt += __popc(mk);
  __syncwarp();
  if (cnt >= 32) {
    stage_emit(p, s, q, stg, 32);
    const uint32_t rem = cnt - 32;
    if (lane < rem) {
      stg.u[lane] = stg.u[32 + lane];
      stg.rs[lane] = stg.rs[32 + lane];
      stg.d[lane] = stg.d[32 + lane];
    }
    __syncwarp();
    cnt = rem;
  }
}


// Push-mode visit of arc (frontier vertex) -> u, warp-collective (all lanes call; `act`
// false for idle lanes).
// One push level over the queue.  Chunk c = edges [32c, 32c+32) of the frontier; a warp item
// is J consecutive chunks (J = kIlp when the frontier has enough edges to keep every warp busy,
// else 1), processed with all J chains' loads in flight together (memory-level parallelism):
// Cf[c] -> 32-entry window of (row start, edge offset) -> owner by 5-step shfl search -> col ->
// vis test-and-set -> rp of the discovered vertex.
template <int J, bool CAND, bool NOVIS = false>
__device__ __forceinline__ void push_item(const SsspParams &p, const LevelState &st, Slot *ns,
                                          uint32_t item, uint32_t &n_new,
                                          unsigned long long &m_new, WarpStage &stg,
                                          uint32_t &cnt) {
  const int q = st.q, qn = q ^ 1;
  const uint32_t lane = lane_id();
  const uint32_t L1 = st.L + 1;
  const uint32_t E = st.qe, cntq = st.qn;
  uint32_t w0[J], u[J], rsd[J], dd[J];
  bool act[J], disc[J];
  uint2 sd[J];
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const uint32_t c = item * J + j;
    w0[j] = (c * kChunk < E) ? ld_cg(p.Cf[q] + c) : 0u;
  }
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const uint32_t idx = w0[j] + lane;
    sd[j] = (idx < cntq) ? ld_cg2(p.Lsd[q] + idx) : make_uint2(0u, 0xffffffffu);
  }
#pragma unroll
  for (int j = 0; j < J; ++j) {
    const uint32_t t = (item * J + j) * kChunk + lane;
    uint32_t k = 0;
#pragma unroll
    for (uint32_t step = 16; step; step >>= 1) {
      const uint32_t e = __shfl_sync(DAWN_FULL, sd[j].y, k + step);
      if (e <= t) k += step;
    }
    const uint32_t ok = __shfl_sync(DAWN_FULL, sd[j].y, k);
    const uint32_t sk = __shfl_sync(DAWN_FULL, sd[j].x, k);
    act[j] = t < E;
    u[j] = act[j] ? (uint32_t)ld_nc(p.col + sk + (t - ok)) : 0u;
  }
  uint32_t cur[J];
  // candidate levels while few vertices are settled (st.novis): most targets are unvisited, so
  // the visited-word read (one random L2 sector per arc) is skipped; cand_filter drops the rest
#pragma unroll
  for (int j = 0; j < J; ++j)
    cur[j] = (act[j] && !NOVIS) ? p.vis[u[j] >> 5] : (act[j] ? 0u : ~0u);  // weak: stale 0 = atomic
  if constexpr (CAND) {
    // bitmap push: mark the candidate, settle later in cand_filter (no returning atomic)
#if DAWN_CAND_FILTER
    // skip targets already marked by an earlier arc of this level (a stale read only costs a
    // redundant reduction)
#pragma unroll
    for (int j = 0; j < J; ++j)
      if (act[j] && !(cur[j] & (1u << (u[j] & 31))))
        cur[j] |= (DAWN_CAND_FILTER == 2) ? ld_cg(p.cand + (u[j] >> 5)) : p.cand[u[j] >> 5];
#endif
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const uint32_t bit = 1u << (u[j] & 31);
      if (!(cur[j] & bit)) red_or(p.cand + (u[j] >> 5), bit);
    }
  } else {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const uint32_t bit = 1u << (u[j] & 31);
      disc[j] = false;
      if (!(cur[j] & bit)) disc[j] = !(atomicOr(p.vis + (u[j] >> 5), bit) & bit);
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      rsd[j] = 0;
      dd[j] = 0;
      if (disc[j]) {
        rsd[j] = ld_nc(p.rp + u[j]);
        dd[j] = ld_nc(p.rp + u[j] + 1);
      }
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (disc[j]) {
        dd[j] -= rsd[j];
        DIST_ST(u[j], L1);
        n_new += 1;
        m_new += dd[j];
      }
      enqueue_frontier(p, ns, qn, disc[j], u[j], rsd[j], dd[j], stg, cnt);
    }
  }
}

// NV: the candidate push may skip the visited read (st.novis).  Only in the 1-CTA/SM kernel: the
// extra instantiation makes the 64-register kernel spill, and a kernel with a stack frame
// running concurrently with other cooperative launches (batch lanes) faulted or hung
// intermittently on B200; every cooperative kernel is kept at 0 bytes of stack.
template <bool NV>
__device__ void push_level(const SsspParams &p, const LevelState &st, Slot *ns, uint32_t gwarp,
                           uint32_t nwarps, uint32_t &n_new, unsigned long long &m_new,
                           WarpStage &stg, long long &t0, unsigned long long *fsm) {
  const uint32_t E = st.qe;
  const uint32_t nchunks = (E + kChunk - 1) / kChunk;
  uint32_t cnt = 0;
  if (st.bm) {
    // candidate mode keeps less state per chain: deeper ILP (8 chunks per item) once there are
    // enough chunks to give every warp an item, else 4 (all warps busy on the first bitmap
    // levels: C2 +1.5%)
    if (nchunks >= nwarps * DAWN_ILP_CAND) {
      constexpr int JB = DAWN_ILP_CAND;
      const uint32_t items = (nchunks + JB - 1) / JB;
      if (NV && DAWN_NOVIS && st.novis) {
        for (uint32_t it = gwarp; it < items; it += nwarps)
          push_item<JB, true, true>(p, st, ns, it, n_new, m_new, stg, cnt);
      } else if (!NV && DAWN_NOVIS && DAWN_NOVIS2 && st.novis) {
        // 64-register kernel: half the chunks per item keeps the extra instantiation spill-free
        constexpr int JH = JB / 2;
        const uint32_t items2 = (nchunks + JH - 1) / JH;
        for (uint32_t it = gwarp; it < items2; it += nwarps)
          push_item<JH, true, true>(p, st, ns, it, n_new, m_new, stg, cnt);
      } else {
        for (uint32_t it = gwarp; it < items; it += nwarps)
          push_item<JB, true>(p, st, ns, it, n_new, m_new, stg, cnt);
      }
    } else {
      constexpr int JB = DAWN_ILP_CAND / 2;
      const uint32_t items = (nchunks + JB - 1) / JB;
      for (uint32_t it = gwarp; it < items; it += nwarps)
        push_item<JB, true>(p, st, ns, it, n_new, m_new, stg, cnt);
    }
    phase_add(p, st.L, 0, t0);
    return;
  }
  if (nchunks >= nwarps * kIlp) {
    const uint32_t items = (nchunks + kIlp - 1) / kIlp;
    for (uint32_t it = gwarp; it < items; it += nwarps)
      push_item<kIlp, false>(p, st, ns, it, n_new, m_new, stg, cnt);
  } else {
    for (uint32_t it = gwarp; it < nchunks; it += nwarps)
      push_item<1, false>(p, st, ns, it, n_new, m_new, stg, cnt);
  }
  phase_add(p, st.L, 0, t0);
  cta_flush(p, ns, st.q ^ 1, stg, cnt, fsm);
  phase_add(p, st.L, 2, t0);
}

// Push level straight from the frontier bitmap fb[b] (the frontier a pull or candidate level
// left), for frontiers whose rows all have <= kDirectRow arcs (tracked by the levels that build
// bitmap frontiers): no bitmap -> queue conversion and no grid barrier before the expansion.  A
// warp takes 32 bitmap words (strided over the grid); each round, every lane contributes the next
// frontier vertex of its word and the round's rows are dealt 32 arcs at a time by the owner
// search of push_item.
__device__ void push_bitmap(const SsspParams &p, const LevelState &st, Slot *ns, uint32_t gwarp,
                            uint32_t nwarps, uint32_t &n_new, unsigned long long &m_new,
                            WarpStage &stg, long long &t0, unsigned long long *fsm) {
  const uint32_t lane = lane_id();
  const uint32_t L1 = st.L + 1;
  const int qn = st.q ^ 1;
  const uint32_t *fb = p.fb[st.b];
  uint32_t cnt = 0;
  // lane l of warp g reads word g + l * nwarps: every warp of the grid gets a share (32
  // consecutive words per warp left most warps without any on a 2^20-vertex graph)
  for (uint32_t base = gwarp; base < p.nwords; base += nwarps * 32) {
    const uint32_t w = base + lane * nwarps;
    uint32_t bits = (w < p.nwords) ? ld_cg(fb + w) : 0u;
    while (__ballot_sync(DAWN_FULL, bits != 0)) {
      uint32_t rs = 0, d = 0;
      if (bits) {
        const uint32_t v = w * 32 + (__ffs(bits) - 1);
        bits &= bits - 1;
        rs = ld_nc(p.rp + v);
        d = ld_nc(p.rp + v + 1) - rs;
      }
      const uint32_t incl = warp_incl_scan(d);
      const uint32_t total = __shfl_sync(DAWN_FULL, incl, 31);
      const uint32_t excl = incl - d;
      for (uint32_t r0 = 0; r0 < total; r0 += 32) {
        const uint32_t t = r0 + lane;
        uint32_t k = 0;
#pragma unroll
        for (uint32_t step = 16; step; step >>= 1) {
          const uint32_t e = __shfl_sync(DAWN_FULL, excl, k + step);
          if (e <= t) k += step;
        }
        const uint32_t ek = __shfl_sync(DAWN_FULL, excl, k);
        const uint32_t sk = __shfl_sync(DAWN_FULL, rs, k);
        const bool act = t < total;
        const uint32_t u = act ? (uint32_t)ld_nc(p.col + sk + (t - ek)) : 0u;
        bool disc = false;
        if (act) {
          const uint32_t bit = 1u << (u & 31);
          if (!(p.vis[u >> 5] & bit)) disc = !(atomicOr(p.vis + (u >> 5), bit) & bit);
        }
        uint32_t urs = 0, ud = 0;
        if (disc) {
          urs = ld_nc(p.rp + u);
          ud = ld_nc(p.rp + u + 1) - urs;
          DIST_ST(u, L1);
          n_new += 1;
          m_new += ud;
        }
        enqueue_frontier(p, ns, qn, disc, u, urs, ud, stg, cnt);
      }
    }
  }
  phase_add(p, st.L, 0, t0);
  cta_flush(p, ns, qn, stg, cnt, fsm);
  phase_add(p, st.L, 2, t0);
}

__device__ __forceinline__ bool fb_test(const uint32_t *fb, uint32_t v) {
  return (fb[v >> 5] >> (v & 31)) & 1u;
}

// PART: 0 the whole level; 1 the light pass only (heavy vertices it settles are claimed with a
// fire-and-forget reduction: the pieces run after a grid barrier and skip settled vertices);
// 2 the heavy pieces only
template <int PR, int J, int PART = 0>  // in-edges probed per lane per round trip (8 when the
                                        // frontier is sparse); J unreached vertices per lane
__device__ void pull_level(const SsspParams &p, const LevelState &st, uint32_t gwarp,
                           uint32_t nwarps, uint32_t &n_new, unsigned long long &m_new,
                           unsigned long long &examined, long long &t0, bool &bigf) {
  const uint32_t lane = lane_id();
  const uint32_t L1 = st.L + 1;
  const uint32_t *fcur = p.fb[st.b];
  uint32_t *fnext = p.fb[(st.b + 1) % 3];
  uint32_t *fclr = p.fb[(st.b + 2) % 3];  // held frontier L-1: cleared for level L+1
  if constexpr (PART != 2) {
  // (0) clear the bitmap of frontier L-1 (becomes the write target of level L+1)
  for (uint32_t w = gwarp * 32 + lane; w < p.nwords; w += nwarps * 32) fclr[w] = 0;
  // (1) unreached vertices, one lane each, from the warp's segment of the unreached list:
  //     the static ascending list of vertices with an in-edge at the first pull level, the
  //     warp's in-place compacted survivors afterwards (order kept, so vis / irp / dist
  //     accesses of a warp stay coalesced).  J entries per lane in flight.
  const uint32_t cap = (p.n_hasin + nwarps - 1) / nwarps;
  const uint32_t seg0 = gwarp * cap;
  const uint32_t *src = (st.ul ? p.ulist : p.hasin) + seg0;
  uint32_t *dst = p.ulist + seg0;
  const uint32_t cnt = st.ul ? ld_cg(p.useg + gwarp)
                             : (seg0 < p.n_hasin ? min(cap, p.n_hasin - seg0) : 0u);
  uint32_t wr = 0;
#if DAWN_PULL_PREFETCH
  // the next iteration's list entries are loaded one iteration ahead (the in-place compaction
  // only writes positions below the current iteration's end, so the read-ahead is never stale)
  uint32_t un[J];
#pragma unroll
  for (int j = 0; j < J; ++j) un[j] = (j * 32 + lane < cnt) ? ld_cg(src + j * 32 + lane) : 0xffffffffu;
#endif
  for (uint32_t ib = 0; ib < cnt; ib += 32 * J) {
    uint32_t u[J], s[J], e[J], j0[J], ef[J], t1[J];
    bool need[J], found[J], hvy[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
#if DAWN_PULL_PREFETCH
      u[j] = un[j];
      const uint32_t i = ib + 32 * J + j * 32 + lane;
      un[j] = i < cnt ? ld_cg(src + i) : 0xffffffffu;
#else
      const uint32_t i = ib + j * 32 + lane;
      u[j] = i < cnt ? ld_cg(src + i) : 0xffffffffu;
#endif
      found[j] = false;
      need[j] = false;
      hvy[j] = false;
      s[j] = e[j] = 0;
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (u[j] != 0xffffffffu) {
        const uint32_t bit = 1u << (u[j] & 31);
        need[j] = !(ld_cg(p.vis + (u[j] >> 5)) & bit);   // settled by a push level since
        hvy[j] = ld_nc(p.hin_bits + (u[j] >> 5)) & bit;
        s[j] = ld_nc(p.irp + u[j]);                       // speculative, same round trip
        e[j] = ld_nc(p.irp + u[j] + 1);
        t1[j] = p.top1 ? ld_nc(p.top1 + u[j]) : 0xffffffffu;  // the row's first entry, ditto
      }
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (!need[j]) e[j] = s[j];
      j0[j] = s[j];
      if (p.top1 && e[j] > s[j]) {
        // the first probe from the per-vertex copy: a hit settles the vertex without a sector
        // of its in-row (the sweep is then bounded by the row offsets, not the in-rows)
        found[j] = fb_test(fcur, t1[j]);
        j0[j] = s[j] + 1;
      }
      // heavy rows (in-degree > kHeavy): only the first kHeavyProbe in-edges here; the
      // static pieces finish the rows still unsettled
      ef[j] = hvy[j] ? min(e[j], s[j] + kHeavyProbe) : e[j];
    }
    for (;;) {
      bool any = false;
      uint32_t v[J][PR];
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const bool go = need[j] && !found[j] && j0[j] < ef[j];
        any |= go;
#pragma unroll
        for (int i = 0; i < PR; ++i)
          v[j][i] = (go && j0[j] + i < ef[j]) ? (uint32_t)ld_nc(p.icol + j0[j] + i) : 0xffffffffu;
      }
      if (!any) break;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        if (v[j][0] == 0xffffffffu) continue;
        uint32_t hit = PR;
#pragma unroll
        for (int i = PR - 1; i >= 0; --i)
          if (v[j][i] != 0xffffffffu && fb_test(fcur, v[j][i])) hit = i;
        if (hit < PR) {
          found[j] = true;
          j0[j] += hit + 1;
        } else {
          j0[j] += PR;
        }
      }
    }
    if constexpr (PART == 1 && DAWN_PULL_HLIST) {
      // heavy rows the first kHeavyProbe probes did not settle: listed for the pieces phase
      // (the free queue buffer Lv[q^1] holds them: at most one entry per unreached vertex)
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const bool left = hvy[j] && need[j] && !found[j];
        const uint32_t lm = __ballot_sync(DAWN_FULL, left);
        if (lm) {
          uint32_t base = 0;
          if (lane == 0) base = atomicAdd(&p.ctrl->hl_cnt[st.L & 1], (uint32_t)__popc(lm));
          base = __shfl_sync(DAWN_FULL, base, 0);
          if (left) p.Lv[st.q ^ 1][base + __popc(lm & lanemask_lt())] = u[j];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
      if (need[j]) examined += min(j0[j], ef[j]) - s[j];
      if (found[j]) {
        const uint32_t w = u[j] >> 5, bit = 1u << (u[j] & 31);
        if (hvy[j] && PART == 0) {
          // a heavy row may be settled concurrently by one of its static pieces: claim with a
          // returning atomic so each vertex is counted exactly once
          if (atomicOr(p.vis + w, bit) & bit) found[j] = false;
        } else {
          red_or(p.vis + w, bit);
        }
      }
      if (found[j]) {
        red_or(fnext + (u[j] >> 5), 1u << (u[j] & 31));
        DIST_ST(u[j], L1);
        n_new += 1;
        const uint32_t dg = p.sym ? (e[j] - s[j]) : (ld_nc(p.rp + u[j] + 1) - ld_nc(p.rp + u[j]));
        m_new += dg;
        bigf |= dg > kDirectRow;  // a long row in the frontier (CTA-reduced by the caller)
      }
      // survivors (still unreached) stay in the warp's segment, order preserved
      const bool keep = need[j] && !found[j];
      const uint32_t km = __ballot_sync(DAWN_FULL, keep);
      if (keep) dst[wr + __popc(km & lanemask_lt())] = u[j];
      wr += __popc(km);
    }
  }
  if (lane == 0) p.useg[gwarp] = wr;
  phase_add(p, st.L, 0, t0);
  }  // PART != 2
  if constexpr (PART == 1) return;
  if constexpr (PART == 2 && DAWN_PULL_HLIST) {
    // (2') the heavy rows the light pass left (listed, one warp each, in-edges from the first
    //      unprobed one, 32 per round trip, early exit); each listed vertex is unique and only
    //      this phase can settle it now, so the claim needs no returning atomic
    const uint32_t cnt = ld_cg(&p.ctrl->hl_cnt[st.L & 1]);
    const uint32_t *hl = p.Lv[st.q ^ 1];
    for (uint32_t i = gwarp; i < cnt; i += nwarps) {
      const uint32_t uk = ld_cg(hl + i);
      if ((ld_cg(p.vis + (uk >> 5)) >> (uk & 31)) & 1u) continue;  // (defensive: settled)
      const uint32_t sk = ld_nc(p.irp + uk) + kHeavyProbe, ek = ld_nc(p.irp + uk + 1);
      for (uint32_t j = sk; j < ek; j += 32) {
        const uint32_t jj = j + lane;
        const bool hit = jj < ek && fb_test(fcur, (uint32_t)ld_nc(p.icol + jj));
        const uint32_t hm = __ballot_sync(DAWN_FULL, hit);
        if (hm) {
          if (lane == 0) {
            examined += (j - sk) + __ffs(hm);
            const uint32_t w = uk >> 5, bit = 1u << (uk & 31);
            red_or(p.vis + w, bit);
            red_or(fnext + w, bit);
            DIST_ST(uk, L1);
            n_new += 1;
            const uint32_t dg = p.sym ? (ek - (sk - kHeavyProbe))
                                      : (ld_nc(p.rp + uk + 1) - ld_nc(p.rp + uk));
            m_new += dg;
            bigf |= dg > kDirectRow;
          }
          break;
        }
        if (j + 32 >= ek && lane == 0) examined += ek - sk;
      }
    }
    phase_add(p, st.L, 1, t0);
    return;
  }
  // (2) heavy rows: static pieces; 32 pieces tested per warp (vis), then a warp scans each
  //     live piece 32 in-edges per round trip
  // every warp gets an equal consecutive share of the piece list (a 32-piece stride left most
  // warps idle and the rest with up to 32 live pieces each: the level's straggler)
  const uint32_t per = (st.n_hp + nwarps - 1) / nwarps;
  const uint32_t pe = min(st.n_hp, (gwarp + 1) * per);
  for (uint32_t pb = gwarp * per; pb < pe; pb += 32) {
    const uint32_t pc = pb + lane;
    uint32_t u = 0, s = 0, e = 0;
    bool need = false;
    if (pc < pe) {
      u = ld_nc(p.hin_v + pc);
      s = ld_nc(p.hin_s + pc);
      e = ld_nc(p.hin_e + pc);
      need = !((ld_cg(p.vis + (u >> 5)) >> (u & 31)) & 1u);
    }
    uint32_t nm = __ballot_sync(DAWN_FULL, need);
    while (nm) {
      const uint32_t k = __ffs(nm) - 1;
      nm &= nm - 1;
      const uint32_t uk = __shfl_sync(DAWN_FULL, u, k);
      const uint32_t sk = __shfl_sync(DAWN_FULL, s, k);
      const uint32_t ek = __shfl_sync(DAWN_FULL, e, k);
      const uint32_t w = uk >> 5, bit = 1u << (uk & 31);
      // kHW in-edges per lane in flight: a whole 256-arc piece per round trip
      constexpr uint32_t kHW = DAWN_HEAVY_ILP;
      for (uint32_t j = sk; j < ek; j += 32 * kHW) {
        uint32_t v[kHW];
#pragma unroll
        for (uint32_t i = 0; i < kHW; ++i) {
          const uint32_t jj = j + i * 32 + lane;
          v[i] = jj < ek ? (uint32_t)ld_nc(p.icol + jj) : 0xffffffffu;
        }
        uint32_t first = 0xffffffffu;  // first round (i) with a hit in this lane
#pragma unroll
        for (int i = (int)kHW - 1; i >= 0; --i)
          if (v[i] != 0xffffffffu && fb_test(fcur, v[i])) first = (uint32_t)i;
        const uint32_t hm = __ballot_sync(DAWN_FULL, first != 0xffffffffu);
        if (hm) {
          const uint32_t fmin = __reduce_min_sync(DAWN_FULL, first);
          const uint32_t hm2 = __ballot_sync(DAWN_FULL, first == fmin);
          if (lane == 0) {
            examined += fmin * 32 + __ffs(hm2);
            const uint32_t old = atomicOr(p.vis + w, bit);
            if (!(old & bit)) {
              red_or(fnext + w, bit);
              DIST_ST(uk, L1);
              n_new += 1;
              const uint32_t dg = p.sym ? (ld_nc(p.irp + uk + 1) - ld_nc(p.irp + uk))
                                        : (ld_nc(p.rp + uk + 1) - ld_nc(p.rp + uk));
              m_new += dg;
              bigf |= dg > kDirectRow;
            }
          }
          break;
        }
        if (lane == 0) examined += min(32u * kHW, ek - j);
        if (ld_cg(p.vis + w) & bit) break;  // settled meanwhile by another piece
      }
    }
  }
  phase_add(p, st.L, 1, t0);
}

// Second half of a bitmap-push level: word owners settle the candidates (new = cand & ~vis),
// write the frontier bitmap fb[b+1] (every word), clear fb[b+2] and cand, set dist = L+1.
// 32 words per warp iteration (one lane each), then lane-per-vertex for words with news.
__device__ void cand_filter(const SsspParams &p, const LevelState &st, uint32_t gwarp,
                            uint32_t nwarps, uint32_t &n_new, unsigned long long &m_new,
                            bool &bigf) {
  const uint32_t lane = lane_id();
  const uint32_t L1 = st.L + 1;
  uint32_t *fnext = p.fb[(st.b + 1) % 3];
  uint32_t *fclr = p.fb[(st.b + 2) % 3];
  for (uint32_t base = gwarp * 32; base < p.nwords; base += nwarps * 32) {
    const uint32_t w = base + lane;
    uint32_t nw = 0;
    if (w < p.nwords) {
      const uint32_t c = ld_cg(p.cand + w);
      if (c) {
        const uint32_t vw = ld_cg(p.vis + w);
        nw = c & ~vw;
        p.cand[w] = 0;
        if (nw) p.vis[w] = vw | nw;
      }
      fnext[w] = nw;
      fclr[w] = 0;
    }
    // lane-parallel over this lane's word: up to 4 new vertices per round trip
    uint32_t bits = nw;
    while (bits) {
      uint32_t u[4], a[4], b[4];
      int k = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        u[i] = 0xffffffffu;
        if (bits) {
          u[i] = w * 32 + (__ffs(bits) - 1);
          bits &= bits - 1;
          k = i + 1;
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < k) {
          a[i] = ld_nc(p.rp + u[i]);
          b[i] = ld_nc(p.rp + u[i] + 1);
          DIST_ST(u[i], L1);
        }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < k) {
          m_new += b[i] - a[i];
          bigf |= b[i] - a[i] > kDirectRow;
        }
      n_new += k;
    }
  }
}

// Block-wide sum of two counters, then one global atomic per CTA.
__device__ __forceinline__ void block_flush(uint32_t a, unsigned long long b, uint32_t *ga,
                                            unsigned long long *gb, unsigned long long *sm) {
  a = warp_sum(a);
  b = warp_sum(b);
  if (threadIdx.x == 0) { sm[0] = 0; sm[1] = 0; }
  __syncthreads();
  if (lane_id() == 0 && (a | b)) {
    atomicAdd(&sm[0], (unsigned long long)a);
    atomicAdd(&sm[1], b);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (sm[0] && ga) atomicAdd(ga, (uint32_t)sm[0]);
    if (sm[1] && gb) atomicAdd(gb, sm[1]);
  }
}

// Level header (thread 0 of every CTA; identical inputs -> identical decisions everywhere):
// read frontier L's counters, apply the stop tests (a5) and choose the direction (a4).
__device__ __forceinline__ void level_header(const SsspParams &p, Ctrl *C, LevelState &st,
                                             uint32_t max_reach, uint32_t nblocks) {
  const Slot *cs = &C->slot[st.L % 3];
  st.nf = ld_cg(&cs->n_new);
  st.mf = ld_cg(&cs->m_new);
  const unsigned long long qp = ld_cg(&cs->qpack);
  st.qn = (uint32_t)(qp >> 32);
  st.qe = (uint32_t)qp;
  st.big = ld_cg(&cs->big);
  if (blockIdx.x == 0) {
    C->slot[(st.L + 2) % 3] = Slot{0, 0, 0, 0, 0};
    C->hl_cnt[(st.L + 1) & 1] = 0;  // last used at level L-1, next at level L+1
  }
  if (st.L > 0) st.reached += st.nf;
  st.explored += st.mf;
  st.stop = 0;
  st.solo = 0;
  if (st.nf == 0) {
    st.stop = 1;
    st.ecc = st.L - 1;
  } else if (st.reached + 1 >= max_reach || st.L + 1 >= p.n) {
    st.stop = 1;  // condition 1: nothing left to discover
    st.ecc = st.L;
  } else {
    if (p.variant == DAWN_PUSH || !p.can_pull) {
      st.dir = kPush;
    } else if (p.variant == DAWN_PULL) {
      st.dir = kPull;
    } else {
      // push costs ~ m_f edge visits; a pull sweep costs ~ n_u scans of expected length
      // min(deg, m_u / m_f) (early exit once a frontier in-neighbour is met), so pull wins once
      // alpha * m_f^2 > n_u * m_u.  (Beamer's linear m_f > m_u / alpha, cited by the paper at
      // L123, picked the slower direction at Kronecker-20 L2 or Kronecker-24 L2 for any alpha.)
      const double mu = (double)(p.m - st.explored);
      const double nu = (double)(max_reach - 1 - min(st.reached, max_reach - 1));
      if (st.dir == kPush) {
        if ((double)st.mf * (double)st.mf * p.alpha > nu * mu && st.nf > st.prev_nf) st.dir = kPull;
      } else {
        if ((double)st.nf * p.beta < (double)p.n && st.nf < st.prev_nf) st.dir = kPush;
      }
    }
    const bool grows = st.nf > st.prev_nf;
    st.prev_nf = st.nf;
    st.solo = (nblocks > 1 && st.dir == kPush && st.rep == kRepQueue && st.qe <= p.solo_e) ? 1u : 0u;
    // bitmap push (candidates + word-owner filter, the next frontier as a bitmap): wide levels,
    // and growing ones from bmpush_grow arcs up — a growing frontier usually turns to pull next,
    // which wants the bitmap and no queue (C2 +3%); a shrinking one keeps the queue
    st.bm = (st.dir == kPush && !st.solo &&
             st.mf >= (grows ? (unsigned long long)p.bmpush_grow : (unsigned long long)p.bmpush_e))
                ? 1u : 0u;
    st.novis = (st.bm && (unsigned long long)(st.reached + 1) * DAWN_NOVIS_FRAC < max_reach) ? 1u : 0u;
    // sparse frontier (a probe hits with probability ~ m_f / (m_f + m_u) < 1/6): probe 8
    // in-edges per round trip instead of 4
    st.deep = (st.dir == kPull && 6.0 * (double)st.mf < (double)(p.m - st.explored) + (double)st.mf)
                  ? 1u : 0u;
  }
  if (p.trace && blockIdx.x == 0 && st.L < kTraceCap) {
    TraceRec r;
    r.t_ns = globaltimer();
    r.level = st.L;
    r.dir = st.stop ? 2u : st.dir;
    r.nf = st.nf;
    r.pad = st.rep | (st.solo << 1) | (st.bm << 2);
    r.mf = st.mf;
    r.t_first = p.trace[st.L].t_first;
    r.t_last = p.trace[st.L].t_last;
    for (int k = 0; k < 4; ++k) r.cyc[k] = p.trace[st.L].cyc[k];
    p.trace[st.L] = r;
    C->trace_n = st.L + 1;
    if (st.L + 1 < kTraceCap - 1) {  // the next level's record (accumulated at its end)
      p.trace[st.L + 1].t_first = ~0ull;
      p.trace[st.L + 1].t_last = 0;
      for (int k = 0; k < 4; ++k) p.trace[st.L + 1].cyc[k] = 0;
    }
  }
}

// CTA-collective (every thread calls it after the level's work)
__device__ __forceinline__ void trace_done(const SsspParams &p, uint32_t L) {
  if (!p.trace) return;
  __syncthreads();
  if (threadIdx.x == 0 && L < kTraceCap) {
    const unsigned long long t = globaltimer();
    atomicMin(&p.trace[L].t_first, t);
    atomicMax(&p.trace[L].t_last, t);
    unsigned long long *a = phase_smem();
    for (int k = 0; k < 4; ++k) {
#if DAWN_TRACE_MAX
      if (a[k]) atomicMax(&p.trace[L].cyc[k], a[k]);
#else
      if (a[k]) atomicAdd(&p.trace[L].cyc[k], a[k]);
#endif
      a[k] = 0;
    }
  }
}

__device__ __forceinline__ void level_advance(LevelState &st) {
  if (st.dir == kPush && st.bm) {  // bitmap push: the next frontier is fb[b+1]
    st.push_levels++;
    st.push_edges += st.mf;
    st.b = (st.b + 1) % 3;
    st.rep = kRepBitmap;
  } else if (st.dir == kPush) {
    st.push_levels++;
    st.push_edges += st.mf;
    st.q ^= 1;
    st.rep = kRepQueue;
  } else {
    st.pull_levels++;
    st.b = (st.b + 1) % 3;
    st.rep = kRepBitmap;
    st.ul = 1;
  }
  st.L++;
}

// MINB = CTAs per SM the register allocation targets: 2 (64 registers, 296 CTAs) hides more
// latency on big graphs (Kronecker-24: 1196 vs 992 GTEPS); 1 (no spills, 148 CTAs, cheaper
// grid barriers and fewer same-address atomics) wins on small ones (Kronecker-20: 364 vs 352).
template <int NT, int MINB = DAWN_SSSP_MINB>
__global__ void __launch_bounds__(NT, MINB) k_sssp(SsspParams p) {
  __shared__ LevelState st;
  __shared__ unsigned long long red[2];
  __shared__ WarpStage stage[NT / 32];
  __shared__ unsigned long long fsm[NT / 32 + 1];
  static_assert(sizeof(LevelState) <= sizeof(((Ctrl *)0)->solo_state), "solo_state too small");
  const uint32_t nblocks = gridDim.x;
  const uint32_t gwarp = blockIdx.x * (NT / 32) + threadIdx.x / 32;
  const uint32_t nwarps = nblocks * (NT / 32);
  const uint32_t gtid = blockIdx.x * NT + threadIdx.x;
  const uint32_t nthreads = nblocks * NT;
  WarpStage &stg = stage[threadIdx.x / 32];
  Ctrl *C = p.ctrl;
  __shared__ unsigned long long bar_target;  // grid_sync's arrival target (thread 0's)
  if (threadIdx.x == 0) bar_target = 0;      // (shared: no register held across the levels)
  if (p.vn && sources_invalid<NT>(p.vsrc, p.vn, p.n, &C->bad_src)) return;
  const uint32_t nsrc = p.nsrc ? p.nsrc : 1u;
  // batch mode: the searches run back to back in this launch, a grid barrier apart (no kernel
  // boundary or launch ramp between them).  Dynamic lanes (p.claim): the batch index of the next
  // search is claimed when the current one ends and read by every CTA after a barrier (claiming
  // one ahead left lanes idle when a batch has about as many sources as lanes)
  __shared__ uint32_t next_sh;  // batch index of the next search (kept in shared memory)
  if (p.claim) {
    if (blockIdx.x == 0 && threadIdx.x == 0) C->next_idx = atomicAdd(p.claim, 1u);
    grid_sync(&C->bar, nblocks, bar_target);
    if (threadIdx.x == 0) next_sh = ld_cg(&C->next_idx);
  } else if (threadIdx.x == 0) {
    next_sh = 0;
  }
  __syncthreads();
  bool prefilled = false;  // this CTA's share of the next search's row already holds UNREACHED
  for (;;) {
  const uint32_t idx = next_sh;  // batch index of this search
  if (idx >= nsrc) break;
  __shared__ uint32_t cur_sh;  // the same, re-read at the search's end (no register held)
  if (threadIdx.x == 0) cur_sh = idx;
  const uint32_t src = p.nsrc ? ld_nc(p.sources + idx) : p.source;
  uint32_t *const drow = p.dist + (size_t)idx * p.n;
  // per-search scalars of thread 0 in shared memory (no registers held across the levels)
  __shared__ uint32_t solo_epoch, max_reach;
  if (threadIdx.x == 0) {
    solo_epoch = 0;
    // condition 1 bound: only vertices with an in-edge (plus s itself) can ever be reached
    max_reach = ld_cg(&C->n_hasin) + ((p.noin[src >> 5] >> (src & 31)) & 1u);
  }

  if (p.trace && gtid == 0) p.trace[kTraceCap - 1].t_ns = globaltimer();  // kernel timeline
  // ---- k_narrow ran first for this call: finished (nothing to do) or hand-over (resume)
  uint32_t narrow = 0;
  if (p.nsrc <= 1 && ld_acquire(&C->narrow_seq) == p.seq) narrow = ld_cg(&C->narrow_status);
  if (narrow == 1) return;
  if (narrow == 2) {
    if (threadIdx.x < 4) phase_smem()[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
      const uint4 *s4 = reinterpret_cast<const uint4 *>(C->solo_state);
      uint4 *d4 = reinterpret_cast<uint4 *>(&st);
      for (int i = 0; i < (int)(sizeof(LevelState) / 16); ++i) d4[i] = __ldcg(s4 + i);
      st.n_hp = ld_cg(&C->n_hp_in);
      st.drow = drow;
    }
    __syncthreads();
  }
  // ---- a1 init: dist <- UNREACHED (d(s) = 0), vis <- no-in-edge vertices | {s}  (Q4, Q7)
  if (narrow != 2) {
  if (!prefilled) {
    for (uint32_t i = gtid; i < p.n; i += nthreads) drow[i] = (i == src) ? 0u : kUnreached;
  } else if (gtid == src % nthreads) {
    drow[src] = 0u;  // this CTA's share was filled during the previous search's solo levels
  }
  prefilled = false;
  for (uint32_t w = gtid; w < p.nwords; w += nthreads)
    p.vis[w] = p.noin[w] | ((w == (src >> 5)) ? (1u << (src & 31)) : 0u);
  {
    // level-0 chunk map (every 32nd arc of s's row starts in entry 0), spread over the grid: a
    // hub source has up to ~10^4 chunks
    const uint32_t d0 = ld_nc(p.rp + src + 1) - ld_nc(p.rp + src);
    for (uint32_t c = gtid; c * kChunk < d0; c += nthreads) p.Cf[0][c] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) C->slot[i] = Slot{0, 0, 0, 0, 0};
    C->examined = 0;
    C->solo_epoch = 0;
    const uint32_t rs = p.rp[src], d = p.rp[src + 1] - rs;
    Slot &s0 = C->slot[0];
    s0.n_new = 1;
    s0.m_new = d;
    if (d > 0) {
      p.Lv[0][0] = src;
      p.Lsd[0][0] = make_uint2(rs, 0u);
      s0.qpack = (1ull << 32) | d;
    }
  }
  if (p.trace && gtid == 0) {  // record 0 (later records are reset by the previous header)
    p.trace[0].t_first = ~0ull;
    p.trace[0].t_last = 0;
    for (int k = 0; k < 4; ++k) p.trace[0].cyc[k] = 0;
  }
  if (threadIdx.x < 4) phase_smem()[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    st = LevelState{};
    st.dir = (p.variant == DAWN_PULL) ? kPull : kPush;
    st.n_hp = ld_cg(&C->n_hp_in);
    st.drow = drow;
  }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) C->hl_cnt[0] = C->hl_cnt[1] = 0;  // (also on resume)
  grid_sync(&C->bar, nblocks, bar_target);
  // the next search's index for the solo-stretch prefill: unknown (none) with dynamic lanes
  if (threadIdx.x == 0) next_sh = p.claim ? nsrc : cur_sh + 1;  // read after a sync
  if (p.trace && gtid == 0) p.trace[kTraceCap - 1].t_first = globaltimer();

  unsigned long long examined = 0;
  bool have_header = false;
  for (;;) {
    if (!have_header) {
      if (threadIdx.x == 0) level_header(p, C, st, max_reach, nblocks);
      __syncthreads();
    }
    have_header = false;
    if (st.stop) break;

    if (st.solo) {
      // ---- solo stretch: narrow push levels on CTA 0 with __syncthreads only
      if (blockIdx.x != 0) {
        __syncthreads();  // every thread has read st.stop / st.solo before thread 0 rewrites st
        const uint32_t nx = next_sh;  // the next search's batch index
        if ((MINB == 1 || DAWN_MINB2_EXTRAS) && nx < nsrc && !prefilled) {
          // idle while CTA 0 runs the narrow levels: initialise this CTA's share of the next
          // search's distance row (independent memory; its source entry is set at its init)
          uint32_t *nrow = p.dist + (size_t)nx * p.n;
          for (uint32_t i = gtid; i < p.n; i += nthreads) nrow[i] = kUnreached;
          prefilled = true;
        }
        if (threadIdx.x == 0) {
          ++solo_epoch;
          while (ld_acquire(&C->solo_epoch) < solo_epoch) {
          }
          fence_acq_rel_gpu();
          const uint4 *src4 = reinterpret_cast<const uint4 *>(C->solo_state);
          uint4 *dst4 = reinterpret_cast<uint4 *>(&st);
#pragma unroll
          for (int i = 0; i < (int)(sizeof(LevelState) / 16); ++i) dst4[i] = __ldcg(src4 + i);
        }
        __syncthreads();
        have_header = true;  // CTA 0 published the post-header state of this level
        continue;
      }
      const uint32_t lw = threadIdx.x / 32;
      for (;;) {
        Slot *ns = &C->slot[(st.L + 1) % 3];
        uint32_t n_new = 0;
        unsigned long long m_new = 0;
        long long t0 = clock64();
        push_level<MINB == 1>(p, st, ns, lw, NT / 32, n_new, m_new, stg, t0, fsm);
        block_flush(n_new, m_new, &ns->n_new, &ns->m_new, red);
        trace_done(p, st.L);
        __syncthreads();
        if (threadIdx.x == 0) {
          level_advance(st);
          level_header(p, C, st, max_reach, nblocks);
        }
        __syncthreads();
        if (st.stop || !st.solo) break;
      }
      if (threadIdx.x == 0) {
        const uint4 *src4 = reinterpret_cast<const uint4 *>(&st);
        uint4 *dst4 = reinterpret_cast<uint4 *>(C->solo_state);
#pragma unroll
        for (int i = 0; i < (int)(sizeof(LevelState) / 16); ++i) dst4[i] = src4[i];
        ++solo_epoch;
        st_release(&C->solo_epoch, solo_epoch);
      }
      have_header = true;
      continue;
    }

    long long tconv = clock64();
    // a push from a bitmap frontier without long rows expands the bitmap directly
    // (1-CTA/SM variant only: in the 64-register one the extra path costs spills, C4 -4%)
    constexpr bool kDirect = DAWN_DIRECT_PUSH && (MINB == 1 || DAWN_MINB2_EXTRAS);
    const bool direct = kDirect && st.dir == kPush && st.rep == kRepBitmap && !st.bm && !st.big;
    if (st.dir == kPull && st.rep == kRepQueue) {
      // queue -> frontier bitmap fb[b] (and a clean fb[b+1] for the pull to write)
      uint32_t *fb = p.fb[st.b];
      uint32_t *fn = p.fb[(st.b + 1) % 3];
      for (uint32_t w = gtid; w < p.nwords; w += nthreads) { fb[w] = 0; fn[w] = 0; }
      grid_sync(&C->bar, nblocks, bar_target);
      for (uint32_t i = gtid; i < st.qn; i += nthreads) {
        const uint32_t v = ld_cg(p.Lv[st.q] + i);
        red_or(fb + (v >> 5), 1u << (v & 31));
      }
      grid_sync(&C->bar, nblocks, bar_target);
      if (threadIdx.x == 0) st.rep = kRepBitmap;
    } else if (st.dir == kPush && st.rep == kRepBitmap && !direct) {
      // frontier bitmap fb[b] -> queue q (ballot/popc compaction), barrier
      Slot *cs = &C->slot[st.L % 3];
      const uint32_t *fb = p.fb[st.b];
      const uint32_t lane = lane_id();
      uint32_t cnt = 0;
      for (uint32_t base = gwarp * 32; base < p.nwords; base += nwarps * 32) {
        const uint32_t w = base + lane;
        uint32_t bits = (w < p.nwords) ? ld_cg(fb + w) : 0u;
        while (__ballot_sync(DAWN_FULL, bits != 0)) {
          const bool has = bits != 0;
          uint32_t u = 0, rs = 0, d = 0;
          if (has) {
            u = w * 32 + (__ffs(bits) - 1);
            bits &= bits - 1;
            rs = ld_nc(p.rp + u);
            d = ld_nc(p.rp + u + 1) - rs;
          }
          enqueue_frontier(p, cs, st.q, has, u, rs, d, stg, cnt);
        }
      }
      cta_flush(p, cs, st.q, stg, cnt, fsm);
      grid_sync(&C->bar, nblocks, bar_target);
      if (threadIdx.x == 0) {
        const unsigned long long qp = ld_cg(&cs->qpack);
        st.qn = (uint32_t)(qp >> 32);
        st.qe = (uint32_t)qp;
        st.rep = kRepQueue;
      }
      __syncthreads();
    }

    Slot *ns = &C->slot[(st.L + 1) % 3];
    uint32_t n_new = 0;
    unsigned long long m_new = 0;
    bool bigf = false;  // a bitmap frontier being built has a row of > kDirectRow arcs
    phase_add(p, st.L, 3, tconv);
    if (kDirect && direct) {
      push_bitmap(p, st, ns, gwarp, nwarps, n_new, m_new, stg, tconv, fsm);
    } else if (st.dir == kPush) {
      push_level<MINB == 1>(p, st, ns, gwarp, nwarps, n_new, m_new, stg, tconv, fsm);
      if (st.bm) {
        grid_sync(&C->bar, nblocks, bar_target);
        cand_filter(p, st, gwarp, nwarps, n_new, m_new, bigf);
        phase_add(p, st.L, 1, tconv);
      }
    } else {
      constexpr int kPrD = MINB == 1 ? DAWN_PULL_DEEP_PR : DAWN_PULL_DEEP_PR2;
      constexpr int kPr = MINB == 1 ? DAWN_PULL_PR : DAWN_PULL_PR2;
      constexpr int kJ = MINB == 1 ? DAWN_PULL_J : DAWN_PULL_J2;
      if constexpr (DAWN_PULL_SPLIT) {
        // light pass, grid barrier, heavy pieces: no returning claim in the light pass
        if (DAWN_PULL_DEEP && st.deep)
          pull_level<kPrD, kJ, 1>(p, st, gwarp, nwarps, n_new, m_new, examined, tconv, bigf);
        else
          pull_level<kPr, kJ, 1>(p, st, gwarp, nwarps, n_new, m_new, examined, tconv, bigf);
        grid_sync(&C->bar, nblocks, bar_target);
        pull_level<kPr, kJ, 2>(p, st, gwarp, nwarps, n_new, m_new, examined, tconv, bigf);
      } else {
        if (DAWN_PULL_DEEP && st.deep)
          pull_level<kPrD, kJ>(p, st, gwarp, nwarps, n_new, m_new, examined, tconv, bigf);
        else
          pull_level<kPr, kJ>(p, st, gwarp, nwarps, n_new, m_new, examined, tconv, bigf);
      }
    }
    block_flush(n_new, m_new, &ns->n_new, &ns->m_new, red);
    if constexpr (kDirect) {
      if (__syncthreads_or(bigf) && threadIdx.x == 0) ns->big = 1;  // one store per CTA at most
    }
    phase_add(p, st.L, 2, tconv);
    trace_done(p, st.L);
    grid_sync(&C->bar, nblocks, bar_target);
    if (threadIdx.x == 0) level_advance(st);
    __syncthreads();
  }

  if (p.trace && gtid == 0) p.trace[kTraceCap - 1].t_last = globaltimer();
  // ---- a7 statistics
  if (p.stats) {
    dawn_sssp_stats *const stats_out = p.stats + *(volatile uint32_t *)&cur_sh;
    block_flush(0u, examined, nullptr, &C->examined, red);
    grid_sync(&C->bar, nblocks, bar_target);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      dawn_sssp_stats s;
      s.levels = st.ecc;
      s.reached = st.reached;
      s.edges_reach = st.explored;
      s.edges_examined = st.push_edges + ld_cg(&C->examined);
      s.push_levels = st.push_levels;
      s.pull_levels = st.pull_levels;
      *stats_out = s;
    }
  }
  if (p.claim) {  // dynamic lanes: claim the next index now, publish it by a barrier
    if (blockIdx.x == 0 && threadIdx.x == 0) C->next_idx = atomicAdd(p.claim, 1u);
    grid_sync(&C->bar, nblocks, bar_target);
    if (threadIdx.x == 0) next_sh = ld_cg(&C->next_idx);
    __syncthreads();
  } else if (next_sh < nsrc) {
    grid_sync(&C->bar, nblocks, bar_target);  // before the next init
  }
  }  // sources
  grid_exit(&C->bar, nblocks);
}

}  // namespace dawn

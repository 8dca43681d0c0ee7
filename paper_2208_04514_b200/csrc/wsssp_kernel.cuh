// wsssp_kernel.cuh — weighted single-source shortest paths by (min,+) DAWN rounds (SURVEY §8(f)
// NEXT-4; "(min,+) operations ... to expand the applicability of DAWN on
// weighted graphs"; reading Q26 of DESIGN.md).
//
// The SOVM round (Algorithm 2) over the (min,+) semiring: the frontier F_k holds the
// vertices whose distance dropped in round k-1; round k relaxes every out-arc of F_k,
// d(u) <- min(d(u), d(v) + w(v,u)) (atomicMin), and u joins F_{k+1} when its distance dropped.
// Stop when a round improves nothing (<= n-1 rounds).  Rounds run inside ONE persistent
// cooperative kernel (grid barrier between rounds, frontier-empty test on the device); the
// relaxations are asynchronous within a round (a vertex may already use a distance lowered in
// the same round), which only speeds convergence: the fixpoint — the shortest-path distances
// for non-negative weights — is unique, so the result equals the synchronous oracle's.
// Frontier rows of <= kHeavy arcs are dealt 32 arcs per warp round from a bitmap scan; longer
// rows go through the graph's static 256-arc out-pieces (32 pieces tested per warp at once).
// Near/far threshold (the "balance ... of (min,+) operations" of L596): a round expands only the
// frontier vertices with d < T and carries the others to the next frontier; T stays while the
// next frontier holds a vertex below it and otherwise jumps to (its minimum distance) + delta.
// Expanding roughly in distance order avoids most Bellman-Ford re-relaxations; any order
// reaches the same fixpoint (a vertex whose distance drops re-enters the frontier).
#pragma once
#include "layout.h"

namespace dawn {

#ifndef DAWN_W_RED
#define DAWN_W_RED 1  // relax with red.min (no returning atomic) instead of atomicMin
#endif
constexpr uint32_t kWInf = 0xFFFFFFFFu;   // unreached
constexpr uint32_t kWSat = 0xFFFFFFFEu;   // largest representable distance (saturating add)

struct WParams {
  uint32_t n, nwords, source;
  const uint32_t *rp;
  const int32_t *col;
  const uint32_t *w;                                   // arc weights aligned with col
  const uint32_t *hout_v, *hout_s, *hout_e, *hout_bits;
  uint32_t *fb[3];                                     // rotating frontier bitmaps
  Ctrl *ctrl;
  uint32_t *dist;                                      // [nsrc][n]
  dawn_sssp_stats *stats;                              // [nsrc] or null
  uint32_t delta;                                      // near/far step (>= 1; ~0u: off)
  // batch (dawn_wsssp_batch): nsrc > 0 sources from the device list, searched one after the
  // other in this launch (a grid barrier apart); 0: the single `source`
  const uint32_t *sources;
  uint32_t nsrc;
  const uint32_t *vsrc;                                // whole device list, validated first
  uint32_t vn;
  uint32_t *bad_src;                                   // sticky flag: an id was >= n
};

__device__ __forceinline__ void w_relax(const WParams &p, uint32_t *dist, uint32_t dv, uint32_t j,
                                        uint32_t *fnext, uint32_t &improved, uint32_t &fmin) {
  const uint32_t u = (uint32_t)ld_nc(p.col + j);
  uint32_t c = dv + ld_nc(p.w + j);
  if (c < dv || c > kWSat) c = kWSat;  // saturate (exact while every distance < 2^32 - 1)
  if (c < ld_cg(dist + u)) {
#if DAWN_W_RED
    // fire-and-forget min: no returning round trip on the chain; u joins the next frontier on
    // the observed improvement (if another arc lowered d(u) further meanwhile, u is expanded
    // with that value — an extra frontier entry at worst)
    asm volatile("red.relaxed.gpu.global.min.u32 [%0], %1;" ::"l"(dist + u), "r"(c) : "memory");
    red_or(fnext + (u >> 5), 1u << (u & 31));
    ++improved;
    fmin = min(fmin, c);
#else
    const uint32_t old = atomicMin(dist + u, c);
    if (c < old) {
      red_or(fnext + (u >> 5), 1u << (u & 31));
      ++improved;
      fmin = min(fmin, c);
    }
#endif
  }
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_wsssp(WParams p) {
  __shared__ uint32_t s_imp, s_stop, s_min, s_T;
  __shared__ unsigned long long red[3];
  const uint32_t lane = lane_id();
  const uint32_t nblocks = gridDim.x;
  const uint32_t gwarp = blockIdx.x * (NT / 32) + threadIdx.x / 32;
  const uint32_t nwarps = nblocks * (NT / 32);
  const uint32_t gtid = blockIdx.x * NT + threadIdx.x, nth = nblocks * NT;
  Ctrl *C = p.ctrl;
  unsigned long long bar = 0;
  if (p.vn) {  // the whole device source list is checked before anything is written
    bool bad = false;
    for (uint32_t i = threadIdx.x; i < p.vn; i += NT) bad |= ld_nc(p.vsrc + i) >= p.n;
    if (__syncthreads_or(bad)) {
      if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(p.bad_src, 1u);
      return;
    }
  }
  const uint32_t nsrc = p.nsrc ? p.nsrc : 1u;
  for (uint32_t si = 0; si < nsrc; ++si) {
  const uint32_t src = p.nsrc ? ld_nc(p.sources + si) : p.source;
  uint32_t *const dist = p.dist + (size_t)si * p.n;
  // init: d = infinity, d(s) = 0, F_0 = {s}, the other two bitmaps clear
  for (uint32_t i = gtid; i < p.n; i += nth) dist[i] = (i == src) ? 0u : kWInf;
  for (uint32_t w = gtid; w < p.nwords; w += nth) {
    p.fb[0][w] = (w == (src >> 5)) ? 1u << (src & 31) : 0u;
    p.fb[1][w] = 0;
    p.fb[2][w] = 0;
  }
  if (gtid == 0) {
    for (int i = 0; i < 3; ++i) C->slot[i] = Slot{0, kWInf, 0, 0, 0};  // n_new, big = min d
    C->examined = 0;
  }
  if (threadIdx.x == 0) s_T = p.delta == kWInf ? kWInf : p.delta;  // F_0 = {s}, d(s) = 0 < T
  grid_sync(&C->bar, nblocks, bar);
  uint32_t b = 0, rounds = 0;
  unsigned long long relaxed = 0;
  for (uint32_t k = 0; k + 1 < p.n || k == 0; ++k) {
    // (selects instead of a runtime-indexed parameter array, which would live in local memory)
    auto pick = [&](uint32_t i) { return i == 0 ? p.fb[0] : (i == 1 ? p.fb[1] : p.fb[2]); };
    const uint32_t *fcur = pick(b);
    uint32_t *fnext = pick((b + 1) % 3);
    uint32_t *fclr = pick((b + 2) % 3);  // F_{k-1}: cleared now, written in round k+1
    uint32_t improved = 0, fmin = kWInf;
    const uint32_t T = s_T;
    for (uint32_t w = gtid; w < p.nwords; w += nth) fclr[w] = 0;
    // (a) every frontier vertex: far ones (d >= T) are carried to the next frontier; near light
    //     rows are expanded here, 32 words per warp, one frontier vertex per lane per round
    //     (near heavy rows: the pieces below)
    for (uint32_t base = gwarp * 32; base < p.nwords; base += nwarps * 32) {
      const uint32_t wd = base + lane;
      uint32_t bits = wd < p.nwords ? ld_cg(fcur + wd) : 0u;
      const uint32_t hvy = wd < p.nwords ? ld_nc(p.hout_bits + wd) : 0u;
      while (__ballot_sync(DAWN_FULL, bits != 0)) {
        uint32_t rs = 0, d = 0, dv = 0;
        if (bits) {
          const uint32_t b0 = __ffs(bits) - 1;
          const uint32_t v = wd * 32 + b0;
          bits &= bits - 1;
          dv = ld_cg(dist + v);
          if (dv >= T) {  // far: stays in the frontier
            red_or(fnext + wd, 1u << b0);
            ++improved;
            fmin = min(fmin, dv);
          } else if (!((hvy >> b0) & 1u)) {
            rs = ld_nc(p.rp + v);
            d = ld_nc(p.rp + v + 1) - rs;
          }
        }
        const uint32_t incl = warp_incl_scan(d);
        const uint32_t total = __shfl_sync(DAWN_FULL, incl, 31);
        const uint32_t excl = incl - d;
        for (uint32_t r0 = 0; r0 < total; r0 += 32) {
          const uint32_t t = r0 + lane;
          uint32_t kk = 0;
#pragma unroll
          for (uint32_t step = 16; step; step >>= 1) {
            const uint32_t e = __shfl_sync(DAWN_FULL, excl, kk + step);
            if (e <= t) kk += step;
          }
          const uint32_t ek = __shfl_sync(DAWN_FULL, excl, kk);
          const uint32_t sk = __shfl_sync(DAWN_FULL, rs, kk);
          const uint32_t dk = __shfl_sync(DAWN_FULL, dv, kk);
          if (t < total) {
            w_relax(p, dist, dk, sk + (t - ek), fnext, improved, fmin);
            ++relaxed;
          }
        }
      }
    }
    // (b) heavy rows: static pieces w + i * nwarps, 32 tested against F_k at once
    const uint32_t hend = ld_cg(&C->n_hp_out);
    for (uint32_t pb = gwarp; pb < hend; pb += 32 * nwarps) {
      const uint32_t pcl = pb + lane * nwarps;
      uint32_t vl = 0;
      bool live = false;
      uint32_t dl = 0;
      if (pcl < hend) {
        vl = ld_nc(p.hout_v + pcl);
        live = (ld_cg(fcur + (vl >> 5)) >> (vl & 31)) & 1u;
        if (live) {
          dl = ld_cg(dist + vl);
          live = dl < T;  // far heavy vertices were carried by (a)
        }
      }
      uint32_t lm = __ballot_sync(DAWN_FULL, live);
      while (lm) {
        const uint32_t kk = __ffs(lm) - 1;
        lm &= lm - 1;
        const uint32_t pc = pb + kk * nwarps;
        const uint32_t dv = __shfl_sync(DAWN_FULL, dl, kk);
        const uint32_t s = ld_nc(p.hout_s + pc), e = ld_nc(p.hout_e + pc);
        for (uint32_t j = s + lane; j < e; j += 32) {
          w_relax(p, dist, dv, j, fnext, improved, fmin);
          ++relaxed;
        }
      }
    }
    // round counters: next-frontier entries (improved + carried) and their minimum distance
    // into slot k % 3 (slot (k+1) % 3 reset for the next round)
    improved = warp_sum(improved);
#pragma unroll
    for (int o = 16; o; o >>= 1) fmin = min(fmin, __shfl_xor_sync(DAWN_FULL, fmin, o));
    if (threadIdx.x == 0) { s_imp = 0; s_min = kWInf; }
    __syncthreads();
    if (lane == 0 && improved) {
      atomicAdd(&s_imp, improved);
      atomicMin(&s_min, fmin);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (s_imp) {
        atomicAdd(&C->slot[k % 3].n_new, s_imp);
        atomicMin(&C->slot[k % 3].big, s_min);
      }
      if (blockIdx.x == 0) C->slot[(k + 1) % 3] = Slot{0, kWInf, 0, 0, 0};
    }
    grid_sync(&C->bar, nblocks, bar);
    if (threadIdx.x == 0) {
      s_stop = ld_cg(&C->slot[k % 3].n_new) == 0;
      const uint32_t mn = ld_cg(&C->slot[k % 3].big);
      // T stays while the next frontier has a vertex below it, else min + delta
      if (p.delta != kWInf && mn >= s_T) s_T = (mn > kWSat - p.delta) ? kWInf : mn + p.delta;
    }
    __syncthreads();
    b = (b + 1) % 3;
    if (s_stop) break;
    ++rounds;
  }
  // statistics: reached / E10 counts over the final distances
  unsigned long long reached = 0, er = 0;
  for (uint32_t v = gtid; v < p.n; v += nth) {
    if (ld_cg(dist + v) != kWInf) {
      reached += (v != src);
      er += ld_nc(p.rp + v + 1) - ld_nc(p.rp + v);
    }
  }
  reached = warp_sum(reached);
  er = warp_sum(er);
  relaxed = warp_sum(relaxed);
  if (threadIdx.x == 0) red[0] = red[1] = red[2] = 0;
  __syncthreads();
  if (lane == 0) {
    atomicAdd(&red[0], reached);
    atomicAdd(&red[1], er);
    atomicAdd(&red[2], relaxed);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&C->slot[0].m_new, red[0]);  // slot 0/1 m_new reused as accumulators
    atomicAdd(&C->slot[1].m_new, red[1]);
    atomicAdd(&C->examined, red[2]);
  }
  grid_sync(&C->bar, nblocks, bar);
  if (gtid == 0 && p.stats) {
    dawn_sssp_stats s;
    s.levels = rounds;  // rounds that improved >= 1 distance
    s.reached = (uint32_t)ld_cg(&C->slot[0].m_new);
    s.edges_reach = ld_cg(&C->slot[1].m_new);
    s.edges_examined = ld_cg(&C->examined);
    s.push_levels = rounds + 1;
    s.pull_levels = 0;
    p.stats[si] = s;
  }
  if (si + 1 < nsrc) grid_sync(&C->bar, nblocks, bar);  // stats read before the next init
  }  // sources
  grid_exit(&C->bar, nblocks);
}

}  // namespace dawn

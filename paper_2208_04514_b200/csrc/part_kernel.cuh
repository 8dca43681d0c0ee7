// part_kernel.cuh — partitioned single-source DAWN over W GPUs (the
// paper's memory-frugality motivation, PAPER.md L312-323 (E13) and L554 — graphs one device
// cannot hold).
//
// 1D vertex partition: rank r owns the ids [lo_r, lo_r + R_r) (blocks of Rmax, a multiple of 32).
// It holds only the arcs whose TARGET it owns, twice grouped:
//   out-slice  CSR over every global source v: the arcs v -> u with u owned (targets local)
//   in-rows    CSR over the owned u: the same arcs grouped by target (sources global)
// so a level needs the global frontier F_L and nothing else: push expands the out-slice rows of
// F_L's vertices (Algorithm 2), pull scans the in-rows of the owned unreached
// vertices until the first in-neighbour in F_L (Algorithm 1, Eq. 4) — every discovery
// is local, no remote write.  The only exchange per level is an all-gather of the ranks' slices
// of the next frontier bitmap (Rmax / 8 bytes each) with a 16-byte header (|F|, sum of
// out-degrees) from which every rank takes the same direction / stop decision.  The caller runs
// that all-gather (NCCL over NVLink, torch.distributed) between two dawn_part_step calls.
#pragma once
#include "layout.h"

namespace dawn {

constexpr uint32_t kPartHdr = 4;  // exchange slice header words: [0] |F_{L+1}| here, [1] bit 31:
                                  // one of them has out-degree > kHeavy, bits 0..30 (level-0
                                  // slices only): this rank's reachable bound (kPartReach),
                                  // [2..3] m_f
constexpr uint32_t kPartHeavy = 0x80000000u;
// Fused push levels list the frontier's heavy out-rows (up to kPartHList vertices) and deal their
// kHPiece-arc chunks over all warps, instead of testing every static piece against F_L.
constexpr uint32_t kPartHList = 512;

struct PartState {
  uint32_t done, dir, prev_nf, ecc;
  uint32_t push_levels, pull_levels, reached, pad;
  unsigned long long explored;
  uint32_t pad2;
  uint32_t hvy;   // F_L holds a vertex of out-degree > kHeavy: push levels test the heavy pieces
  uint32_t maxr;  // vertices the search can reach: those with an in-edge (+ s if it has none)
  uint32_t pad3[3];
};
static_assert(sizeof(PartState) % 16 == 0, "PartState");

struct PartCtrl {
  PartState st[2];               // level L reads st[L & 1], CTA 0 writes st[(L + 1) & 1]
  unsigned long long examined;   // adjacency entries read on this rank
  uint32_t n_hp[2];              // static heavy pieces: [0] out-slice rows, [1] in-rows
  unsigned long long xbase;      // fused exchange: this rank's arrival counter at search start
  uint32_t pad[10];              // [0..3]: the fused kernel's grid barrier, [4]: hlist count
};
static_assert(sizeof(GridBarrier) <= 40, "grid barrier in PartCtrl::pad");

struct PartParams {
  uint32_t n, R, Rmax, lo, world, S;  // S = exchange slice words = kPartHdr + Rmax / 32
  uint32_t nwg;                       // words of the global frontier bitmap = ceil(n / 32)
  uint32_t src_local;                 // dawn_part_begin: source - lo if owned, else ~0
  uint32_t rank;
  const uint32_t *rp;                 // out-slice offsets over the n global sources
  const int32_t *col;                 // out-slice targets (local ids)
  const uint32_t *irp;                // in-row offsets over the R owned vertices
  const int32_t *icol;                // in-row sources (global ids)
  const uint32_t *deg;                // global out-degree of the owned vertices (E10 counts)
  const uint32_t *hout_v, *hout_s, *hout_e, *hout_bits;  // out-slice rows > kHeavy: pieces
  const uint32_t *hin_v, *hin_s, *hin_e, *hin_bits;      // in-rows > kHeavy: pieces
  uint32_t *vis;                      // owned vertices reached so far (bitmap)
  uint32_t *cand;                     // candidate bitmap of wide push levels (zero between uses)
  const uint32_t *hasin;              // owned vertices with an in-edge, ascending (n_has)
  uint32_t *ulist, *useg;             // unreached list in per-warp segments, segment counts
  uint32_t *hlist;                    // fused push: heavy frontier vertices (count: ctrl->pad[4])
  uint32_t *hlist2;                   // fused pull: heavy vertices the light pass left (pad[5])
  const uint32_t *top1;               // [R]: first entry of each degree-ordered in-row, or null
  uint32_t n_has;
  uint8_t *lev;                       // deferred distances (as k_sssp: byte L+1, 255 = direct)
  uint32_t *dist;                     // caller's distance slice [R]
  const uint32_t *recv;               // gathered slices of F_L: world x S words
  uint32_t *send;                     // this rank's slice of F_{L+1} (zeroed before the step)
  PartCtrl *ctrl;
  uint32_t variant, can_pull;
  float alpha, beta;
  unsigned long long m_total;         // arcs of the whole graph
};

// Global-memory load of exchange data: the non-coherent path inside one level launch (the
// buffer is read-only there); in the persistent kernel, whose slots are rewritten by peers
// between its levels, a plain (weak, L1-cacheable) load: the slot read in level L is not written
// during level L (peers write the other one), and every CTA passes an acquire of the arrival
// counter and a grid barrier (fence.acq_rel, which invalidates the SM's L1) between the peers'
// stores into it and its first read — hot frontier words then stay in L1 across the level.
template <bool CG>
__device__ __forceinline__ uint32_t xld(const uint32_t *a) {
  if constexpr (CG) return ld_gbl(a); else return ld_nc(a);
}

// Is global vertex v in the frontier held by the gathered slices `rv`?
template <bool CG>
__device__ __forceinline__ bool part_ftest(const PartParams &p, const uint32_t *rv, uint32_t v) {
  const uint32_t q = p.world == 1 ? 0u : v / p.Rmax, r = v - q * p.Rmax;
  return (xld<CG>(rv + (size_t)q * p.S + kPartHdr + (r >> 5)) >> (r & 31)) & 1u;
}

// per-CTA flag: this level discovered a vertex of out-degree > kHeavy (one shared store per
// discovery; part_counters ORs it into the slice header once per CTA — a store per discovery
// straight to the header word serialised millions of same-address stores in L2)
__device__ __forceinline__ uint32_t *part_hv_smem() {
  __shared__ uint32_t hv;
  return &hv;
}

__device__ __forceinline__ void part_discover(const PartParams &p, uint32_t *sd, uint32_t t,
                                              uint32_t L1, uint32_t &n_new,
                                              unsigned long long &m_new) {
  if (L1 < 255u) {
    p.lev[t] = (uint8_t)L1;
  } else {
    p.dist[t] = L1;
    p.lev[t] = 255u;
  }
  red_or(sd + kPartHdr + (t >> 5), 1u << (t & 31));
  n_new += 1;
  const uint32_t dg = ld_nc(p.deg + t);
  m_new += dg;
  if (dg > kHeavy) *part_hv_smem() = 1u;  // a heavy row: the next push level tests the pieces
}

// Claim owned vertex t for level L+1 (test-and-set on vis; each vertex is discovered once).
__device__ __forceinline__ void part_claim(const PartParams &p, uint32_t *sd, uint32_t t,
                                           uint32_t L1, uint32_t &n_new,
                                           unsigned long long &m_new) {
  const uint32_t w = t >> 5, bit = 1u << (t & 31);
  if (!(p.vis[w] & bit) && !(atomicOr(p.vis + w, bit) & bit)) part_discover(p, sd, t, L1, n_new, m_new);
}

// Push visit of owned target t.  MODE 0: claim (test-and-set, discover now); 1: mark a
// candidate unless visited (settled by part_settle after a grid barrier); 2: mark without the
// visited read (few vertices settled yet: most targets are new, part_settle drops the rest).
template <int MODE>
__device__ __forceinline__ void part_visit(const PartParams &p, uint32_t *sd, uint32_t t,
                                           uint32_t L1, uint32_t &n_new,
                                           unsigned long long &m_new) {
  if constexpr (MODE == 0) {
    part_claim(p, sd, t, L1, n_new, m_new);
  } else {
    const uint32_t w = t >> 5, bit = 1u << (t & 31);
    if (MODE == 2 || !(p.vis[w] & bit)) red_or(p.cand + w, bit);
  }
}

// Second half of a candidate push level (after a grid barrier): new = cand & ~vis per owned word.
__device__ __forceinline__ void part_settle(const PartParams &p, uint32_t *sd, uint32_t L1,
                                            uint32_t gtid, uint32_t nth, uint32_t &n_new,
                                            unsigned long long &m_new) {
  const uint32_t nwo = (p.R + 31) / 32;
  for (uint32_t w = gtid; w < nwo; w += nth) {
    const uint32_t c = ld_cg(p.cand + w);
    if (!c) continue;
    p.cand[w] = 0;
    const uint32_t vw = ld_cg(p.vis + w);
    const uint32_t nw = c & ~vw;
    if (!nw) continue;
    p.vis[w] = vw | nw;
    sd[kPartHdr + w] = nw;  // this thread owns the word of the (zeroed) slice
    uint32_t bits = nw;
    while (bits) {
      const uint32_t t = w * 32 + (__ffs(bits) - 1);
      bits &= bits - 1;
      if (L1 < 255u) {
        p.lev[t] = (uint8_t)L1;
      } else {
        p.dist[t] = L1;
        p.lev[t] = 255u;
      }
      n_new += 1;
      const uint32_t dg = ld_nc(p.deg + t);
      m_new += dg;
      if (dg > kHeavy) *part_hv_smem() = 1u;
    }
  }
}

// Level header on the gathered slices rv (thread 0; identical inputs -> identical decisions on
// every CTA of every rank): stop tests and direction, PartState updated in place.
__device__ __forceinline__ void part_header(const PartParams &p, const uint32_t *rv, uint32_t L,
                                            PartState &st) {
  if (st.done) return;
  if (L > 0 && st.dir == kPull) st.pad2 = 1;  // a pull level ran: the unreached list is compacted
  uint32_t nf = 0, hv = 0, reach = 0;
  unsigned long long mf = 0;
  for (uint32_t q = 0; q < p.world; ++q) {
    const uint32_t *h = rv + (size_t)q * p.S;
    nf += ld_cg(h);
    const uint32_t h1 = ld_cg(h + 1);
    hv |= h1 & kPartHeavy;
    reach += h1 & ~kPartHeavy;
    mf += ((unsigned long long)ld_cg(h + 3) << 32) | ld_cg(h + 2);
  }
  st.hvy = hv ? 1u : 0u;
  // condition 1 bound (k_sssp's max_reach, reading Q9): the ranks' level-0 headers carry their
  // counts of owned vertices with an in-edge (the source's owner adds s if it has none)
  if (L == 0) st.maxr = reach;
  const uint32_t L1 = L + 1;
  if (nf == 0) {  // condition 2: F_L is empty
    st.done = 1;
    st.ecc = L ? L - 1 : 0;
    return;
  }
  if (L > 0) st.reached += nf;
  st.explored += mf;
  if (st.reached + 1 >= st.maxr || L1 >= p.n) {  // condition 1 (L177) / the n-1 round bound
    st.done = 1;
    st.ecc = L;
    return;
  }
  if (p.variant == DAWN_PUSH || !p.can_pull) {
    st.dir = kPush;
  } else if (p.variant == DAWN_PULL) {
    st.dir = kPull;
  } else {  // the k_sssp rule (level_header), on the global counters
    const double mu = (double)(p.m_total - min(st.explored, p.m_total));
    const double nu = (double)(st.maxr - 1 - min(st.reached, st.maxr - 1));
    if (st.dir == kPush) {
      if ((double)mf * (double)mf * p.alpha > nu * mu && nf > st.prev_nf) st.dir = kPull;
    } else {
      if ((double)nf * p.beta < (double)p.n && nf < st.prev_nf) st.dir = kPush;
    }
  }
  st.prev_nf = nf;
  st.pad = (st.dir == kPush && mf >= (1ull << 18)) ? 1u : 0u;  // wide push: candidate mode
  if (st.dir == kPush) st.push_levels++; else st.pull_levels++;
}

// The level's work: F_L in rv (all ranks' slices) -> this rank's slice of F_{L+1} in sd.
// LIST (fused kernel): push step (a) also lists the frontier's heavy out-rows; the caller runs
// part_push_heavy after a grid barrier instead of step (b).
// PPART (pull levels): 0 light pass and heavy pieces; 1 the light pass only (fused kernel):
// heavy vertices it settles are claimed without a returning atomic and those it leaves are
// listed for part_pull_heavy, which runs after a grid barrier
template <int NT, bool CG, int MODE = 0, bool LIST = false, int PPART = 0>
__device__ void part_work(const PartParams &p, const PartState &st, uint32_t L, const uint32_t *rv,
                          uint32_t *sd, uint32_t gwarp, uint32_t nwarps, uint32_t &n_new,
                          unsigned long long &m_new, unsigned long long &exam) {
  const uint32_t lane = lane_id();
  const uint32_t L1 = L + 1;
  if (st.dir == kPush) {
    // (a) light out-slice rows (<= kHeavy arcs): 32 words of F_L per warp, each round every lane
    //     contributes its word's next vertex; the round's rows are dealt 32 arcs at a time
    const uint32_t wpr = p.Rmax / 32;
    for (uint32_t base = gwarp * 32; base < p.nwg; base += nwarps * 32) {
      const uint32_t gw = base + lane;
      uint32_t bits = 0;
      if (gw < p.nwg) {
        const uint32_t q = p.world == 1 ? 0u : gw / wpr;
        const uint32_t fw = xld<CG>(rv + (size_t)q * p.S + kPartHdr + (gw - q * wpr));
        const uint32_t hw = ld_nc(p.hout_bits + gw);
        bits = fw & ~hw;
        if (LIST && st.hvy) {
          for (uint32_t hb = fw & hw; hb; hb &= hb - 1) {  // rare: heavy frontier vertices
            const uint32_t i = atomicAdd(&p.ctrl->pad[4], 1u);
            if (i < kPartHList) p.hlist[i] = gw * 32 + (__ffs(hb) - 1);
          }
        }
      }
      while (__ballot_sync(DAWN_FULL, bits != 0)) {
        uint32_t rs = 0, d = 0;
        if (bits) {
          const uint32_t v = gw * 32 + (__ffs(bits) - 1);
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
          if (t < total) {
            part_visit<MODE>(p, sd, (uint32_t)ld_nc(p.col + sk + (t - ek)), L1, n_new, m_new);
            ++exam;
          }
        }
      }
    }
    // (b) heavy out-slice rows: static pieces; warp w takes pieces w + k * nwarps, 32 tested at
    //     once against F_L, then each live piece is expanded 32 arcs per round
    //     (only when F_L holds a vertex whose global out-degree exceeds kHeavy: no out-slice row
    //     of a lighter vertex is heavy on any rank)
    const uint32_t hend = (st.hvy && !LIST) ? ld_cg(&p.ctrl->n_hp[0]) : 0u;
    for (uint32_t pb = gwarp; pb < hend; pb += 32 * nwarps) {
      const uint32_t pcl = pb + lane * nwarps;
      const bool live = pcl < hend && part_ftest<CG>(p, rv, ld_nc(p.hout_v + pcl));
      uint32_t lm = __ballot_sync(DAWN_FULL, live);
      while (lm) {
        const uint32_t kk = __ffs(lm) - 1;
        lm &= lm - 1;
        const uint32_t pc = pb + kk * nwarps;
        const uint32_t s = ld_nc(p.hout_s + pc), e = ld_nc(p.hout_e + pc);
        for (uint32_t j = s + lane; j < e; j += 32) {
          part_visit<MODE>(p, sd, (uint32_t)ld_nc(p.col + j), L1, n_new, m_new);
          ++exam;
        }
      }
    }
  } else {
    // (a) light in-rows over the warp's segment of the unreached list (the static list of owned
    //     vertices with an in-edge at the first pull level, the warp's compacted survivors after;
    //     as k_sssp's pull): two vertices per lane in flight, each scanning its in-row until the
    //     first in-neighbour in F_L (early exit, Eq. 4), 4 independent probes per round trip.
    //     Vertices with heavy in-rows probe their first kHeavyProbe in-edges here (the
    //     highest-degree sources come first, so most settle) and claim with a returning atomic
    //     (a piece may find them concurrently); the pieces finish the rest.
    constexpr int PJ = 2;
    const uint32_t cap = (p.n_has + nwarps - 1) / nwarps;
    const uint32_t seg0 = gwarp * cap;
    const uint32_t *srcl = (st.pad2 ? p.ulist : p.hasin) + seg0;
    uint32_t *dstl = p.ulist + seg0;
    const uint32_t cnt = st.pad2 ? ld_cg(p.useg + gwarp)
                                 : (seg0 < p.n_has ? min(cap, p.n_has - seg0) : 0u);
    uint32_t wr = 0;
    for (uint32_t ib = 0; ib < cnt; ib += 32 * PJ) {
      uint32_t t[PJ], s[PJ], e[PJ], dg[PJ], t1[PJ];
      bool need[PJ], keep[PJ], found[PJ], hv[PJ];
#pragma unroll
      for (int k = 0; k < PJ; ++k) {
        const uint32_t i2 = ib + k * 32 + lane;
        t[k] = i2 < cnt ? ld_cg(srcl + i2) : 0xffffffffu;
        need[k] = keep[k] = found[k] = hv[k] = false;
        s[k] = e[k] = dg[k] = 0;
        if (t[k] != 0xffffffffu) {
          const uint32_t bit = 1u << (t[k] & 31);
          keep[k] = !(ld_cg(p.vis + (t[k] >> 5)) & bit);
          need[k] = keep[k];
          hv[k] = ld_nc(p.hin_bits + (t[k] >> 5)) & bit;
          s[k] = ld_nc(p.irp + t[k]);  // speculative, same round trip
          e[k] = ld_nc(p.irp + t[k] + 1);
          dg[k] = ld_nc(p.deg + t[k]);
          t1[k] = p.top1 ? ld_nc(p.top1 + t[k]) : 0xffffffffu;  // the in-row's first entry
        }
      }
#pragma unroll
      for (int k = 0; k < PJ; ++k) {
        if (hv[k]) e[k] = min(e[k], s[k] + kHeavyProbe);  // the pieces scan the rest
        if (p.top1 && need[k] && e[k] > s[k]) {
          // first probe from the per-vertex copy: no in-row sector when it settles the vertex
          found[k] = part_ftest<CG>(p, rv, t1[k]);
          exam += 1;
          s[k] += 1;
        }
      }
      for (;;) {
        bool any = false;
        uint32_t v[PJ][4];
#pragma unroll
        for (int k = 0; k < PJ; ++k) {
          const bool go = need[k] && !found[k] && s[k] < e[k];
          any |= go;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            v[k][i] = (go && s[k] + i < e[k]) ? (uint32_t)ld_nc(p.icol + s[k] + i) : 0xffffffffu;
        }
        if (!any) break;
#pragma unroll
        for (int k = 0; k < PJ; ++k) {
          if (v[k][0] == 0xffffffffu) continue;
          uint32_t hit = 4;
#pragma unroll
          for (int i = 3; i >= 0; --i)
            if (v[k][i] != 0xffffffffu && part_ftest<CG>(p, rv, v[k][i])) hit = (uint32_t)i;
          const uint32_t adv = hit < 4 ? hit + 1 : min(4u, e[k] - s[k]);
          exam += adv;
          s[k] += adv;
          found[k] = hit < 4;
        }
      }
      if constexpr (PPART == 1) {
        // heavy in-rows the first kHeavyProbe probes left unsettled: listed for the heavy phase
#pragma unroll
        for (int k = 0; k < PJ; ++k) {
          const bool left = hv[k] && need[k] && !found[k];
          const uint32_t lm = __ballot_sync(DAWN_FULL, left);
          if (lm) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(&p.ctrl->pad[5], (uint32_t)__popc(lm));
            base = __shfl_sync(DAWN_FULL, base, 0);
            if (left) p.hlist2[base + __popc(lm & lanemask_lt())] = t[k];
          }
        }
      }
#pragma unroll
      for (int k = 0; k < PJ; ++k) {
        if (found[k]) {
          const uint32_t w = t[k] >> 5, bit = 1u << (t[k] & 31);
          if (hv[k] && PPART == 0) {
            if (atomicOr(p.vis + w, bit) & bit) found[k] = false;  // a piece settled t first
          } else {
            red_or(p.vis + w, bit);  // light rows: this lane alone settles t
          }
        }
        if (found[k]) {
          if (dg[k] > kHeavy) *part_hv_smem() = 1u;  // a heavy out-row in F_{L+1}
          if (L1 < 255u) {
            p.lev[t[k]] = (uint8_t)L1;
          } else {
            p.dist[t[k]] = L1;
            p.lev[t[k]] = 255u;
          }
          red_or(sd + kPartHdr + (t[k] >> 5), 1u << (t[k] & 31));
          n_new += 1;
          m_new += dg[k];
        }
        // survivors (still unreached) stay in the warp's segment, order preserved
        const bool kp = keep[k] && !found[k];
        const uint32_t km = __ballot_sync(DAWN_FULL, kp);
        if (kp) dstl[wr + __popc(km & lanemask_lt())] = t[k];
        wr += __popc(km);
      }
    }
    if (lane == 0) p.useg[gwarp] = wr;
    if constexpr (PPART == 1) return;
    // (b) heavy in-rows: static pieces, 32 in-edges per round, stop at the first hit or once
    //     another piece settled the vertex
    const uint32_t hend = ld_cg(&p.ctrl->n_hp[1]);
    for (uint32_t pb = gwarp; pb < hend; pb += 32 * nwarps) {
      const uint32_t pcl = pb + lane * nwarps;
      uint32_t tl = 0;
      bool need = false;
      if (pcl < hend) {
        tl = ld_nc(p.hin_v + pcl);
        need = !((ld_cg(p.vis + (tl >> 5)) >> (tl & 31)) & 1u);
      }
      uint32_t nm = __ballot_sync(DAWN_FULL, need);
      while (nm) {
        const uint32_t kk = __ffs(nm) - 1;
        nm &= nm - 1;
        const uint32_t pc = pb + kk * nwarps;
        const uint32_t t = __shfl_sync(DAWN_FULL, tl, kk);
        const uint32_t s = ld_nc(p.hin_s + pc), e = ld_nc(p.hin_e + pc);
        for (uint32_t j = s; j < e; j += 32) {
          const uint32_t jj = j + lane;
          const bool hit = jj < e && part_ftest<CG>(p, rv, (uint32_t)ld_nc(p.icol + jj));
          const uint32_t hm = __ballot_sync(DAWN_FULL, hit);
          if (hm) {
            if (lane == 0) {
              exam += __ffs(hm);
              const uint32_t w = t >> 5, bit = 1u << (t & 31);
              if (!(atomicOr(p.vis + w, bit) & bit)) part_discover(p, sd, t, L1, n_new, m_new);
            }
            break;
          }
          if (lane == 0) exam += min(32u, e - j);
          if ((ld_cg(p.vis + (t >> 5)) >> (t & 31)) & 1u) break;
        }
      }
    }
  }
}

// Fused push levels, after the grid barrier that follows step (a): the listed heavy out-rows are
// cut into kHPiece-arc chunks numbered across the list (a warp prefix scan per 32 entries) and
// chunk c goes to warp c mod nwarps; a list that overflowed falls back to testing every static
// piece against F_L (step (b) of part_work).
template <bool CG, int MODE>
__device__ void part_push_heavy(const PartParams &p, const PartState &st, uint32_t L,
                                const uint32_t *rv, uint32_t *sd, uint32_t gwarp, uint32_t nwarps,
                                uint32_t &n_new, unsigned long long &m_new,
                                unsigned long long &exam) {
  if (!st.hvy) return;
  const uint32_t lane = lane_id(), L1 = L + 1;
  const uint32_t cnt = ld_cg(&p.ctrl->pad[4]);
  if (cnt > kPartHList) {
    const uint32_t hend = ld_cg(&p.ctrl->n_hp[0]);
    for (uint32_t pb = gwarp; pb < hend; pb += 32 * nwarps) {
      const uint32_t pcl = pb + lane * nwarps;
      const bool live = pcl < hend && part_ftest<CG>(p, rv, ld_nc(p.hout_v + pcl));
      uint32_t lm = __ballot_sync(DAWN_FULL, live);
      while (lm) {
        const uint32_t kk = __ffs(lm) - 1;
        lm &= lm - 1;
        const uint32_t pc = pb + kk * nwarps;
        const uint32_t s = ld_nc(p.hout_s + pc), e = ld_nc(p.hout_e + pc);
        for (uint32_t j = s + lane; j < e; j += 32) {
          part_visit<MODE>(p, sd, (uint32_t)ld_nc(p.col + j), L1, n_new, m_new);
          ++exam;
        }
      }
    }
    return;
  }
  uint32_t base = 0;  // chunks of the entries before this group of 32
  for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {
    uint32_t rs = 0, re = 0, nc = 0;
    if (i0 + lane < cnt) {
      const uint32_t v = ld_cg(p.hlist + i0 + lane);
      rs = ld_nc(p.rp + v);
      re = ld_nc(p.rp + v + 1);
      nc = (re - rs + kHPiece - 1) / kHPiece;
    }
    const uint32_t incl = warp_incl_scan(nc), tot = __shfl_sync(DAWN_FULL, incl, 31);
    const uint32_t excl = incl - nc;
    // this warp's chunks c in [base, base + tot) with c mod nwarps == gwarp
    uint32_t c = base + (gwarp + nwarps - base % nwarps) % nwarps;
    for (; c < base + tot; c += nwarps) {
      const uint32_t t = c - base;
      uint32_t k = 0;  // the entry holding chunk t (last lane with excl <= t)
#pragma unroll
      for (uint32_t step = 16; step; step >>= 1) {
        const uint32_t e = __shfl_sync(DAWN_FULL, excl, k + step);
        if (k + step < 32 && e <= t) k += step;
      }
      const uint32_t s0 = __shfl_sync(DAWN_FULL, rs, k) + (t - __shfl_sync(DAWN_FULL, excl, k)) * kHPiece;
      const uint32_t e0 = min(__shfl_sync(DAWN_FULL, re, k), s0 + kHPiece);
      for (uint32_t j = s0 + lane; j < e0; j += 32) {
        part_visit<MODE>(p, sd, (uint32_t)ld_nc(p.col + j), L1, n_new, m_new);
        ++exam;
      }
    }
    base += tot;
  }
}

// Fused pull levels, after the grid barrier that follows the light pass: each heavy vertex it
// left is scanned by one warp from its (kHeavyProbe+1)-th in-edge, 32 per round trip, early
// exit; the listed vertices are unique and nothing else settles them now (no returning claim).
template <bool CG>
__device__ void part_pull_heavy(const PartParams &p, uint32_t L, const uint32_t *rv, uint32_t *sd,
                                uint32_t gwarp, uint32_t nwarps, uint32_t &n_new,
                                unsigned long long &m_new, unsigned long long &exam) {
  const uint32_t lane = lane_id(), L1 = L + 1;
  const uint32_t cnt = ld_cg(&p.ctrl->pad[5]);
  for (uint32_t i = gwarp; i < cnt; i += nwarps) {
    const uint32_t t = ld_cg(p.hlist2 + i);
    const uint32_t w = t >> 5, bit = 1u << (t & 31);
    if (ld_cg(p.vis + w) & bit) continue;
    const uint32_t s = ld_nc(p.irp + t) + kHeavyProbe, e = ld_nc(p.irp + t + 1);
    for (uint32_t j = s; j < e; j += 32) {
      const uint32_t jj = j + lane;
      const bool hit = jj < e && part_ftest<CG>(p, rv, (uint32_t)ld_nc(p.icol + jj));
      const uint32_t hm = __ballot_sync(DAWN_FULL, hit);
      if (hm) {
        if (lane == 0) {
          exam += (j - s) + __ffs(hm);
          red_or(p.vis + w, bit);
          part_discover(p, sd, t, L1, n_new, m_new);
        }
        break;
      }
      if (j + 32 >= e && lane == 0) exam += e - s;
    }
  }
}

// CTA-collective: this CTA's counters into the slice header (|F_{L+1}|, m_f) and `examined`.
__device__ __forceinline__ void part_counters(const PartParams &p, uint32_t *sd, uint32_t n_new,
                                              unsigned long long m_new, unsigned long long exam,
                                              unsigned long long *red) {
  const uint32_t lane = lane_id();
  n_new = warp_sum(n_new);
  m_new = warp_sum(m_new);
  exam = warp_sum(exam);
  if (threadIdx.x == 0) red[0] = red[1] = red[2] = 0;
  __syncthreads();
  if (threadIdx.x == 0 && *part_hv_smem()) {
    sd[1] = kPartHeavy;  // (the reach bound bits are used in level-0 slices only)
    *part_hv_smem() = 0u;
  }
  if (lane == 0) {
    if (n_new) atomicAdd(&red[0], (unsigned long long)n_new);
    if (m_new) atomicAdd(&red[1], m_new);
    if (exam) atomicAdd(&red[2], exam);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (red[0]) atomicAdd(sd, (uint32_t)red[0]);
    if (red[1]) atomicAdd(reinterpret_cast<unsigned long long *>(sd + 2), red[1]);
    if (red[2]) atomicAdd(&p.ctrl->examined, red[2]);
  }
}

// This rank's share of the reachable bound: its owned vertices with an in-edge, plus the source
// when this rank owns it and it has none (k_sssp's max_reach split over the ranks).
__device__ __forceinline__ uint32_t part_reach(const PartParams &p) {
  const bool s_noin = p.src_local != 0xffffffffu &&
                      ld_nc(p.irp + p.src_local + 1) == ld_nc(p.irp + p.src_local);
  return p.n_has + (s_noin ? 1u : 0u);
}

// dawn_part_begin: vis <- {s} on the owner, level-0 slice (the caller zeroed `send`), state.
__global__ void k_part_begin(PartParams p) {
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  const uint32_t nwo = (p.R + 31) / 32;
  for (uint32_t w = gtid; w < nwo; w += nth)
    p.vis[w] = (p.src_local != 0xffffffffu && w == (p.src_local >> 5)) ? 1u << (p.src_local & 31) : 0u;
  if (gtid == 0) {
    p.send[1] = part_reach(p);
    if (p.src_local != 0xffffffffu) {
      p.send[kPartHdr + (p.src_local >> 5)] = 1u << (p.src_local & 31);
      p.send[0] = 1;
      const unsigned long long d = ld_nc(p.deg + p.src_local);
      if (d > kHeavy) p.send[1] |= kPartHeavy;
      p.send[2] = (uint32_t)d;
      p.send[3] = (uint32_t)(d >> 32);
    }
    PartState s{};
    s.dir = (p.variant == DAWN_PULL) ? kPull : kPush;
    p.ctrl->st[0] = s;
    p.ctrl->examined = 0;
  }
}

// One level: F_L (gathered) -> this rank's slice of F_{L+1}.  Every CTA takes the same decision
// from the identical headers; CTA 0 records the next state.
template <int NT>
__global__ void __launch_bounds__(NT, 2) k_part_level(PartParams p, uint32_t L) {
  __shared__ PartState st;
  __shared__ unsigned long long red[3];
  const uint32_t gwarp = blockIdx.x * (NT / 32) + threadIdx.x / 32;
  const uint32_t nwarps = gridDim.x * (NT / 32);
  if (threadIdx.x == 0) {
    const uint4 *s4 = reinterpret_cast<const uint4 *>(&p.ctrl->st[L & 1]);
    uint4 *d4 = reinterpret_cast<uint4 *>(&st);
    for (int i = 0; i < (int)(sizeof(PartState) / 16); ++i) d4[i] = __ldcg(s4 + i);
    part_header(p, p.recv, L, st);
    if (blockIdx.x == 0) p.ctrl->st[(L + 1) & 1] = st;
    *part_hv_smem() = 0u;
  }
  __syncthreads();
  if (st.done) return;
  uint32_t n_new = 0;
  unsigned long long m_new = 0, exam = 0;
  part_work<NT, false>(p, st, L, p.recv, p.send, gwarp, nwarps, n_new, m_new, exam);
  part_counters(p, p.send, n_new, m_new, exam, red);
}

// ---- fused exchange: the whole search in ONE persistent kernel per rank ---------------------
// Each level, the rank builds its slice of F_{L+1} in `send` and writes it straight into slot
// (L+1) & 1 of EVERY rank's receive buffers (its own included) — plain stores into peer memory
// over NVLink / NVSwitch (peer pointers from CUDA IPC) or local memory when the ranks share a
// device — then, after a system-scope release fence, adds 1 to every rank's arrival counter.
// A rank starts level L+1 once its counter reached base + W * (L + 1): all W slices landed.
// No host round trip, NCCL call or kernel boundary per level.  Counters are monotonic across
// searches (base = the counter at the start of the search, kept in PartCtrl), so nothing is
// reset while a fast peer may already be signalling.
constexpr int kPartMaxW = 16;
struct PartPeers {
  uint32_t *recv[kPartMaxW];             // rank q's two receive slots (2 x world x S words)
  unsigned long long *flag[kPartMaxW];   // rank q's arrival counter (monotonic, starts at 0)
};

__device__ __forceinline__ void red_add_release_sys64(unsigned long long *p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys64(const unsigned long long *p) {
  unsigned long long r;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
  return r;
}

template <int NT>
__global__ void __launch_bounds__(NT, 2) k_part_fused(PartParams p, PartPeers peers,
                                                      dawn_sssp_stats *stats) {
  __shared__ PartState st;
  __shared__ unsigned long long red[3];
  const uint32_t nblocks = gridDim.x;
  const uint32_t gwarp = blockIdx.x * (NT / 32) + threadIdx.x / 32;
  const uint32_t nwarps = nblocks * (NT / 32);
  const uint32_t gtid = blockIdx.x * NT + threadIdx.x, nth = nblocks * NT;
  PartCtrl *C = p.ctrl;
  GridBarrier *gb = reinterpret_cast<GridBarrier *>(&C->pad[0]);
  unsigned long long bar = 0;
  const unsigned long long base = ld_cg(&C->xbase);
  const uint32_t *const myrecv = peers.recv[p.rank];
  const unsigned long long *const xbar = peers.flag[p.rank];
  const size_t slot_words = (size_t)p.world * p.S;
  const size_t my_off = (size_t)p.rank * p.S;
  // ---- begin: vis <- {s} on the owner, the level-0 slice, state
  const uint32_t nwo = (p.R + 31) / 32;
  for (uint32_t w = gtid; w < nwo; w += nth)
    p.vis[w] = (p.src_local != 0xffffffffu && w == (p.src_local >> 5)) ? 1u << (p.src_local & 31) : 0u;
  for (uint32_t i = gtid; i < p.S; i += nth) {
    uint32_t x = (i == 1) ? part_reach(p) : 0u;
    if (p.src_local != 0xffffffffu) {
      if (i == 0) x = 1;
      else if (i == 1) x |= ld_nc(p.deg + p.src_local) > kHeavy ? kPartHeavy : 0u;
      else if (i == 2) x = ld_nc(p.deg + p.src_local);
      else if (i == kPartHdr + (p.src_local >> 5)) x = 1u << (p.src_local & 31);
    }
    for (uint32_t q = 0; q < p.world; ++q) peers.recv[q][my_off + i] = x;  // slot 0 of every rank
  }
  if (gtid == 0) C->examined = 0;
  if (threadIdx.x == 0) {
    st = PartState{};
    st.dir = (p.variant == DAWN_PULL) ? kPull : kPush;
    *part_hv_smem() = 0u;
  }
  grid_sync(gb, nblocks, bar);
  if (gtid == 0) {
    __threadfence_system();
    for (uint32_t q = 0; q < p.world; ++q) red_add_release_sys64(peers.flag[q], 1ull);
  }
  uint32_t L = 0;
  for (;; ++L) {
    // wait for every rank's slice of F_L, then decide (identical on every CTA of every rank)
    if (threadIdx.x == 0) {
      const unsigned long long target = base + (unsigned long long)p.world * (L + 1);
      while (ld_acquire_sys64(xbar) < target) {
      }
      part_header(p, myrecv + (L & 1) * slot_words, L, st);
    }
    __syncthreads();
    if (st.done) break;
    const uint32_t *rv = myrecv + (L & 1) * slot_words;
    for (uint32_t i = gtid; i < p.S; i += nth) p.send[i] = 0;
    if (gtid == 0) C->pad[4] = C->pad[5] = 0;  // heavy lists of this level (last read before a barrier)
    grid_sync(gb, nblocks, bar);
    uint32_t n_new = 0;
    unsigned long long m_new = 0, exam = 0;
    if (st.dir == kPush && st.pad) {
      // wide push level: candidates (fire-and-forget marks), settled after a grid barrier
      if ((unsigned long long)(st.reached + 1) * 32 < p.n) {
        part_work<NT, true, 2, true>(p, st, L, rv, p.send, gwarp, nwarps, n_new, m_new, exam);
        if (st.hvy) grid_sync(gb, nblocks, bar);
        part_push_heavy<true, 2>(p, st, L, rv, p.send, gwarp, nwarps, n_new, m_new, exam);
      } else {
        part_work<NT, true, 1, true>(p, st, L, rv, p.send, gwarp, nwarps, n_new, m_new, exam);
        if (st.hvy) grid_sync(gb, nblocks, bar);
        part_push_heavy<true, 1>(p, st, L, rv, p.send, gwarp, nwarps, n_new, m_new, exam);
      }
      grid_sync(gb, nblocks, bar);
      part_settle(p, p.send, L + 1, gtid, nth, n_new, m_new);
    } else if (st.dir == kPush) {
      part_work<NT, true, 0, true>(p, st, L, rv, p.send, gwarp, nwarps, n_new, m_new, exam);
      if (st.hvy) grid_sync(gb, nblocks, bar);
      part_push_heavy<true, 0>(p, st, L, rv, p.send, gwarp, nwarps, n_new, m_new, exam);
    } else {
      // pull: light pass, grid barrier, the heavy in-rows it left
      part_work<NT, true, 0, false, 1>(p, st, L, rv, p.send, gwarp, nwarps, n_new, m_new, exam);
      grid_sync(gb, nblocks, bar);
      part_pull_heavy<true>(p, L, rv, p.send, gwarp, nwarps, n_new, m_new, exam);
    }
    part_counters(p, p.send, n_new, m_new, exam, red);
    grid_sync(gb, nblocks, bar);
    // fan out F_{L+1}'s slice into slot (L+1) & 1 of every rank, then signal
    const size_t dst = ((L + 1) & 1) * slot_words + my_off;
    for (uint32_t i = gtid; i < p.S; i += nth) {
      const uint32_t x = ld_cg(p.send + i);
      for (uint32_t q = 0; q < p.world; ++q) peers.recv[q][dst + i] = x;
    }
    grid_sync(gb, nblocks, bar);
    if (gtid == 0) {
      __threadfence_system();
      for (uint32_t q = 0; q < p.world; ++q) red_add_release_sys64(peers.flag[q], 1ull);
    }
  }
  // ---- finish: the distance slice from the deferred bytes, statistics
  for (uint32_t t = gtid; t < p.R; t += nth) {
    const uint32_t reached = (ld_cg(p.vis + (t >> 5)) >> (t & 31)) & 1u;
    const uint32_t lb = ld_cg(reinterpret_cast<const uint32_t *>(p.lev) + (t >> 2));
    const uint32_t d = (t == p.src_local) ? 0u : (reached ? (lb >> (8 * (t & 3))) & 0xffu : kUnreached);
    if (d != 255u) p.dist[t] = d;
  }
  grid_sync(gb, nblocks, bar);
  if (gtid == 0) {
    C->xbase = base + (unsigned long long)p.world * (L + 1);  // every rank signalled L+1 times
    if (stats) {
      dawn_sssp_stats o;
      o.levels = st.ecc;
      o.reached = st.reached;
      o.edges_reach = st.explored;
      o.edges_examined = ld_cg(&C->examined);
      o.push_levels = st.push_levels;
      o.pull_levels = st.pull_levels;
      *stats = o;
    }
  }
  grid_exit(gb, nblocks);
}

// dawn_part_finish: the distance slice from the deferred bytes (as dist_final), statistics.
__global__ void k_part_finish(PartParams p, uint32_t parity, dawn_sssp_stats *stats) {
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  for (uint32_t t = gtid; t < p.R; t += nth) {
    const uint32_t reached = (ld_cg(p.vis + (t >> 5)) >> (t & 31)) & 1u;
    const uint32_t d = (t == p.src_local) ? 0u : (reached ? (uint32_t)ld_cg(reinterpret_cast<const uint32_t *>(p.lev) + (t >> 2)) >> (8 * (t & 3)) & 0xffu : kUnreached);
    if (d != 255u) p.dist[t] = d;
  }
  if (gtid == 0 && stats) {
    const PartState s = p.ctrl->st[parity];
    dawn_sssp_stats o;
    o.levels = s.ecc;
    o.reached = s.reached;
    o.edges_reach = s.explored;
    o.edges_examined = p.ctrl->examined;
    o.push_levels = s.push_levels;
    o.pull_levels = s.pull_levels;
    *stats = o;
  }
}

}  // namespace dawn

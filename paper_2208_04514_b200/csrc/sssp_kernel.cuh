// sssp_kernel.cuh — single-source DAWN as ONE persistent cooperative kernel (sm_100a).
//
// One launch = init + every level + statistics.  Each level is either
//   PUSH (SOVM, Algorithm 2; Eq. 9): the frontier queue's CSR rows
//        are expanded; a target u is claimed by an atomic test-and-set on the `vis` bitmap
//        (the "distance[col[j]] = 0" filter of line 6, reading Q1), dist[u] = L+1, and u is
//        appended to the next queue with a warp-aggregated atomic (ballot + popc);
//   PULL (BOVM, Algorithm 1; Eq. 4): every unreached vertex scans
//        its CSC row until the first in-neighbour in the level-L frontier bitmap (early exit),
//        a warp owns 32 vertices = one bitmap word, so the next bitmap is written without
//        atomics and the frontier read is a level-start snapshot (reading Q2).
// The direction is chosen on the device from the frontier's measured size (n_f, m_f) against
// the unexplored edges (Beamer's rule, cited by the paper at L123), and the frontier-empty
// test (PAPER.md L174-179 conditions 1-2) is evaluated after each grid barrier: no host
// round trip per level.
#pragma once
#include "layout.h"

namespace dawn {

struct SsspParams {
  uint32_t n, nwords;
  unsigned long long m;
  const uint32_t *rp, *irp;
  const int32_t *col, *icol;
  const uint32_t *noin;
  uint32_t *vis, *fb[2];
  uint32_t *Lv[2];
  uint2 *Lsd[2];
  uint32_t *Hv[2];
  uint2 *Hsd[2];
  uint32_t *Hp[2], *Pm[2];
  Ctrl *ctrl;
  uint32_t *dist;
  dawn_sssp_stats *stats;
  uint32_t source, variant, can_pull, sym;
  float alpha, beta;
};


struct LevelState {
  uint32_t L, nf, prev_nf, dir, rep, q, b, stop, ecc;
  uint32_t push_levels, pull_levels, reached;
  uint32_t n_light, n_heavy, n_pieces;
  unsigned long long mf, explored, push_edges;
};

// Warp-collective append of discovered vertices to queue `q` (light rows / heavy pieces).
// Vertices with out-degree 0 are not enqueued ("skipping ... reachable nodes
// with an out-degree of 0").
__device__ __forceinline__ void enqueue_frontier(const SsspParams &p, Slot *s, int q, bool has,
                                                 uint32_t u, uint32_t rs, uint32_t d) {
  const uint32_t lane = lane_id();
  const bool isL = has && d > 0 && d <= kLight;
  const bool isH = has && d > kLight;
  const uint32_t mL = __ballot_sync(DAWN_FULL, isL);
  if (mL) {
    const uint32_t leader = __ffs(mL) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(&s->n_light, __popc(mL));
    base = __shfl_sync(DAWN_FULL, base, leader);
    if (isL) {
      const uint32_t pos = base + __popc(mL & lanemask_lt());
      p.Lv[q][pos] = u;
      p.Lsd[q][pos] = make_uint2(rs, d);
    }
  }
  const uint32_t mH = __ballot_sync(DAWN_FULL, isH);
  if (mH) {
    const uint32_t np = isH ? (d + kPiece - 1) / kPiece : 0;
    const uint32_t incl = warp_incl_scan(np);
    const uint32_t tot = __shfl_sync(DAWN_FULL, incl, 31);
    const uint32_t leader = __ffs(mH) - 1;
    uint32_t hb = 0, pb = 0;
    if (lane == leader) {
      hb = atomicAdd(&s->n_heavy, __popc(mH));
      pb = atomicAdd(&s->n_pieces, tot);
    }
    hb = __shfl_sync(DAWN_FULL, hb, leader);
    pb = __shfl_sync(DAWN_FULL, pb, leader);
    if (isH) {
      const uint32_t pos = hb + __popc(mH & lanemask_lt());
      const uint32_t first = pb + incl - np;
      p.Hv[q][pos] = u;
      p.Hsd[q][pos] = make_uint2(rs, d);
      p.Hp[q][pos] = first;
      for (uint32_t i = 0; i < np; ++i) p.Pm[q][first + i] = pos;
    }
  }
}

// Push-mode visit of arc (frontier vertex) -> u, warp-collective (all lanes call; `act`
// false for idle lanes).
__device__ __forceinline__ void push_visit(const SsspParams &p, Slot *ns, int qn, uint32_t L1,
                                           bool act, uint32_t u, uint32_t &n_new,
                                           unsigned long long &m_new) {
  bool disc = false;
  uint32_t rs = 0, d = 0;
  if (act) {
    const uint32_t w = u >> 5, bit = 1u << (u & 31);
    const uint32_t cur = p.vis[w];  // weak load: a stale 0 only costs an atomic
    if (!(cur & bit)) disc = !(atomicOr(&p.vis[w], bit) & bit);
  }
  if (disc) {
    rs = ld_nc(p.rp + u);
    d = ld_nc(p.rp + u + 1) - rs;
    p.dist[u] = L1;
    n_new += 1;
    m_new += d;
  }
  enqueue_frontier(p, ns, qn, disc, u, rs, d);
}

__device__ void push_level(const SsspParams &p, const LevelState &st, Slot *ns, uint32_t gwarp,
                           uint32_t nwarps, uint32_t &n_new, unsigned long long &m_new) {
  const int q = st.q, qn = q ^ 1;
  const uint32_t lane = lane_id();
  const uint32_t L1 = st.L + 1;
  const uint32_t G = (st.n_light + 31) / 32;
  const uint32_t items = G + st.n_pieces;
  for (uint32_t it = gwarp; it < items; it += nwarps) {
    if (it < G) {
      // 32 light rows; edges of the group dealt to lanes round-robin (owner by shfl search)
      const uint32_t idx = it * 32 + lane;
      uint32_t s = 0, d = 0;
      if (idx < st.n_light) {
        const uint2 sd = ld_cg2(p.Lsd[q] + idx);
        s = sd.x;
        d = sd.y;
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
        const bool act = t < total;
        const uint32_t u = act ? (uint32_t)ld_nc(p.col + sk + (t - ek)) : 0u;
        push_visit(p, ns, qn, L1, act, u, n_new, m_new);
      }
    } else {
      const uint32_t pc = it - G;
      const uint32_t h = ld_cg(p.Pm[q] + pc);
      const uint2 sd = ld_cg2(p.Hsd[q] + h);
      const uint32_t p0 = ld_cg(p.Hp[q] + h);
      const uint32_t off = (pc - p0) * kPiece;
      const uint32_t len = min(kPiece, sd.y - off);
      const int32_t *row = p.col + sd.x + off;
      for (uint32_t i = 0; i < len; i += 32) {
        const bool act = i + lane < len;
        const uint32_t u = act ? (uint32_t)ld_nc(row + i + lane) : 0u;
        push_visit(p, ns, qn, L1, act, u, n_new, m_new);
      }
    }
  }
}

__device__ void pull_level(const SsspParams &p, const LevelState &st, uint32_t gwarp,
                           uint32_t nwarps, uint32_t &n_new, unsigned long long &m_new,
                           unsigned long long &examined) {
  const uint32_t lane = lane_id();
  const uint32_t L1 = st.L + 1;
  const uint32_t *fcur = p.fb[st.b];
  uint32_t *fnext = p.fb[st.b ^ 1];
  const uint32_t tail_bits = p.n & 31;
  for (uint32_t w = gwarp; w < p.nwords; w += nwarps) {
    const uint32_t vw = ld_cg(p.vis + w);
    uint32_t todo = ~vw;
    if (w == p.nwords - 1 && tail_bits) todo &= (1u << tail_bits) - 1;
    bool found = false;
    uint32_t s = 0, e = 0;
    const uint32_t u = w * 32 + lane;
    if ((todo >> lane) & 1u) {
      s = ld_nc(p.irp + u);
      e = ld_nc(p.irp + u + 1);
      uint32_t j = s;
      for (; j < e; ++j) {
        const uint32_t v = (uint32_t)ld_nc(p.icol + j);
        if ((fcur[v >> 5] >> (v & 31)) & 1u) {
          found = true;
          ++j;
          break;
        }
      }
      examined += j - s;
    }
    const uint32_t nb = __ballot_sync(DAWN_FULL, found);
    if (lane == 0) {
      fnext[w] = nb;
      if (nb) p.vis[w] = vw | nb;
    }
    if (found) {
      p.dist[u] = L1;
      n_new += 1;
      m_new += p.sym ? (e - s) : (ld_nc(p.rp + u + 1) - ld_nc(p.rp + u));
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

template <int NT>
__global__ void __launch_bounds__(NT) k_sssp(SsspParams p) {
  __shared__ LevelState st;
  __shared__ unsigned long long red[2];
  const uint32_t nblocks = gridDim.x;
  const uint32_t gwarp = blockIdx.x * (NT / 32) + threadIdx.x / 32;
  const uint32_t nwarps = nblocks * (NT / 32);
  const uint32_t gtid = blockIdx.x * NT + threadIdx.x;
  const uint32_t nthreads = nblocks * NT;
  Ctrl *C = p.ctrl;
  const uint32_t src = p.source;
  // condition 1 bound: only vertices with an in-edge (plus s itself) can ever be reached
  const uint32_t max_reach = ld_cg(&C->n_hasin) + ((p.noin[src >> 5] >> (src & 31)) & 1u);

  // ---- a1 init: dist <- UNREACHED (d(s) = 0), vis <- no-in-edge vertices | {s}  (Q4, Q7)
  for (uint32_t i = gtid; i < p.n; i += nthreads) p.dist[i] = (i == src) ? 0u : kUnreached;
  for (uint32_t w = gtid; w < p.nwords; w += nthreads)
    p.vis[w] = p.noin[w] | ((w == (src >> 5)) ? (1u << (src & 31)) : 0u);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) C->slot[i] = Slot{0, 0, 0, 0, 0, 0};
    C->examined = 0;
    const uint32_t rs = p.rp[src], d = p.rp[src + 1] - rs;
    Slot &s0 = C->slot[0];
    s0.n_new = 1;
    s0.m_new = d;
    if (d > 0 && d <= kLight) {
      p.Lv[0][0] = src;
      p.Lsd[0][0] = make_uint2(rs, d);
      s0.n_light = 1;
    } else if (d > kLight) {
      const uint32_t np = (d + kPiece - 1) / kPiece;
      p.Hv[0][0] = src;
      p.Hsd[0][0] = make_uint2(rs, d);
      p.Hp[0][0] = 0;
      for (uint32_t i = 0; i < np; ++i) p.Pm[0][i] = 0;
      s0.n_heavy = 1;
      s0.n_pieces = np;
    }
  }
  if (threadIdx.x == 0) {
    st = LevelState{};
    st.dir = (p.variant == DAWN_PULL) ? kPull : kPush;
  }
  grid_sync(&C->bar, nblocks);

  unsigned long long examined = 0;
  for (;;) {
    if (threadIdx.x == 0) {
      const Slot *cs = &C->slot[st.L % 3];
      st.nf = ld_cg(&cs->n_new);
      st.mf = ld_cg(&cs->m_new);
      st.n_light = ld_cg(&cs->n_light);
      st.n_heavy = ld_cg(&cs->n_heavy);
      st.n_pieces = ld_cg(&cs->n_pieces);
      if (blockIdx.x == 0) C->slot[(st.L + 2) % 3] = Slot{0, 0, 0, 0, 0, 0};
      if (st.L > 0) st.reached += st.nf;
      st.explored += st.mf;
      st.stop = 0;
      if (st.nf == 0) {
        st.stop = 1;
        st.ecc = st.L - 1;
      } else if (st.reached + 1 >= max_reach || st.L + 1 >= p.n) {
        st.stop = 1;  // condition 1: nothing left to discover
        st.ecc = st.L;
      } else {
        // a4 direction choice (identical in every CTA: same inputs)
        if (p.variant == DAWN_PUSH || !p.can_pull) {
          st.dir = kPush;
        } else if (p.variant == DAWN_PULL) {
          st.dir = kPull;
        } else {
          const double mu = (double)(p.m - st.explored);
          if (st.dir == kPush) {
            if ((double)st.mf * p.alpha > mu && st.nf > st.prev_nf) st.dir = kPull;
          } else {
            if ((double)st.nf * p.beta < (double)p.n && st.nf < st.prev_nf) st.dir = kPush;
          }
        }
        st.prev_nf = st.nf;
      }
    }
    __syncthreads();
    if (st.stop) break;

    if (st.dir == kPull && st.rep == kRepQueue) {
      // queue -> frontier bitmap fb[b]: clear, barrier, scatter, barrier
      uint32_t *fb = p.fb[st.b];
      for (uint32_t w = gtid; w < p.nwords; w += nthreads) fb[w] = 0;
      grid_sync(&C->bar, nblocks);
      for (uint32_t i = gtid; i < st.n_light; i += nthreads) {
        const uint32_t v = ld_cg(p.Lv[st.q] + i);
        red_or(fb + (v >> 5), 1u << (v & 31));
      }
      for (uint32_t i = gtid; i < st.n_heavy; i += nthreads) {
        const uint32_t v = ld_cg(p.Hv[st.q] + i);
        red_or(fb + (v >> 5), 1u << (v & 31));
      }
      grid_sync(&C->bar, nblocks);
      if (threadIdx.x == 0) st.rep = kRepBitmap;
    } else if (st.dir == kPush && st.rep == kRepBitmap) {
      // frontier bitmap fb[b] -> queue q (ballot/popc compaction), barrier
      Slot *cs = &C->slot[st.L % 3];
      const uint32_t *fb = p.fb[st.b];
      const uint32_t lane = lane_id();
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
          enqueue_frontier(p, cs, st.q, has, u, rs, d);
        }
      }
      grid_sync(&C->bar, nblocks);
      if (threadIdx.x == 0) {
        st.n_light = ld_cg(&cs->n_light);
        st.n_heavy = ld_cg(&cs->n_heavy);
        st.n_pieces = ld_cg(&cs->n_pieces);
        st.rep = kRepQueue;
      }
      __syncthreads();
    }

    Slot *ns = &C->slot[(st.L + 1) % 3];
    uint32_t n_new = 0;
    unsigned long long m_new = 0;
    if (st.dir == kPush) {
      push_level(p, st, ns, gwarp, nwarps, n_new, m_new);
    } else {
      pull_level(p, st, gwarp, nwarps, n_new, m_new, examined);
    }
    block_flush(n_new, m_new, &ns->n_new, &ns->m_new, red);
    grid_sync(&C->bar, nblocks);
    if (threadIdx.x == 0) {
      if (st.dir == kPush) {
        st.push_levels++;
        st.push_edges += st.mf;
        st.q ^= 1;
        st.rep = kRepQueue;
      } else {
        st.pull_levels++;
        st.b ^= 1;
        st.rep = kRepBitmap;
      }
      st.L++;
    }
    __syncthreads();
  }

  // ---- a7 statistics
  if (p.stats) {
    block_flush(0u, examined, nullptr, &C->examined, red);
    grid_sync(&C->bar, nblocks);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      dawn_sssp_stats s;
      s.levels = st.ecc;
      s.reached = st.reached;
      s.edges_reach = st.explored;
      s.edges_examined = st.push_edges + ld_cg(&C->examined);
      s.push_levels = st.push_levels;
      s.pull_levels = st.pull_levels;
      *p.stats = s;
    }
  }
}

}  // namespace dawn

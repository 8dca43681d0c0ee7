// narrow_kernel.cuh — high-diameter graphs (BASELINE configs[2]: the 4096 x 4096 grid, 8191
// levels of <= 4096 vertices).  Level-synchronous DAWN is latency-bound there:
// each level is a dependent chain frontier -> row -> target -> visited test -> enqueue.  k_narrow
// runs the search on ONE CTA with the frontier queue in shared memory, so a level costs three
// global round trips (col, visited test-and-set with the target's row bounds loaded alongside,
// dist store) plus a __syncthreads — no grid barrier, no global queue, no counters in L2.
// Each level is the SOVM step (Algorithm 2): frontier rows expanded, targets
// claimed by atomicOr on the visited bitmap (A2 line 6 filter, reading Q1), distance L+1.
//
// The other CTAs of the launch only initialise dist / vis (a grid-wide fill) and exit.  When
// the next frontier outgrows shared memory, CTA 0 writes it as a regular k_sssp queue
// (vertex, row start, edge offset + chunk map) plus the level state and k_sssp — enqueued by
// dawn_sssp right behind k_narrow — resumes from it.  When the search finishes inside k_narrow,
// k_sssp exits at once.
#pragma once
#include "sssp_kernel.cuh"

namespace dawn {

constexpr uint32_t kNarrowCap = 6144;  // frontier entries held in shared memory (x2 buffers)

struct NarrowParams {
  uint32_t n, nwords;
  unsigned long long m;
  const uint32_t *rp;
  const int32_t *col;
  const uint32_t *noin;
  uint32_t *vis, *dist;
  uint32_t *Lv0;
  uint2 *Lsd0;
  uint32_t *Cf0;
  Ctrl *ctrl;
  dawn_sssp_stats *stats;
  uint32_t source, max_reach_base, seq;
};

struct NarrowSmem {
  uint32_t u[2][kNarrowCap];
  uint32_t rs[2][kNarrowCap];
  uint32_t off[2][kNarrowCap];  // exclusive edge offset of the entry within its frontier
  unsigned long long cnt[2];    // (entries << 32) | edges, allocated together
  unsigned long long m_new;
  uint32_t n_new, overflow;
};

inline size_t narrow_smem_bytes() { return sizeof(NarrowSmem); }

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_narrow(NarrowParams p) {
  extern __shared__ __align__(16) unsigned char smraw[];
  NarrowSmem &S = *reinterpret_cast<NarrowSmem *>(smraw);
  Ctrl *C = p.ctrl;
  const uint32_t src = p.source;
  const uint32_t gtid = blockIdx.x * NT + threadIdx.x, nthreads = gridDim.x * NT;
  // ---- a1 init (all CTAs): dist <- UNREACHED (d(s) = 0), vis <- no-in-edge | {s}
  for (uint32_t i = gtid; i < p.n; i += nthreads) p.dist[i] = (i == src) ? 0u : kUnreached;
  for (uint32_t w = gtid; w < p.nwords; w += nthreads)
    p.vis[w] = p.noin[w] | ((w == (src >> 5)) ? (1u << (src & 31)) : 0u);
  __syncthreads();
  if (blockIdx.x != 0) {
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&C->narrow_init, 1u);
    }
    return;
  }
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    while (ld_acquire(&C->narrow_init) < gridDim.x - 1) {
    }
    C->narrow_init = 0;
    fence_acq_rel_gpu();
  }
  const uint32_t max_reach = p.max_reach_base + ((p.noin[src >> 5] >> (src & 31)) & 1u);
  if (tid == 0) {
    const uint32_t rs = ld_nc(p.rp + src), d = ld_nc(p.rp + src + 1) - rs;
    S.u[0][0] = src;
    S.rs[0][0] = rs;
    S.off[0][0] = 0;
    S.cnt[0] = d ? ((1ull << 32) | d) : 0ull;
    S.overflow = 0;
  }
  __syncthreads();
  uint32_t L = 0, cur = 0, reached = 0, levels = 0, ecc = 0;
  unsigned long long explored = ld_nc(p.rp + src + 1) - ld_nc(p.rp + src), push_edges = 0;
  uint32_t status = 1;  // 1 = finished, 2 = handed over to k_sssp
  for (;;) {
    const unsigned long long cq = S.cnt[cur];
    const uint32_t nq = (uint32_t)(cq >> 32), E = (uint32_t)cq;
    if (tid == 0) {
      S.cnt[cur ^ 1] = 0;
      S.m_new = 0;
      S.n_new = 0;
    }
    __syncthreads();
    // thread per frontier entry (entries tid, tid + NT, ...; grids / road networks have short
    // rows), kU arcs in flight per thread: col loads, then row bounds + claims together.
    // Discovered vertices are appended with ONE shared atomic per warp per batch.
    constexpr int kU = 8;
    const uint32_t lane = lane_id();
    uint32_t my_new = 0;
    unsigned long long my_m = 0;
    uint32_t ei = tid, ej = 0;  // next arc: entry ei, arc ej of its row
    uint32_t ed = 0, ers = 0;
    if (ei < nq) {
      ers = S.rs[cur][ei];
      ed = ((ei + 1 < nq) ? S.off[cur][ei + 1] : E) - S.off[cur][ei];
    }
    for (;;) {
      uint32_t u[kU];
      int got = 0;
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        u[k] = 0xffffffffu;
        while (ei < nq && ej >= ed) {  // next entry of this thread
          ei += NT;
          ej = 0;
          if (ei < nq) {
            ers = S.rs[cur][ei];
            ed = ((ei + 1 < nq) ? S.off[cur][ei + 1] : E) - S.off[cur][ei];
          }
        }
        if (ei < nq) {
          u[k] = (uint32_t)ld_nc(p.col + ers + ej);
          ++ej;
          ++got;
        }
      }
      if (!__any_sync(DAWN_FULL, got > 0)) break;
      uint32_t a[kU], b[kU], old[kU];
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        old[k] = ~0u;
        if (u[k] != 0xffffffffu) {
          a[k] = ld_nc(p.rp + u[k]);
          b[k] = ld_nc(p.rp + u[k] + 1);
          old[k] = atomicOr(p.vis + (u[k] >> 5), 1u << (u[k] & 31));
        }
      }
      uint32_t nput = 0, dput = 0;
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        const bool fresh = !((old[k] >> (u[k] & 31)) & 1u);
        if (fresh) {
          p.dist[u[k]] = L + 1;
          my_new += 1;
          my_m += b[k] - a[k];
          if (b[k] > a[k]) {
            ++nput;
            dput += b[k] - a[k];
          }
        } else {
          u[k] = 0xffffffffu;
        }
      }
      // warp-aggregated reservation of (entries, arcs) for this batch
      const uint32_t cinc = warp_incl_scan(nput), dinc = warp_incl_scan(dput);
      unsigned long long base = 0;
      if (lane == 31 && cinc)
        base = atomicAdd(&S.cnt[cur ^ 1], ((unsigned long long)cinc << 32) | dinc);
      base = __shfl_sync(DAWN_FULL, base, 31);
      uint32_t i = (uint32_t)(base >> 32) + cinc - nput;
      uint32_t o = (uint32_t)base + dinc - dput;
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        if (u[k] == 0xffffffffu || b[k] <= a[k]) continue;
        if (i < kNarrowCap) {
          S.u[cur ^ 1][i] = u[k];
          S.rs[cur ^ 1][i] = a[k];
          S.off[cur ^ 1][i] = o;
        } else {
          // overflow: park the entry in the global queue slot it will need anyway
          p.Lv0[i] = u[k];
          p.Lsd0[i] = make_uint2(a[k], o);
          S.overflow = 1;
        }
        ++i;
        o += b[k] - a[k];
      }
    }
    my_new = warp_sum(my_new);
    my_m = warp_sum(my_m);
    if (lane_id() == 0 && my_new) {
      atomicAdd(&S.n_new, my_new);
      atomicAdd(&S.m_new, my_m);
    }
    __syncthreads();
    ++levels;
    push_edges += E;
    const uint32_t nn = S.n_new;
    const unsigned long long mn = S.m_new;
    const unsigned long long cn = S.cnt[cur ^ 1];
    const bool ovf = S.overflow != 0;
    __syncthreads();  // everyone has read the counters before thread 0 resets them
    if (nn == 0) { ecc = L; break; }       // condition 2
    reached += nn;
    explored += mn;
    ++L;
    cur ^= 1;
    if (reached + 1 >= max_reach || L + 1 >= p.n) { ecc = L; break; }  // condition 1 / Q8
    if (ovf || (cn >> 32) == 0) {
      if ((cn >> 32) == 0) continue;  // frontier of out-degree-0 vertices: next level is empty
      // ---- hand over: frontier L (cnt cn) becomes k_sssp's queue 0, level state published
      const uint32_t q = (uint32_t)(cn >> 32), qe = (uint32_t)cn;
      for (uint32_t i = tid; i < min(q, kNarrowCap); i += NT) {
        p.Lv0[i] = S.u[cur][i];
        p.Lsd0[i] = make_uint2(S.rs[cur][i], S.off[cur][i]);
      }
      __syncthreads();
      // chunk map for all q entries (edge offsets are exclusive and monotone in slot order)
      for (uint32_t i = tid; i < q; i += NT) {
        const uint2 sd = (i < kNarrowCap) ? make_uint2(S.rs[cur][i], S.off[cur][i]) : __ldcg(p.Lsd0 + i);
        const uint32_t o = sd.y;
        const uint32_t e = (i + 1 < q) ? ((i + 1 < kNarrowCap) ? S.off[cur][i + 1] : __ldcg(p.Lsd0 + i + 1).y) : qe;
        for (uint32_t c = (o + kChunk - 1) / kChunk; c * kChunk < e; ++c) p.Cf0[c] = i;
      }
      if (tid == 0) {
        for (int k = 0; k < 3; ++k) C->slot[k] = Slot{0, 0, 0, 0, 0};
        Slot &s = C->slot[L % 3];
        s.n_new = nn;
        s.qpack = cn;
        s.m_new = mn;
        C->examined = 0;
        LevelState st{};
        st.L = L;
        st.prev_nf = 0;
        st.dir = kPush;
        st.rep = kRepQueue;
        st.q = 0;
        st.b = 0;
        st.push_levels = levels;
        st.reached = reached - nn;      // the header of level L adds nn again
        st.explored = explored - mn;    // ... and mn
        st.push_edges = push_edges;
        const uint4 *s4 = reinterpret_cast<const uint4 *>(&st);
        uint4 *d4 = reinterpret_cast<uint4 *>(C->solo_state);
        for (int k = 0; k < (int)(sizeof(LevelState) / 16); ++k) d4[k] = s4[k];
      }
      status = 2;
      break;
    }
  }
  if (tid == 0) {
    if (status == 1 && p.stats) {
      dawn_sssp_stats s;
      s.levels = ecc;
      s.reached = reached;
      s.edges_reach = explored;
      s.edges_examined = push_edges;
      s.push_levels = levels;
      s.pull_levels = 0;
      *p.stats = s;
    }
    C->narrow_status = status;
    C->solo_epoch = 0;  // k_sssp skips its init on hand-over: its solo stretches count from 0
    __threadfence();
    st_release(&C->narrow_seq, p.seq);
  }
}

}  // namespace dawn

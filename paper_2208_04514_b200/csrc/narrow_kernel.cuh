// narrow_kernel.cuh — high-diameter graphs (BASELINE configs[2]: the 4096 x 4096 grid, 8,191
// levels of <= 4,096 vertices).  Level-synchronous DAWN is latency-bound there:
// a level is a dependent chain frontier row -> target -> visited test -> enqueue, and the
// grid-wide kernel pays a grid barrier plus ~7 global round trips for it (7.7 us per level).
//
// k_narrow runs the search on ONE 16-CTA thread-block cluster (non-portable size; 16 SMs of one
// GPC) and keeps every piece of per-level state on chip:
//   * the visited bitmap (the "distance[col[j]] = 0" filter of Algorithm 2 line 6, reading Q1)
//     is spread over the 16 CTAs' shared memory (2 MB for n = 2^24 = 128 KB per CTA); a claim is
//     one DSMEM atomic OR (236 cycles, scripts/dsmem_bench.cu) instead of an L2 atomic;
//   * owner computes: a frontier vertex is queued at, and expanded by, the CTA that owns its
//     visited word.  On meshes and road networks (ids follow space) a vertex's neighbours share
//     its word or sit a multiple of 16 words away — the same owner — so claims are local
//     shared-memory atomics (0.14 cycles/op vs 3.14 for DSMEM, scripts/dsmem_bench.cu) and
//     only word-boundary arcs go remote; the frontier spreads over the 16 owners word by word;
//   * per-level counters travel by DSMEM exchange; levels are separated by a relaxed
//     barrier.cluster (181 cycles) — no grid barrier, no global counters.
// The only global round trip per level is the row itself, from the "augmented arc" array
// arc[j] = (col[j], row_ptr[col[j]], row_ptr[col[j] + 1]) built at load, so a discovered
// vertex's row bounds arrive with the arc that discovers it (no separate row_ptr round trip),
// and the new vertex's row is prefetched into L2 right away.  Each level is the SOVM step
// (Algorithm 2): frontier rows expanded, targets claimed, distance L+1.
// The arc back to the vertex's own discoverer is skipped (it is visited by construction).
//
// The other clusters of the launch only initialise dist and the hand-over bitmaps (a grid-wide
// fill) and exit; cluster 0 waits for that fill before its first level.  If a CTA's next
// frontier outgrows its shared queue, the overflowing vertices go straight to a global frontier
// bitmap, and at the end of that level the cluster hands over: queue entries join the bitmap,
// the visited slices are written to the global bitmap, the level state is published, and
// k_sssp — enqueued by dawn_sssp right behind k_narrow — resumes from the bitmap.  When the
// search ends inside k_narrow, k_sssp exits at once.
#pragma once
#include <cooperative_groups.h>

#include "sssp_kernel.cuh"

namespace dawn {

#ifndef DAWN_NARROW_PROF
#define DAWN_NARROW_PROF 0  // experiment: per-stage cycle stamps of the entry-0 lane (trace builds)
#endif
#ifndef DAWN_NARROW_RELEASE
#define DAWN_NARROW_RELEASE 0  // experiment: release/acquire level barrier
#endif
#ifndef DAWN_NARROW_CG
#define DAWN_NARROW_CG 0  // experiment: arc loads ld.global.cg instead of .nc
#endif
#ifndef DAWN_NARROW_TMA
#define DAWN_NARROW_TMA 1  // stage rows with one TMA bulk copy each (else 16-B cp.async pieces)
#endif
#ifndef DAWN_NARROW_PF2
#define DAWN_NARROW_PF2 0  // experiment: L2 prefetch of every target row before its claim (C3: 19.8 -> 27.7 ms)
#endif
#ifndef DAWN_NARROW_CBAR
#define DAWN_NARROW_CBAR 0  // experiment: exchange by returning atomics + barrier.cluster
#endif
#ifndef DAWN_NARROW_NOPF
#define DAWN_NARROW_NOPF 0  // experiment: no L2 prefetch of a discovered vertex's row
#endif
#ifndef DAWN_NARROW_NT
#define DAWN_NARROW_NT 512
#endif
constexpr uint32_t kNarrowThreads = DAWN_NARROW_NT;  // (cluster size, slice, degree limits: layout.h)

struct NarrowParams {
  uint32_t n, nwords;
  uint32_t wpc;     // visited words per CTA (word w lives in CTA w % 16 at index w / 16)
  uint32_t qcap;    // queue entries per buffer per CTA
  const uint32_t *rp;
  const uint4 *arc;  // (target, target row start, target row end, 0) per arc, or NULL:
  const int32_t *col;  //   then targets come from col and their rows from rp (two round trips)
  uint32_t owner;      // 1: owner computes (mesh-like ids); 0: a CTA queues what it discovers
  unsigned long long handover_m;  // hand over once the next frontier has more arcs than this
  const uint32_t *noin;
  uint32_t *vis, *dist, *fb0, *fb1;
  Ctrl *ctrl;
  dawn_sssp_stats *stats;
  uint32_t source, max_reach_base, seq;  // max_reach_base = #vertices with an in-edge
  const uint32_t *src_dev;               // source id on the device (dawn_sssp_batch) or NULL
  const uint32_t *vsrc;                  // dawn_sssp_batch: the whole device source list,
  uint32_t vn;                           //   validated before any write (vn = 0: none)
  TraceRec *trace;                 // per-level trace (DAWN_GRAPH_TRACE) or NULL
};

// shared memory: [NarrowCtl][vis slice: wpc words][queue 0: qcap uint4][queue 1: qcap uint4]
//                [row arcs 0: qcap x kNarrowStage uint4][row arcs 1: same]
// queue entry = (vertex, row start, row end, discoverer | staged << 31); a "staged" entry's
// arcs (rows of <= kNarrowStage arcs) were copied into its row-arcs slot by cp.async in the
// level that discovered it, so expanding it needs no global load.
constexpr uint32_t kNarrowBig = 64;  // long rows per CTA per level listed for CTA-wide expansion
struct NarrowCtl {
  unsigned long long rbase[kNarrowCluster];  // generic address of CTA r's shared window
  uint32_t qn[2];                 // entries appended to this CTA's queue b (may exceed qcap)
  uint32_t n_new, m_new;          // discoveries made by this CTA this level, out-degree sum
  uint32_t ovf, pad;              // this CTA overflowed a queue this level
  // per-level exchange, written by CTA r into slot r of every CTA before the cluster barrier
  // slot [b][r] = (CTA r's discoveries | overflow << 31, their out-degree sum)
  uint2 x[2][kNarrowCluster];
  unsigned long long mbar[2];     // level barrier b = L & 1 (phase parity (L >> 1) & 1)
  uint32_t nbig[2];               // rows of > 16 arcs of level L in nbig[L & 1] (expanded by the
                                  // whole CTA); level L resets nbig[(L+1) & 1], last read at L-1
  uint4 big[kNarrowBig];          // (vertex, row start, row end, discoverer)
};
constexpr size_t kNarrowCtlBytes = (sizeof(NarrowCtl) + 255) & ~size_t(255);

constexpr uint32_t kNarrowStage = 4;  // rows this short travel with their queue entry
constexpr size_t kNarrowEntryBytes = 2 * (16 + 16 * kNarrowStage);  // both buffers
inline size_t narrow_smem_bytes(uint32_t wpc, uint32_t qcap) {
  return kNarrowCtlBytes + 4 * (size_t)wpc + kNarrowEntryBytes * (size_t)qcap;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
// Level barrier of k_narrow.  Relaxed arrive: a release arrive waits for every outstanding
// global store of the thread (the level's scattered dist writes: +2,650 cycles measured,
// scripts/dsmem_bench.cu), while everything a peer reads after the barrier was completed
// before arriving — the exchange slots by returning atomics whose results were consumed,
// the queue entries by local stores ordered by __syncthreads, the visited words by atomics.
__device__ __forceinline__ void cluster_sync_level() {
#if DAWN_NARROW_RELEASE
  cluster_sync_all();
#else
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;"
               ::: "memory");
#endif
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint4 ld_nc4(const uint4 *p) {
  uint4 r;
#if DAWN_NARROW_CG
  asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
#else
  asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
#endif
  return r;
}
// Bulk L2 prefetch of a discovered vertex's whole row (every sector: a plain prefetch.global.L2
// brings only the first 32-B sector, and the row's second sector then missed L2 on demand —
// half of all arc loads, ncu lts__t_sectors_srcunit_tex_op_read_lookup_miss).
__device__ __forceinline__ void prefetch_row_l2(const uint4 *p, uint32_t n) {
  const uint32_t bytes = 16u * min(n, 256u);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t cluster_map(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  } while (!done);
}
// a location of CTA r's shared memory, by byte offset from the start of its dynamic smem
template <class T>
__device__ __forceinline__ T *remote(const NarrowCtl &S, uint32_t r, size_t off) {
  return reinterpret_cast<T *>(S.rbase[r] + off);
}

// Arc j as (target, target row start, target row end): one load from the augmented arc array,
// else col then row_ptr (two dependent loads).
__device__ __forceinline__ uint4 narrow_arc(const NarrowParams &p, uint32_t j) {
  if (p.arc) return ld_nc4(p.arc + j);
  const uint32_t u = (uint32_t)ld_nc(p.col + j);
  const uint2 r = make_uint2(ld_nc(p.rp + u), ld_nc(p.rp + u + 1));
  return make_uint4(u, r.x, r.y, 0u);
}

// One arc per lane, of the row of frontier vertex `parent` (whose own discoverer is `skip`):
// claim the target (shared-memory atomic OR on its visited word when this CTA owns the word,
// DSMEM atomic otherwise), write its distance, and append it to its owner's next queue.
// Local appends: one shared atomic per warp, slots from a ballot; the new entry's row (<= 4
// arcs) is copied into its row-arcs slot by cp.async.  Remote appends: a DSMEM slot
// reservation and the entry written by four returning atomics (complete before this thread
// reaches the level barrier), row prefetched into L2.  Overflowing entries go straight to the
// hand-over frontier bitmap.  Warp-collective.
__device__ __forceinline__ void narrow_visit(const NarrowParams &p, NarrowCtl &S, uint32_t *vis_s,
                                             uint32_t rank, uint32_t L1, uint32_t nxt,
                                             size_t qnxt_off, uint4 *qn_buf, uint4 *an_buf,
                                             uint4 a, bool act, uint32_t parent, uint32_t skip,
                                             uint32_t &n_new, uint32_t &m_new, uint32_t lvl_bar) {
  act = act && a.x != skip;  // the row owner's discoverer is visited: skip that arc
  const uint32_t w = a.x >> 5, o = w % kNarrowCluster, bit = 1u << (a.x & 31);
  const bool loc = o == rank;           // claim in this CTA's visited slice
  const bool qloc = loc || !p.owner;    // append to this CTA's queue
  uint32_t old = ~0u;
  if (act) {
    old = loc ? atomicOr(vis_s + w / kNarrowCluster, bit)
              : atomicOr(remote<uint32_t>(S, o, kNarrowCtlBytes + 4 * (size_t)(w / kNarrowCluster)),
                         bit);
  }
  const bool fresh = !(old & bit);
  const uint32_t d = a.z - a.y;
  const bool put = fresh && d > 0;
  if (fresh) {
    p.dist[a.x] = L1;
    n_new += 1;
    m_new += d;
  }
  const uint32_t bl = __ballot_sync(DAWN_FULL, put && qloc);
  if (bl) {
    uint32_t base = 0;
    if (lane_id() == 0) base = atomicAdd(&S.qn[nxt], (uint32_t)__popc(bl));
    const uint32_t slot = __shfl_sync(DAWN_FULL, base, 0) + __popc(bl & lanemask_lt());
    if (put && qloc) {
      if (slot < p.qcap) {
        const bool stage = p.arc && d <= kNarrowStage;
        qn_buf[slot] = make_uint4(a.x, a.y, a.z, parent | (stage ? 0x80000000u : 0u));
        if (stage) {
          const uint32_t dst =
              (uint32_t)__cvta_generic_to_shared(an_buf + (size_t)slot * kNarrowStage);
#if DAWN_NARROW_TMA
          // one TMA bulk copy of the whole row, completing on this level's barrier
          asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;"
                       ::"r"(lvl_bar), "r"(16u * d) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
                       " [%0], [%1], %2, [%3];"
                       ::"r"(dst), "l"(p.arc + a.y), "r"(16u * d), "r"(lvl_bar) : "memory");
#else
#pragma unroll
          for (uint32_t i = 0; i < kNarrowStage; ++i)
            if (i < d)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;"
                           ::"r"(dst + 16 * i), "l"(p.arc + a.y + i) : "memory");
#endif
        } else if (p.arc) {
          prefetch_row_l2(p.arc + a.y, d);
        }
      } else {
        red_or(p.fb0 + (a.x >> 5), bit);
        S.ovf = 1;
      }
    }
  }
  if (put && !qloc) {
    const uint32_t s2 = atomicAdd(remote<uint32_t>(S, o, offsetof(NarrowCtl, qn) + 4 * nxt), 1u);
    if (s2 < p.qcap) {
      uint32_t *e = remote<uint32_t>(S, o, qnxt_off + 16 * (size_t)s2);
      const uint32_t r0 = atomicExch(e, a.x), r1 = atomicExch(e + 1, a.y);
      const uint32_t r2 = atomicExch(e + 2, a.z), r3 = atomicExch(e + 3, parent);
      if ((r0 ^ r1 ^ r2 ^ r3) == 0x9e3779b9u) S.pad = 1;  // consume the results
      if (p.arc) prefetch_row_l2(p.arc + a.y, d);
    } else {
      red_or(p.fb0 + (a.x >> 5), bit);
      S.ovf = 1;
    }
  }
}

__global__ void __launch_bounds__(kNarrowThreads, 1) k_narrow(NarrowParams p) {
  extern __shared__ __align__(16) unsigned char smraw[];
  NarrowCtl &S = *reinterpret_cast<NarrowCtl *>(smraw);
  uint32_t *vis_s = reinterpret_cast<uint32_t *>(smraw + kNarrowCtlBytes);
  const size_t q0off = kNarrowCtlBytes + 4 * (size_t)p.wpc;  // byte offset of queue 0
  uint4 *qbuf0 = reinterpret_cast<uint4 *>(smraw + q0off);
  uint4 *abuf0 = qbuf0 + 2 * (size_t)p.qcap;  // row arcs of the staged entries
  Ctrl *C = p.ctrl;
  if (p.vn) {  // every CTA checks the whole batch list first: a bad id -> nothing written
    bool bad = false;
    for (uint32_t i = threadIdx.x; i < p.vn; i += kNarrowThreads) bad |= ld_nc(p.vsrc + i) >= p.n;
    if (__syncthreads_or(bad)) {
      if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&C->bad_src, 1u);
      return;
    }
  }
  const uint32_t src = p.src_dev ? ld_nc(p.src_dev) : p.source, tid = threadIdx.x;
  const uint32_t gtid = blockIdx.x * kNarrowThreads + tid, nthreads = gridDim.x * kNarrowThreads;

  // ---- a1 init, grid-wide: dist <- UNREACHED (d(s) = 0); hand-over bitmaps cleared
  for (uint32_t i = gtid; i < p.n; i += nthreads) p.dist[i] = (i == src) ? 0u : kUnreached;
  for (uint32_t w = gtid; w < p.nwords; w += nthreads) {
    p.fb0[w] = 0;
    p.fb1[w] = 0;
  }
  if (p.trace) {  // every record k_narrow may use (it runs at most n levels)
    const uint32_t ntr = min(p.n + 1, kTraceCap - 1);
    for (uint32_t i = gtid; i < ntr; i += nthreads) {
      p.trace[i].t_first = ~0ull;
      p.trace[i].t_last = 0;
      for (int k = 0; k < 4; ++k) p.trace[i].cyc[k] = 0;
    }
  }
  __syncthreads();
  // fill ticket: every launch of this graph handle adds exactly gridDim.x, so the launch owning
  // ticket t is complete once the counter reaches (t / gridDim.x + 1) * gridDim.x (no host-side
  // epoch: the launch stays correct when replayed from a CUDA graph)
  unsigned long long fill_target = 0;
  if (tid == 0) {
    __threadfence();
    const unsigned long long t = atomicAdd(&C->narrow_fill, 1ull);
    fill_target = (t / gridDim.x + 1) * (unsigned long long)gridDim.x;
  }
  if (cluster_id_x() != 0) return;

  // ---- cluster 0: visited slice <- no-in-edge | {s}; the source entry in CTA 0's queue 0
  const uint32_t rank = cluster_rank();
  for (uint32_t i = tid; i < p.wpc; i += kNarrowThreads) {
    const uint32_t w = i * kNarrowCluster + rank;
    uint32_t x = (w < p.nwords) ? ld_nc(p.noin + w) : ~0u;
    if (w == (src >> 5)) x |= 1u << (src & 31);
    vis_s[i] = x;
  }
  const uint32_t rs0 = ld_nc(p.rp + src), re0 = ld_nc(p.rp + src + 1);
  if (tid < kNarrowCluster)
    S.rbase[tid] = reinterpret_cast<unsigned long long>(
        cooperative_groups::this_cluster().map_shared_rank(reinterpret_cast<void *>(smraw), tid));
  if (tid == 0) {
    // level barrier b completes when all 16 CTAs' slot stores (st.async, 8 B each) landed, this
    // thread arrived with the expected bytes, and every thread's row copies (cp.async) landed
    for (int b = 0; b < 2; ++b)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;"
                   ::"r"(smem_u32(&S.mbar[b])), "r"(kNarrowThreads + 1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    S.qn[0] = S.qn[1] = 0;
    S.n_new = S.m_new = S.ovf = 0;
    S.nbig[0] = S.nbig[1] = 0;
    if (((src >> 5) % kNarrowCluster) == rank && re0 > rs0) {  // the source's owner queues it
      qbuf0[0] = make_uint4(src, rs0, re0, 0x7fffffffu);
      S.qn[0] = 1;
    }
    while (ld_acquire64(&C->narrow_fill) < fill_target) {
    }
    fence_acq_rel_gpu();
  }
  cluster_sync_all();

  const uint32_t lane = lane_id(), warp = tid / 32;
  constexpr uint32_t nwarp = kNarrowThreads / 32;
  const uint32_t max_reach = p.max_reach_base + ((ld_nc(p.noin + (src >> 5)) >> (src & 31)) & 1u);
  uint32_t L = 0, cur = 0, reached = 0, ecc = 0, levels = 0, prev_n = 1, status = 1;
  unsigned long long explored = re0 - rs0, push_edges = 0, mf = re0 - rs0;
  for (;;) {
    const uint32_t nxt = cur ^ 1;
    const uint4 *qcur = qbuf0 + (size_t)cur * p.qcap;
    const size_t qnxt_off = q0off + 16 * (size_t)nxt * p.qcap;
    uint4 *qnxt = qbuf0 + (size_t)nxt * p.qcap;
    const uint4 *acur = abuf0 + (size_t)cur * p.qcap * kNarrowStage;
    uint4 *anxt = abuf0 + (size_t)nxt * p.qcap * kNarrowStage;
    const uint32_t nq = min(S.qn[cur], p.qcap);  // this CTA's share of frontier L
    const uint32_t L1 = L + 1;
    const uint32_t lvl_bar = smem_u32(&S.mbar[L & 1]);  // this level's barrier (row copies land)
#if DAWN_NARROW_TMA
    // the row slots the TMA writes this level were last read (generic proxy) two levels ago
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#endif
    uint32_t n_new = 0, m_new = 0;
    long long tc0 = 0;
    if (p.trace && tid == 0) {
      tc0 = clock64();
      if (rank == 0 && L < kTraceCap) {
        p.trace[L].t_ns = globaltimer();
        p.trace[L].level = L;
        p.trace[L].dir = 0;
        p.trace[L].nf = prev_n;
        p.trace[L].pad = 8;  // narrow
        p.trace[L].mf = mf;
        C->trace_n = L + 1;
      }
    }
#if DAWN_NARROW_PROF
    long long ts[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    const bool prof = p.trace && nq > 0 && tid == 0;
    if (prof) ts[0] = clock64();
#endif
    // Four lanes per frontier entry (8 entries per warp round), one arc per lane per round:
    // rows of <= 4 arcs (meshes, road networks) take one round, their arcs read from the
    // entry's staged row slot; rows of 5..16 arcs take up to four rounds from global memory;
    // longer rows are expanded by the whole warp, 32 arcs per round.
    for (uint32_t base = warp * 8; base < nq; base += nwarp * 8) {
      const uint32_t g = base + lane / 4, k0 = lane & 3;
      const uint4 e = (g < nq) ? qcur[g] : make_uint4(0u, 0u, 0u, 0u);
#if DAWN_NARROW_PROF
      if (prof && base == 0 && lane == 0) ts[1] = clock64() + (e.x == 0x12345u ? 1 : 0);
#endif
      const uint32_t d = e.z - e.y, skip = e.w & 0x7fffffffu;
      const bool big = d > 16, staged = e.w >> 31;
      for (uint32_t k = k0; __any_sync(DAWN_FULL, !big && k < d); k += 4) {
        const bool act = !big && k < d;
        const uint4 a = !act ? make_uint4(0u, 0u, 0u, 0u)
                        : staged ? acur[(size_t)g * kNarrowStage + k] : narrow_arc(p, e.y + k);
#if DAWN_NARROW_PF2
        // two hops ahead: the target's row goes to L2 now; if the claim below wins, its TMA
        // staging copy (issued a few hundred cycles later) then reads L2, not HBM
        if (p.arc && act && a.x != skip && a.z > a.y) prefetch_row_l2(p.arc + a.y, a.z - a.y);
#endif
#if DAWN_NARROW_PROF
        if (prof && base == 0 && lane == 0 && ts[2] == 0) {
          uint32_t x = a.x;
          asm volatile("mov.u32 %0, %0;" : "+r"(x));
          ts[2] = clock64() + (x == 0x12345u ? 1 : 0);
        }
#endif
        narrow_visit(p, S, vis_s, rank, L1, nxt, qnxt_off, qnxt, anxt, a, act, e.x, skip, n_new,
                     m_new, lvl_bar);
#if DAWN_NARROW_PROF
        if (prof && base == 0 && lane == 0 && ts[4] == 0) ts[4] = ts[3] = clock64();
#endif
      }
      // rows of > 16 arcs: listed for the CTA-wide pass below (a row beyond the list's
      // capacity is expanded by this warp alone)
      uint32_t bm = __ballot_sync(DAWN_FULL, big && k0 == 0);
      while (bm) {
        const uint32_t k = __ffs(bm) - 1;
        bm &= bm - 1;
        const uint4 eb = make_uint4(__shfl_sync(DAWN_FULL, e.x, k), __shfl_sync(DAWN_FULL, e.y, k),
                                    __shfl_sync(DAWN_FULL, e.z, k), __shfl_sync(DAWN_FULL, skip, k));
        uint32_t slot = 0;
        if (lane == 0) slot = atomicAdd(&S.nbig[L & 1], 1u);
        slot = __shfl_sync(DAWN_FULL, slot, 0);
        if (slot < kNarrowBig) {
          if (lane == 0) S.big[slot] = eb;
          continue;
        }
        for (uint32_t jj = eb.y; jj < eb.z; jj += 32) {
          const bool act = jj + lane < eb.z;
          const uint4 a = act ? narrow_arc(p, jj + lane) : make_uint4(0u, 0u, 0u, 0u);
          narrow_visit(p, S, vis_s, rank, L1, nxt, qnxt_off, qnxt, anxt, a, act, eb.x, eb.w, n_new,
                       m_new, lvl_bar);
        }
      }
    }
    // ---- level totals: warp reductions into this CTA's counters
    auto fold = [&]() {
      n_new = __reduce_add_sync(DAWN_FULL, n_new);
      m_new = __reduce_add_sync(DAWN_FULL, m_new);
      if (lane == 0 && n_new) {
        atomicAdd(&S.n_new, n_new);
        atomicAdd(&S.m_new, m_new);
      }
      n_new = m_new = 0;
    };
    fold();
    __syncthreads();
    if (S.nbig[L & 1]) {  // uniform after the barrier: listed long rows, one arc per thread per round
      const uint32_t nb = min(S.nbig[L & 1], kNarrowBig);
      for (uint32_t b = 0; b < nb; ++b) {
        const uint4 eb = S.big[b];
        for (uint32_t j0 = eb.y + warp * 32; j0 < eb.z; j0 += kNarrowThreads) {
          const bool act = j0 + lane < eb.z;
          const uint4 a = act ? narrow_arc(p, j0 + lane) : make_uint4(0u, 0u, 0u, 0u);
          narrow_visit(p, S, vis_s, rank, L1, nxt, qnxt_off, qnxt, anxt, a, act, eb.x, eb.w, n_new,
                       m_new, lvl_bar);
        }
      }
      fold();
      __syncthreads();
    }
#if DAWN_NARROW_PROF
    if (prof) ts[5] = ts[6] = clock64();
#endif
    long long tc1 = 0;
    if (p.trace && tid == 0) {
      tc1 = clock64();
      if (L < kTraceCap) {
        atomicMax(&p.trace[L].cyc[2], (unsigned long long)(tc1 - tc0));
        if (rank == 0) p.trace[L].cyc[0] = tc1 - tc0;
      }
    }
    const uint32_t bb = L & 1;
    if (warp == 0) {
      const uint32_t xn = S.n_new | (S.ovf ? 0x80000000u : 0u), xm = S.m_new;
      __syncwarp();
      // queue `cur` has been read by this CTA only: it becomes the append target of level L+1
      // (peers append to it only after this level's barrier, which needs this CTA's slot)
      if (lane == 31) {
        S.n_new = S.m_new = S.ovf = 0;  // this level's local totals are sent below
        S.nbig[(L + 1) & 1] = 0;  // read for the last time at level L-1 (before its barrier)
        S.qn[cur] = 0;
      }
      __syncwarp();
#if DAWN_NARROW_CBAR
      if (lane < kNarrowCluster) {
        uint32_t *sl = remote<uint32_t>(S, lane, offsetof(NarrowCtl, x) + 8 * (bb * kNarrowCluster + rank));
        const uint32_t a = atomicExch(sl, xn), b = atomicExch(sl + 1, xm);
        if ((a ^ b) == 0x9e3779b9u) S.pad = 1;  // consume both results
      }
#else
      if (lane < kNarrowCluster) {
        const uint32_t dst = cluster_map(smem_u32(&S.x[bb][rank]), lane);
        const uint32_t bar = cluster_map(smem_u32(&S.mbar[bb]), lane);
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.u32 [%0], {%1, %2}, [%3];"
                     ::"r"(dst), "r"(xn), "r"(xm), "r"(bar) : "memory");
      }
#endif
    }
#if DAWN_NARROW_PROF
    if (prof) ts[7] = clock64();
#endif
#if DAWN_NARROW_CBAR
    cluster_sync_level();
    asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's row copies (next level)
    __syncthreads();  // also: every thread's row copies have landed
#else
    {
      const uint32_t bar = smem_u32(&S.mbar[bb]);
#if DAWN_NARROW_TMA
      asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}"
                   ::"r"(bar) : "memory");
#else
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
#endif
      if (tid == 0)
        asm volatile("{\n\t.reg .b64 st;\n\t"
                     "mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 st, [%0], %1;\n\t}"
                     ::"r"(bar), "r"(8u * kNarrowCluster) : "memory");
      mbar_wait(bar, (L >> 1) & 1);
    }
#endif
#if DAWN_NARROW_PROF
    if (prof) ts[8] = clock64();
#endif
    if (p.trace && tid == 0 && rank == 0 && L < kTraceCap) p.trace[L].cyc[1] = clock64() - tc1;
    // every warp folds the 16 slots itself (lane r < 16 reads CTA r's): totals and overflow
    const bool in = lane < kNarrowCluster;
    const uint2 xs = in ? S.x[bb][lane] : make_uint2(0u, 0u);
    const uint32_t N = __reduce_add_sync(DAWN_FULL, xs.x & 0x7fffffffu);
    const uint32_t O = __reduce_or_sync(DAWN_FULL, xs.x >> 31);
    const unsigned long long M =
        ((unsigned long long)__reduce_add_sync(DAWN_FULL, xs.y >> 16) << 16) +
        __reduce_add_sync(DAWN_FULL, xs.y & 0xffffu);
#if DAWN_NARROW_PROF
    if (prof && L < kTraceCap / 2) {
      ts[9] = clock64();
      uint32_t *o = reinterpret_cast<uint32_t *>(&p.trace[L + kTraceCap / 2].t_first);  // 12 u32
      for (int k = 1; k < 10; ++k) o[k - 1] = (uint32_t)(ts[k] - ts[0]);
      o[9] = rank;
    }
#endif
    ++levels;
    push_edges += mf;
    if (N == 0) { ecc = L; break; }  // condition 2: frontier empty
    reached += N;
    explored += M;
    mf = M;
    ++L;
    cur = nxt;
    if (reached + 1 >= max_reach || L + 1 >= p.n) { ecc = L; break; }  // condition 1 / Q8
    if (O || M > p.handover_m) {
      // ---- hand over frontier L (queues + overflow bitmap) to k_sssp: a queue overflowed, or
      // the frontier is wide enough for the grid-wide kernel (push or pull by its own rule)
      const uint32_t nq2 = min(S.qn[cur], p.qcap);
      const uint4 *q2 = qbuf0 + (size_t)cur * p.qcap;
      for (uint32_t i = tid; i < nq2; i += kNarrowThreads) {
        const uint32_t v = q2[i].x;
        red_or(p.fb0 + (v >> 5), 1u << (v & 31));
      }
      for (uint32_t i = tid; i < p.wpc; i += kNarrowThreads) {
        const uint32_t w = i * kNarrowCluster + rank;
        if (w < p.nwords) p.vis[w] = vis_s[i];
      }
      if (rank == 0 && tid == 0) {
        for (int k = 0; k < 3; ++k) C->slot[k] = Slot{0, 0, 0, 0, 0};
        Slot &s = C->slot[L % 3];
        s.n_new = N;
        s.m_new = M;
        C->examined = 0;
        LevelState st{};
        st.L = L;
        st.prev_nf = prev_n;
        st.dir = kPush;
        st.rep = kRepBitmap;
        st.q = 0;
        st.b = 0;
        st.push_levels = levels;
        st.reached = reached - N;    // the header of level L adds N again
        st.explored = explored - M;  // ... and M
        st.push_edges = push_edges;
        const uint4 *s4 = reinterpret_cast<const uint4 *>(&st);
        uint4 *d4 = reinterpret_cast<uint4 *>(C->solo_state);
        for (int k = 0; k < (int)(sizeof(LevelState) / 16); ++k) d4[k] = s4[k];
      }
      status = 2;
      break;
    }
    prev_n = N;
  }
#if DAWN_NARROW_PROF
  if (rank == 0 && tid == 0 && p.trace) C->trace_n = kTraceCap;  // stamps live at L + kTraceCap/2
#endif
  if (rank == 0 && tid == 0) {
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
  cluster_sync_all();  // no CTA exits while peers may still address its shared memory
}

}  // namespace dawn

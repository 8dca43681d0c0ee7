// layout.h — workspace layout shared by the host API (dawn.cu) and the kernels.
// Everything the library touches on the device lives in one caller-owned workspace.
#pragma once
#include <cstddef>
#include <cstdint>

#include "../../include/dawn.h"
#include "common.cuh"

namespace dawn {

// Push-mode frontier queue (SURVEY §2.5 k_push load balancing): every entry carries its row
// start and its exclusive edge offset within the frontier (allocated together with its slot
// by one 64-bit atomic per 32 entries), so the frontier's edges split into kChunk-edge chunks
// of equal size; Cf[c] names the entry holding chunk c's first edge.  Hub rows (64K arcs at
// scale 20) therefore spread over many warps with no separate heavy path.
constexpr uint32_t kChunk = 32;   // Cf granularity = one warp round
#ifndef DAWN_ILP
#define DAWN_ILP 4
#endif
#ifndef DAWN_ILP_CAND
#define DAWN_ILP_CAND 8  // chunks per warp item of a candidate (bitmap) push level
#endif
constexpr uint32_t kIlp = DAWN_ILP;      // chunks per warp item when the frontier is wide
// Solo levels (DAWN_PARAM_SOLO_EDGES): a narrow push level runs on CTA 0 alone with
// __syncthreads instead of the grid barrier (the other CTAs wait for the stretch to end).
// Bitmap push (DAWN_PARAM_BITMAP_PUSH_EDGES): a wide push level marks candidates with
// fire-and-forget red.or into a bitmap and settles them in a word-owner filter pass.
// Static heavy rows (built once at load): rows with degree > kHeavy are scanned in kHPiece-edge
// pieces by whole warps in the pull step and in the 64-source kernel; lighter rows are scanned
// by one lane each (early exit, 4 probes per round trip).
constexpr uint32_t kHeavy = 32;
constexpr uint32_t kHPiece = 256;
constexpr uint32_t kHeavyProbe = 16;
constexpr uint32_t kTopK = 8;  // in-row prefix ordered by in-neighbour out-degree (pull probes)  // in-edges a heavy row probes lane-parallel in the sweep
constexpr uint32_t kScanBlock = 2048;  // elements per CTA in the load-time piece scan
constexpr uint32_t kMaxBlocks = 2048;  // cap on persistent grid size (partials buffer)
constexpr uint32_t kTraceCap = 1 << 16;
// k_narrow (narrow_kernel.cuh): one 16-CTA cluster, visited bitmap in distributed shared memory
constexpr uint32_t kNarrowCluster = 16;            // CTAs per cluster (non-portable size)
constexpr uint32_t kNarrowVisBytes = 160 * 1024;   // max visited-slice bytes per CTA
constexpr uint64_t kNarrowMaxN = (uint64_t)kNarrowCluster * kNarrowVisBytes * 8;  // 20,971,520
constexpr uint32_t kNarrowMaxAvgDeg = 8;           // arc array kept when m <= 8 n
// Multi-source kernel: kMsW 64-bit words per vertex = kMsBatch sources per adjacency pass.
#ifndef DAWN_MS_W
#define DAWN_MS_W 4  // 64-bit words per vertex of the multi-source kernel
#endif
#ifndef DAWN_MS_NT
#define DAWN_MS_NT 640  // threads per CTA of k_ms64 (20 warps at 96 registers, spill-free; C5 512 -> 640: 843K -> 894K sources/s)
#endif
constexpr int kMsW = DAWN_MS_W;
constexpr int kMsNT = DAWN_MS_NT;
constexpr uint32_t kMsBatch = 64 * kMsW;

static_assert(kMsBatch == DAWN_MS_BATCH, "dawn.h DAWN_MS_BATCH must match kMsW");

#ifndef DAWN_PULL_DEEP
#define DAWN_PULL_DEEP 1  // 8-probe pull rounds on sparse frontiers
#endif
#ifndef DAWN_SSSP_MINB
#define DAWN_SSSP_MINB 2  // __launch_bounds__ min blocks of k_sssp: 2 x 16 warps per SM (64 regs)
#endif
#ifndef DAWN_PULL_DEEP_PR
#define DAWN_PULL_DEEP_PR 8  // in-edges probed per lane per round trip on sparse frontiers
#endif
#ifndef DAWN_PULL_PR
#define DAWN_PULL_PR 4       // ... on dense frontiers
#endif
// The same two for the 2-CTA/SM (64-register) variant: fewer probes in flight per lane keep its
// pull loop free of spills, and the doubled warp count supplies the parallelism (Kronecker-24
// 1224 -> 1323 GTEPS with 2 / 4 instead of 4 / 8)
#ifndef DAWN_PULL_DEEP_PR2
#define DAWN_PULL_DEEP_PR2 4
#endif
#ifndef DAWN_PULL_PR2
#define DAWN_PULL_PR2 2
#endif
#ifndef DAWN_PULL_J2
#define DAWN_PULL_J2 2  // DAWN_PULL_J of the 2-CTA/SM variant
#endif
// Push levels read a bitmap frontier directly (no conversion to a queue) when none of its rows
// is longer than kDirectRow arcs (DAWN_DIRECT_PUSH=0: always convert).
constexpr uint32_t kDirectRow = 256;
#ifndef DAWN_MINB2_EXTRAS
#define DAWN_MINB2_EXTRAS 0  // direct bitmap push and next-row prefill in the 2-CTA/SM variant too
#endif
#ifndef DAWN_DIRECT_PUSH
#define DAWN_DIRECT_PUSH 1
#endif
#ifndef DAWN_CAND_FILTER
#define DAWN_CAND_FILTER 0   // experiment: 1 weak / 2 L2 load of the candidate word before each
#endif                       // bitmap-push reduction (slower on C2 and C4)
#ifndef DAWN_HEAVY_ILP
#define DAWN_HEAVY_ILP 1     // in-edges per lane in flight when a warp scans a heavy pull piece
#endif
#ifndef DAWN_NOVIS
#define DAWN_NOVIS 1       // candidate push levels skip the visited read while few are settled
#endif
#ifndef DAWN_NOVIS2
#define DAWN_NOVIS2 1      // ... also in the 64-register kernel (4 chunks per item there)
#endif
#ifndef DAWN_NOVIS_FRAC
#define DAWN_NOVIS_FRAC 32  // ... while (reached + 1) * FRAC < reachable vertices (C4 1325 -> 1350 GTEPS; 8: forced push C2 -9%)
#endif
#ifndef DAWN_PULL_HLIST
#define DAWN_PULL_HLIST 1  // pull pieces phase: only the heavy in-rows the light pass left
#endif
#ifndef DAWN_PULL_SPLIT
#define DAWN_PULL_SPLIT 1  // pull level = light pass, grid barrier, heavy pieces (C4 +4.5%)
#endif
#ifndef DAWN_PULL_TOP1
#define DAWN_PULL_TOP1 1  // pull sweep: the first in-neighbour from a per-vertex array
#endif
#ifndef DAWN_PULL_PREFETCH
#define DAWN_PULL_PREFETCH 1  // pull sweep: unreached-list entries loaded one iteration ahead
#endif
#ifndef DAWN_PULL_J
#define DAWN_PULL_J 2  // vis words per warp iteration of the pull sweep (independent scans)
#endif

enum : uint32_t { kPush = 0, kPull = 1, kRepQueue = 0, kRepBitmap = 1 };

struct Slot {                 // counters of one frontier (3 rotate: written, read, reset)
  uint32_t n_new;             // vertices discovered into this frontier
  uint32_t big;               // 1: a vertex of this (bitmap) frontier has > kDirectRow arcs
  unsigned long long qpack;   // queue: (entries << 32) | edges  (push-mode representation)
  unsigned long long m_new;   // sum of out-degrees of the frontier (m_f)
  unsigned long long pad1;
};

struct Ctrl {
  GridBarrier bar;
  uint32_t pad0[12];
  Slot slot[3];
  unsigned long long examined;  // per-source accumulator (reduced per CTA)
  uint32_t n_hasin;             // #vertices with in-degree > 0 (written at load)
  uint32_t err;                 // graph validation result (written at load)
  uint32_t n_hp_out, n_hp_in;   // static heavy-piece counts (written at load)
  uint32_t trace_n;
  uint32_t solo_epoch;          // CTA 0 -> others: a solo stretch ended (see k_sssp)
  uint32_t narrow_status;       // k_narrow -> k_sssp: 1 finished, 2 resume from the bitmap
  uint32_t narrow_seq;          // dawn_sssp call number the status belongs to
  unsigned long long narrow_fill;  // k_narrow: CTAs done with the init fill (monotonic)
  uint32_t bad_src;             // sticky: a dawn_sssp_batch device source id was >= n
  uint32_t wcc_cnt, wcc_arcs, wcc_root, wcc_k;  // dawn_largest_wcc selection / output size
  uint32_t claim;               // lane 0's: next unclaimed index of a dawn_sssp_batch call
  uint32_t next_idx;            // the batch index this lane searches next
  uint32_t hl_cnt[2];           // pull level L: heavy in-rows the light pass left (parity L & 1)
  alignas(16) unsigned char solo_state[256];  // LevelState snapshot published with solo_epoch
};

struct MsCtrl {
  GridBarrier bar;
  uint32_t pad0[12];
  unsigned long long cnt[3][4];   // per level slot: [0] n_active, [1] m_active, [2] m_full
  // executed-schedule counters, accumulated over launches until dawn_graph_ms_counters reads
  // them: [0] levels, [1] adjacency entries gathered (push arcs + pull probes), [2] word
  // reductions issued (red.or.b64), [3] batches
  unsigned long long stat[4];
  uint32_t pad1[8];
};

// One trace record per level of the last traced dawn_sssp call (DAWN_TRACE=1).
struct TraceRec {
  unsigned long long t_ns;  // %globaltimer at the level start (after the barrier)
  uint32_t level, dir, nf, pad;
  unsigned long long mf;
  unsigned long long t_first, t_last;  // first / last CTA done with the level's work
  unsigned long long cyc[4];           // sum over warps of clock64 cycles: [0] light/push work,
                                       // [1] heavy pull pieces, [2] flush, [3] conversions
};

struct HeavyList {  // static pieces of rows with degree > kHeavy
  size_t v, s, e, bits;
};

// dawn_sssp_batch lanes: the grid-wide kernel's per-search state, replicated so that up to
// kMaxLanes cooperative launches (one per lane, each on its own share of the SMs and its own
// stream) run independent searches of one batch at the same time (sources are
// independent).  Lane 0 is the state every other call uses.
constexpr int kMaxLanes = 16;   // allocated: 16 up to 2^22 vertices, 8 above (make_layout)
constexpr int kMsMaxLanes = 4;
#ifndef DAWN_MS_LANES
#define DAWN_MS_LANES 4  // default multi-source lanes (C5: 1 -> 707K, 2 -> 815K, 3 -> 829K, 4 -> 847K sources/s)
#endif  // multi-source lanes allocated (<= kMaxLanes)
struct LaneLayout {
  size_t vis, cand, fb[3], Lv[2], Lsd[2], Cf[2], ctrl, ulist, useg;
};

// Multi-source lanes: the bit-parallel kernel's per-batch state, replicated so that several
// k_ms64 launches (one per lane, each on its own share of the SMs and its own stream) run
// different 256-source batches of one msssp / apsp call at the same time.
struct MsLaneLayout {
  size_t seen, F0, F1, nxt, msctrl, part, srcbuf;
};

struct Layout {
  size_t rp, irp, noin, vis, cand, fb[3], Lv[2], Lsd[2], Cf[2], ctrl, trace;
  LaneLayout lane[kMaxLanes];
  int nlanes;
  MsLaneLayout ms[kMaxLanes];
  int ms_nlanes;
  HeavyList hout, hin;
  size_t scan_tmp, piece_tmp, hasin, ulist, useg, icol2, top1, arc;
  size_t seen, F0, F1, nxt, msctrl, part, srcbuf, total;
  uint64_t srccap, capCf, capHP;
  bool own_irp;
};

inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

inline Layout make_layout(int64_t n, int64_t m, uint32_t flags) {
  Layout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = align_up(o + (bytes ? bytes : 1));
    return at;
  };
  const uint64_t W = (uint64_t)(n + 31) / 32;
  L.capCf = (uint64_t)m / kChunk + 2;
  L.capHP = (uint64_t)m / kHPiece + (uint64_t)m / kHeavy + 1;
  L.own_irp = !(flags & DAWN_GRAPH_SYMMETRIC);
  const bool lean = flags & DAWN_GRAPH_LEAN;  // no ms64 words, no icol2, no augmented arcs
  L.rp = take(4 * (size_t)(n + 1));
  L.irp = L.own_irp ? take(4 * (size_t)(n + 1)) : L.rp;
  L.noin = take(4 * W);
  L.vis = take(4 * W);
  L.cand = take(4 * W);
  for (int i = 0; i < 3; ++i) L.fb[i] = take(4 * W);
  for (int i = 0; i < 2; ++i) {
    L.Lv[i] = take(4 * (size_t)n);
    L.Lsd[i] = take(8 * (size_t)n);
    L.Cf[i] = take(4 * L.capCf);
  }
  L.ctrl = take(sizeof(Ctrl));
  L.trace = take(sizeof(TraceRec) * kTraceCap);
  auto heavy = [&](HeavyList &h) {
    h.v = take(4 * L.capHP);
    h.s = take(4 * L.capHP);
    h.e = take(4 * L.capHP);
    h.bits = take(4 * W);
  };
  heavy(L.hout);
  if (L.own_irp) heavy(L.hin); else L.hin = L.hout;
  L.scan_tmp = take(4 * ((size_t)n / kScanBlock + 2));
  L.piece_tmp = take(4 * (3 * ((size_t)m / kHPiece + 3) + 1));
  L.hasin = take(4 * (size_t)n);
  L.ulist = take(4 * (size_t)n);
  L.useg = take(4 * (size_t)kMaxBlocks * 32);
  L.icol2 = (lean || m == 0) ? 0 : take(4 * (size_t)m);  // in-rows, highest-degree in-neighbours first
  // k_narrow's augmented arcs (target, target row start, target row end, 0): low-degree graphs
  L.arc = (!lean && m > 0 && (uint64_t)n <= kNarrowMaxN &&
           (uint64_t)m <= (uint64_t)kNarrowMaxAvgDeg * (uint64_t)n)
              ? take(16 * (size_t)m) : 0;
  L.msctrl = take(sizeof(MsCtrl));
  L.srccap = (uint64_t)(n > 65536 ? n : 65536);
  if (!lean) {
    L.seen = take(8 * kMsW * (size_t)n);
    L.F0 = take(8 * kMsW * (size_t)n);
    L.F1 = take(8 * kMsW * (size_t)n);
    L.nxt = take(8 * kMsW * (size_t)n);
    L.part = take(sizeof(uint32_t) * 4 * kMsBatch * 2 * kMaxBlocks);
    L.srcbuf = take(4 * L.srccap);
  }
  L.ms[0] = MsLaneLayout{L.seen, L.F0, L.F1, L.nxt, L.msctrl, L.part, L.srcbuf};
  // extra multi-source lanes up to 2^22 vertices (their 4 x 32-byte words per vertex stay
  // L2-resident next to the graph), none in lean mode
  L.ms_nlanes = lean ? 1 : ((uint64_t)n <= (1ull << 22) ? kMsMaxLanes : 1);
  for (int l = 1; l < L.ms_nlanes; ++l) {
    MsLaneLayout &q = L.ms[l];
    q.seen = take(8 * kMsW * (size_t)n);
    q.F0 = take(8 * kMsW * (size_t)n);
    q.F1 = take(8 * kMsW * (size_t)n);
    q.nxt = take(8 * kMsW * (size_t)n);
    q.msctrl = take(sizeof(MsCtrl));
    q.part = take(sizeof(uint32_t) * 4 * kMsBatch * 2 * kMaxBlocks);
    q.srcbuf = take(4 * L.srccap);
  }
  // extra lanes (lane 0 = the arrays above): not in lean mode; 4 lanes up to 2^22 vertices
  // (latency-bound searches overlap best), 2 above
  L.nlanes = lean ? 1 : ((uint64_t)n <= (1ull << 22) ? kMaxLanes : 8);
  L.lane[0] = LaneLayout{L.vis, L.cand, {L.fb[0], L.fb[1], L.fb[2]}, {L.Lv[0], L.Lv[1]},
                         {L.Lsd[0], L.Lsd[1]}, {L.Cf[0], L.Cf[1]}, L.ctrl, L.ulist, L.useg};
  for (int l = 1; l < L.nlanes; ++l) {
    LaneLayout &q = L.lane[l];
    q.vis = take(4 * W);
    q.cand = take(4 * W);
    for (int i = 0; i < 3; ++i) q.fb[i] = take(4 * W);
    for (int i = 0; i < 2; ++i) {
      q.Lv[i] = take(4 * (size_t)n);
      q.Lsd[i] = take(8 * (size_t)n);
      q.Cf[i] = take(4 * L.capCf);
    }
    q.ctrl = take(sizeof(Ctrl));
    q.ulist = take(4 * (size_t)n);
    q.useg = take(4 * (size_t)kMaxBlocks * 32);
  }
  // the first entry of every degree-ordered in-row (0xffffffff: empty row), read beside the
  // row offsets so a pull probe of it needs no in-row sector; last, so the other arrays keep
  // their offsets
  L.top1 = L.icol2 ? take(4 * (size_t)n) : 0;
  L.total = o;
  return L;
}

}  // namespace dawn

// layout.h — workspace layout shared by the host API (dawn.cu) and the kernels.
// Everything the library touches on the device lives in one caller-owned workspace.
#pragma once
#include <cstddef>
#include <cstdint>

#include "../../include/dawn.h"
#include "common.cuh"

namespace dawn {

// Light/heavy split of push-mode frontier entries (SURVEY §2.5 k_push load balancing):
// rows with deg <= kLight go to 32-entry warp groups; longer rows are cut into kPiece-edge
// pieces that warps take independently (hub rows: max degree 64K at scale 20, 406K at 24).
constexpr uint32_t kLight = 128;
constexpr uint32_t kPiece = 512;

enum : uint32_t { kPush = 0, kPull = 1, kRepQueue = 0, kRepBitmap = 1 };

struct Slot {                 // counters of one frontier (3 rotate: written, read, reset)
  uint32_t n_new;             // vertices discovered into this frontier
  uint32_t n_light;           // queue entries (push-mode representation)
  uint32_t n_heavy;
  uint32_t n_pieces;
  unsigned long long m_new;   // sum of out-degrees of the frontier (m_f)
  unsigned long long pad;
};

struct Ctrl {
  GridBarrier bar;
  uint32_t pad0[14];
  Slot slot[3];
  unsigned long long examined;  // per-source accumulator (reduced per CTA)
  uint32_t n_hasin;             // #vertices with in-degree > 0 (written at load)
  uint32_t err;                 // graph validation result (written at load)
  uint32_t pad1[12];
};

constexpr uint32_t kMaxBlocks = 2048;  // cap on persistent grid size (partials buffer)

struct MsCtrl {
  GridBarrier bar;
  uint32_t pad0[14];
  unsigned long long cnt[3][4];   // per level slot: [0] n_active words, [1] m_active, [2] any new
  uint32_t pad1[8];
};

struct Layout {
  size_t rp, irp, noin, vis, fb0, fb1, Lv[2], Lsd[2], Hv[2], Hsd[2], Hp[2], Pm[2], ctrl;
  size_t seen, F0, F1, nxt, msctrl, part, srcbuf, total;
  uint64_t srccap;
  uint64_t capH, capP;
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
  L.capH = (uint64_t)m / kLight + 1;
  L.capP = (uint64_t)m / kPiece + L.capH + 1;
  L.own_irp = !(flags & DAWN_GRAPH_SYMMETRIC);
  L.rp = take(4 * (size_t)(n + 1));
  L.irp = L.own_irp ? take(4 * (size_t)(n + 1)) : L.rp;
  L.noin = take(4 * W);
  L.vis = take(4 * W);
  L.fb0 = take(4 * W);
  L.fb1 = take(4 * W);
  for (int i = 0; i < 2; ++i) {
    L.Lv[i] = take(4 * (size_t)n);
    L.Lsd[i] = take(8 * (size_t)n);
    L.Hv[i] = take(4 * L.capH);
    L.Hsd[i] = take(8 * L.capH);
    L.Hp[i] = take(4 * L.capH);
    L.Pm[i] = take(4 * L.capP);
  }
  L.ctrl = take(sizeof(Ctrl));
  L.seen = take(8 * (size_t)n);
  L.F0 = take(8 * (size_t)n);
  L.F1 = take(8 * (size_t)n);
  L.nxt = take(8 * (size_t)n);
  L.msctrl = take(sizeof(MsCtrl));
  L.part = take(sizeof(uint32_t) * 4 * 64 * 2 * kMaxBlocks);
  L.srccap = (uint64_t)(n > 65536 ? n : 65536);
  L.srcbuf = take(4 * L.srccap);
  L.total = o;
  return L;
}

}  // namespace dawn

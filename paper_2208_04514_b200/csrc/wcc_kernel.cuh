// wcc_kernel.cuh — the largest weakly connected component on the device (dawn_largest_wcc).
//
// PAPER.md Table 1 (L95-98) characterises every graph by its largest WCC (S_wcc nodes, E_wcc
// arcs) and APSP (E11-E12, L303-308) runs over that component's vertices (BASELINE north_star).
// Lock-free union-find: every arc (v, u) joins the components of v and u (a directed arc joins
// them too: weak connectivity); roots are hooked larger-onto-smaller by CAS, so par[x] <= x
// always holds and a root is the minimum id of its component.  Then per-root node / arc counts
// (warp-aggregated atomics), a three-pass selection (most nodes, then most arcs, then smallest
// root = minimum vertex id: DESIGN.md reading Q15) and an order-preserving compaction.
#pragma once
#include "layout.h"

namespace dawn {

// Root of x with path halving.  par[] only ever decreases and stays inside x's tree, so the
// concurrent shortcut stores are benign (each one still points at an ancestor).
__device__ __forceinline__ uint32_t wcc_find(uint32_t *par, uint32_t x) {
  uint32_t cur = ld_cg(par + x);
  if (cur != x) {
    uint32_t prev = x, next;
    while (cur > (next = ld_cg(par + cur))) {
      par[prev] = next;
      prev = cur;
      cur = next;
    }
  }
  return cur;
}

__device__ __forceinline__ void wcc_union(uint32_t *par, uint32_t a, uint32_t b) {
  uint32_t ra = wcc_find(par, a), rb = wcc_find(par, b);
  while (ra != rb) {
    const uint32_t hi = max(ra, rb), lo = min(ra, rb);
    const uint32_t old = atomicCAS(par + hi, hi, lo);
    if (old == hi) break;  // hooked
    ra = wcc_find(par, old);  // hi stopped being a root meanwhile: retry from its new root
    rb = wcc_find(par, lo);
  }
}

__global__ void k_wcc_init(uint32_t *par, uint32_t n) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    par[v] = v;
}

// Light rows (degree <= kHeavy): one thread per vertex.  Heavy rows go through the static
// 256-arc piece list (k_wcc_hook_pieces), so a hub row is spread over many warps.
__global__ void k_wcc_hook_light(const uint32_t *__restrict__ rp, const int32_t *__restrict__ col,
                                 uint32_t n, uint32_t *par) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint32_t s = rp[v], e = rp[v + 1];
    if (e - s > kHeavy) continue;
    for (uint32_t j = s; j < e; ++j) {
      const uint32_t u = (uint32_t)col[j];
      if (u != v) wcc_union(par, v, u);
    }
  }
}

__global__ void k_wcc_hook_pieces(const uint32_t *__restrict__ hv, const uint32_t *__restrict__ hs,
                                  const uint32_t *__restrict__ he, const uint32_t *npieces,
                                  const int32_t *__restrict__ col, uint32_t *par) {
  const uint32_t np = *npieces;
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t pc = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; pc < np;
       pc += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t v = hv[pc];
    for (uint32_t j = hs[pc] + lane; j < he[pc]; j += 32) {
      const uint32_t u = (uint32_t)col[j];
      if (u != v) wcc_union(par, v, u);
    }
  }
}

// Root of x without path compression (the forest is final: no writes, so concurrent readers
// never see an entry move).
__device__ __forceinline__ uint32_t wcc_root(const uint32_t *par, uint32_t x) {
  uint32_t cur = x, next;
  while ((next = ld_cg(par + cur)) != cur) cur = next;
  return cur;
}

// Final labels lab[v] = root (= component minimum) and per-root node / arc counts (cnt, arcs
// zeroed).  The labels go to a separate array: rewriting par[v] here raced with concurrent
// path-halving stores of the same entry (a stale ancestor could overwrite the root).
__global__ void k_wcc_count(const uint32_t *__restrict__ rp, uint32_t n, const uint32_t *par,
                            uint32_t *__restrict__ lab, uint32_t *cnt, uint32_t *arcs) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += stride) {
    const uint32_t v = base + threadIdx.x;
    const bool in = v < n;
    const uint32_t r = in ? wcc_root(par, v) : 0xffffffffu;
    if (in) lab[v] = r;
    const uint32_t d = in ? rp[v + 1] - rp[v] : 0u;
    // warp aggregation: one atomic pair per distinct root in the warp (the giant component's
    // root would otherwise take one same-address atomic per vertex).  The __match_any groups
    // are disjoint and each member passes its group's mask.
    const uint32_t peers = __match_any_sync(DAWN_FULL, r);
    const uint32_t ds = __reduce_add_sync(peers, d);
    if (in && (threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) {
      atomicAdd(cnt + r, (uint32_t)__popc(peers));
      atomicAdd(arcs + r, ds);
    }
  }
}

// Selection passes over the roots (lab[v] == v).  pass 0: max nodes; pass 1: max arcs among
// max-node roots; pass 2: min root among those.
__global__ void k_wcc_select(const uint32_t *__restrict__ lab, const uint32_t *__restrict__ cnt,
                             const uint32_t *__restrict__ arcs, uint32_t n, int pass, Ctrl *C) {
  const uint32_t bc = pass > 0 ? ld_cg(&C->wcc_cnt) : 0u;
  const uint32_t ba = pass > 1 ? ld_cg(&C->wcc_arcs) : 0u;
  uint32_t best = pass == 2 ? 0xffffffffu : 0u;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (lab[v] != v) continue;
    if (pass == 0) best = max(best, cnt[v]);
    else if (pass == 1) { if (cnt[v] == bc) best = max(best, arcs[v]); }
    else if (cnt[v] == bc && arcs[v] == ba) best = min(best, v);
  }
  for (int o = 16; o; o >>= 1) {
    const uint32_t y = __shfl_xor_sync(DAWN_FULL, best, o);
    best = pass == 2 ? min(best, y) : max(best, y);
  }
  if ((threadIdx.x & 31) == 0) {
    if (pass == 0 && best) atomicMax(&C->wcc_cnt, best);
    if (pass == 1 && best) atomicMax(&C->wcc_arcs, best);
    if (pass == 2 && best != 0xffffffffu) atomicMin(&C->wcc_root, best);
  }
}

// Order-preserving compaction of {v : lab[v] == root}: per-block counts, a serial scan of the
// block counts (k_hscan), then each block writes its vertices ascending.
__global__ void k_wcc_bcount(const uint32_t *__restrict__ lab, uint32_t n, const Ctrl *C,
                             uint32_t *__restrict__ tmp) {
  __shared__ uint32_t sm[32];
  const uint32_t root = ld_cg(&C->wcc_root);
  const uint32_t base = blockIdx.x * kScanBlock;
  uint32_t c = 0;
  for (uint32_t i = threadIdx.x; i < kScanBlock; i += blockDim.x) {
    const uint32_t v = base + i;
    if (v < n && lab[v] == root) ++c;
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x / 32] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (uint32_t i = 0; i < blockDim.x / 32; ++i) t += sm[i];
    tmp[blockIdx.x] = t;
  }
}

__global__ void k_wcc_bfill(const uint32_t *__restrict__ lab, uint32_t n, const Ctrl *C,
                            const uint32_t *__restrict__ tmp, uint32_t *__restrict__ out) {
  __shared__ uint32_t sm[256];
  constexpr uint32_t kPer = kScanBlock / 256;  // blockDim.x == 256
  const uint32_t root = ld_cg(&C->wcc_root);
  const uint32_t v0 = blockIdx.x * kScanBlock + threadIdx.x * kPer;
  uint32_t c = 0;
  for (uint32_t i = 0; i < kPer; ++i)
    if (v0 + i < n && lab[v0 + i] == root) ++c;
  sm[threadIdx.x] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t run = tmp[blockIdx.x];
    for (uint32_t i = 0; i < blockDim.x; ++i) {
      const uint32_t x = sm[i];
      sm[i] = run;
      run += x;
    }
  }
  __syncthreads();
  uint32_t o = sm[threadIdx.x];
  for (uint32_t i = 0; i < kPer; ++i) {
    const uint32_t v = v0 + i;
    if (v < n && lab[v] == root) out[o++] = v;
  }
}

}  // namespace dawn

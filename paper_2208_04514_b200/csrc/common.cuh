// common.cuh — device helpers for the DAWN B200 kernels (sm_100a).
// Grid barrier, cache-policy loads, warp scans.  No DAWN arithmetic lives here.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define DAWN_FULL 0xffffffffu

namespace dawn {

constexpr uint32_t kUnreached = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// Read-only for the whole kernel (graph arrays): non-coherent texture path.
__device__ __forceinline__ uint32_t ld_nc(const uint32_t *p) {
  uint32_t r;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ int32_t ld_nc(const int32_t *p) {
  int32_t r;
  asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_nc2(const uint32_t *p) {  // 8-B aligned pair
  uint2 r;
  asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
// Mutable data written by other CTAs in an EARLIER phase (after a grid barrier): L2 only.
__device__ __forceinline__ uint32_t ld_cg(const uint32_t *p) {
  uint32_t r;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ unsigned long long ld_cg(const unsigned long long *p) {
  unsigned long long r;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_cg2(const uint2 *p) {
  uint2 r;
  asm volatile("ld.global.cg.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
  uint32_t r;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_or(uint32_t *p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_or64(unsigned long long *p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.or.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Sense-free generation barrier across all CTAs of a cooperative launch.
// count/gen live in the workspace control block; gen only grows.
struct GridBarrier {
  uint32_t count;
  uint32_t gen;
};

__device__ __forceinline__ void grid_sync(GridBarrier *b, uint32_t nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (nblocks > 1) {
      uint32_t gen = ld_acquire(&b->gen);
      __threadfence();
      uint32_t arrived = atomicAdd(&b->count, 1u);
      if (arrived == nblocks - 1) {
        b->count = 0;
        st_release(&b->gen, gen + 1);
      } else {
        while (ld_acquire(&b->gen) == gen) {
        }
      }
    }
    __threadfence();  // invalidates this SM's L1 (CCTL.IVALL): later weak loads see peers' data
  }
  __syncthreads();
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(DAWN_FULL, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  return x;
}

template <class T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(DAWN_FULL, x, o);
  return x;
}

// Record hash term of SURVEY §8(c): splitmix64 finaliser of (v << 32 | d).
__device__ __forceinline__ unsigned long long rec_hash(uint32_t v, uint32_t d) {
  unsigned long long z = (((unsigned long long)v) << 32) | d;
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace dawn

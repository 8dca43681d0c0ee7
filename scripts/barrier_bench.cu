// Microbenchmark of grid-barrier designs for the persistent kernels (run on the B200 box).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bb scripts/barrier_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct Bar { unsigned int count, gen; unsigned long long mono; unsigned int flags[4096]; unsigned long long subs[16 * 16]; };

__device__ __forceinline__ unsigned ld_acq(const unsigned *p) { unsigned r; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory"); return r; }
__device__ __forceinline__ unsigned long long ld_acq64(const unsigned long long *p) { unsigned long long r; asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory"); return r; }
__device__ __forceinline__ void st_rel(unsigned *p, unsigned v) { asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ unsigned long long atom_add_rel64(unsigned long long *p, unsigned long long v) { unsigned long long r; asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(v) : "memory"); return r; }
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned *p, unsigned v) { unsigned r; asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory"); return r; }
__device__ __forceinline__ void fence_acqrel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// V0: current (threadfence + atomicAdd + gen spin + threadfence)
__device__ void bar0(Bar *b, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned gen = ld_acq(&b->gen);
    __threadfence();
    unsigned a = atomicAdd(&b->count, 1u);
    if (a == nb - 1) { b->count = 0; st_rel(&b->gen, gen + 1); }
    else while (ld_acq(&b->gen) == gen) {}
    __threadfence();
  }
  __syncthreads();
}
// V1: acq_rel atomic on count, gen release, acquire spin, fence.acq_rel at the end
__device__ void bar1(Bar *b, unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned gen = ld_acq(&b->gen);
    unsigned a = atom_add_acqrel(&b->count, 1u);
    if (a == nb - 1) { b->count = 0; st_rel(&b->gen, gen + 1); }
    else while (ld_acq(&b->gen) == gen) {}
    fence_acqrel();
  }
  __syncthreads();
}
// V2: monotonic 64-bit counter, spin until >= target
__device__ void bar2(Bar *b, unsigned nb, unsigned long long &target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += nb;
    atom_add_rel64(&b->mono, 1ull);
    while (ld_acq64(&b->mono) < target) {}
    fence_acqrel();
  }
  __syncthreads();
}
// V3: flag array: each CTA writes its flag (release), CTA 0 gathers (warp-parallel), then gen
__device__ void bar3(Bar *b, unsigned nb, unsigned &epoch) {
  __syncthreads();
  epoch++;
  if (blockIdx.x == 0) {
    if (threadIdx.x < 32) {
      for (unsigned i = threadIdx.x + 1; i < nb; i += 32) while (ld_acq(&b->flags[i]) != epoch) {}
      __syncwarp();
      if (threadIdx.x == 0) st_rel(&b->gen, epoch);
    }
  } else if (threadIdx.x == 0) {
    st_rel(&b->flags[blockIdx.x], epoch);
    while (ld_acq(&b->gen) != epoch) {}
  }
  if (threadIdx.x == 0) fence_acqrel();
  __syncthreads();
}

__device__ __forceinline__ void red_add_rel64(unsigned long long *p, unsigned long long v) { asm volatile("red.release.gpu.global.add.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory"); }
// V4: the production barrier (common.cuh grid_sync): red.release on one monotonic counter
__device__ void bar4(Bar *b, unsigned nb, unsigned long long &target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += nb;
    red_add_rel64(&b->mono, 1ull);
    while (ld_acq64(&b->mono) < target) {}
    fence_acqrel();
  }
  __syncthreads();
}
// V5/V6: S monotonic sub-counters on separate 128-byte lines (CTA b arrives on b mod S, no
// same-address serialisation of the arrivals); lanes 0..S-1 of warp 0 poll them in parallel
template <int S>
__device__ void barS(Bar *b, unsigned nb, unsigned long long &target) {
  __syncthreads();
  if (threadIdx.x < 32) {
    target += nb;
    if (threadIdx.x == 0) red_add_rel64(&b->subs[16 * (blockIdx.x % S)], 1ull);
    for (;;) {
      unsigned long long v = threadIdx.x < S ? ld_acq64(&b->subs[16 * threadIdx.x]) : 0ull;
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (v >= target) break;
    }
    fence_acqrel();
  }
  __syncthreads();
}

template <int V>
__global__ void kbench(Bar *b, int iters, unsigned long long *out) {
  unsigned long long target = 0; unsigned epoch = 0;
  if (V == 2 && threadIdx.x == 0) target = 0;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (V == 0) bar0(b, gridDim.x);
    if (V == 1) bar1(b, gridDim.x);
    if (V == 2) bar2(b, gridDim.x, target);
    if (V == 3) bar3(b, gridDim.x, epoch);
    if (V == 4) bar4(b, gridDim.x, target);
    if (V == 5) barS<8>(b, gridDim.x, target);
    if (V == 6) barS<16>(b, gridDim.x, target);
    if (V == 7) barS<4>(b, gridDim.x, target);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

int main() {
  Bar *b; unsigned long long *out;
  cudaMalloc(&b, sizeof(Bar)); cudaMalloc(&out, 8);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int bps : {1, 2, 4}) {
    for (int v = 0; v < 8; ++v) {
      cudaMemset(b, 0, sizeof(Bar));
      int iters = 2000, grid = nsm * bps;
      void *args[] = {&b, &iters, &out};
      void *fns[] = {(void *)kbench<0>, (void *)kbench<1>, (void *)kbench<2>, (void *)kbench<3>,
                     (void *)kbench<4>, (void *)kbench<5>, (void *)kbench<6>, (void *)kbench<7>};
      void *fn = fns[v];
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaLaunchCooperativeKernel(fn, grid, 512, args, 0, 0);  // warm
      cudaMemset(b, 0, sizeof(Bar));
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      cudaLaunchCooperativeKernel(fn, grid, 512, args, 0, 0);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("bps=%d grid=%d V%d: %.3f us/barrier (%s)\n", bps, grid, v, ms * 1e3 / iters, cudaGetErrorString(err));
    }
  }
  // empty cooperative launch overhead
  {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 0; void *args[] = {&b, &iters, &out};
    for (int w = 0; w < 10; ++w) cudaLaunchCooperativeKernel((void *)kbench<0>, nsm * 2, 512, args, 0, 0);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int w = 0; w < 100; ++w) cudaLaunchCooperativeKernel((void *)kbench<0>, nsm * 2, 512, args, 0, 0);
    cudaEventRecord(e1); cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("empty cooperative launch (296x512): %.3f us each\n", ms * 1e3 / 100);
    cudaEventRecord(e0);
    for (int w = 0; w < 100; ++w) kbench<0><<<nsm * 2, 512>>>(b, 0, out);
    cudaEventRecord(e1); cudaDeviceSynchronize();
    cudaEventElapsedTime(&ms, e0, e1);
    printf("empty normal launch (296x512): %.3f us each\n", ms * 1e3 / 100);
  }
  return 0;
}

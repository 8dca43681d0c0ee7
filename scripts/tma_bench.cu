// Small-copy staging throughput on one SM (the k_narrow row staging question): K threads each
// stage one 64-byte row global -> shared, (a) one cp.async.bulk per row completing on an
// mbarrier, (b) four 16-byte cp.async per row.  Source rows random in a 1 GB buffer (HBM) or in
// a 4 MB one (L2).  Prints cycles from the first issue to the last byte landed.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bench scripts/tma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

template <int MODE>
__global__ void kb(const uint4 *src, uint32_t nrows, int K, int reps, unsigned long long *out) {
  __shared__ alignas(128) uint4 buf[512 * 4];
  __shared__ alignas(8) unsigned long long bar;
  const uint32_t tid = threadIdx.x;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  __syncthreads();
  unsigned long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    const long long t0 = clock64();
    if (MODE == 0) {
      if (tid == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(64u * K) : "memory");
      __syncthreads();
      if ((int)tid < K) {
        const uint32_t row = hash(tid * 7919 + r * 104729) % nrows;
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf + 4 * tid);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 64, [%2];"
                     ::"r"(dst), "l"(src + 4 * (size_t)row), "r"(b) : "memory");
      }
      if (tid == 0) {
        uint32_t done = 0;
        while (!done)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                       : "=r"(done) : "r"(b), "r"((uint32_t)(r & 1)) : "memory");
      }
    } else {
      if ((int)tid < K) {
        const uint32_t row = hash(tid * 7919 + r * 104729) % nrows;
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(buf + 4 * tid);
        for (int i = 0; i < 4; ++i)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16 * i), "l"(src + 4 * (size_t)row + i) : "memory");
      }
      asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
    }
    __syncthreads();
    tot += clock64() - t0;
  }
  if (tid == 0) *out = tot / reps + (buf[0].x == 0xdeadbeef);
}

int main() {
  uint4 *src; unsigned long long *out;
  const size_t bytes = (size_t)1 << 30;
  cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes); cudaMalloc(&out, 8);
  for (int l2 = 0; l2 < 2; ++l2) {
    const uint32_t nrows = l2 ? (4u << 20) / 64 : (uint32_t)(bytes / 64);
    for (int K : {1, 8, 32, 128, 256, 512}) {
      for (int mode = 0; mode < 2; ++mode) {
        void (*f)(const uint4 *, uint32_t, int, int, unsigned long long *) = mode ? kb<1> : kb<0>;
        f<<<1, 512>>>(src, nrows, K, 50, out);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long c; cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
        printf("%s K=%3d %-28s %7llu cycles (%5.1f per row) %s\n", l2 ? "L2 " : "HBM", K,
               mode ? "4x cp.async 16B per row" : "1 cp.async.bulk 64B per row", c, (double)c / K,
               cudaGetErrorString(e));
      }
    }
  }
  return 0;
}

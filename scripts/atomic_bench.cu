// atomic_bench.cu — cost of same-address returning 64-bit atomics from many warps at once
// (k_sssp's frontier-queue reservation `qpack`).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kat(unsigned long long *ctr, unsigned long long *out, int nwarps_active, int naddr, int ret) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if ((threadIdx.x & 31) == 0 && gw < nwarps_active) {
    long long t0 = clock64();
    unsigned long long r = 0;
    if (ret) r = atomicAdd(ctr + 16 * (gw % naddr), (1ull << 32) | 31);
    else asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(ctr + 16 * (gw % naddr)), "l"((1ull << 32) | 31) : "memory");
    if (r == 0xdeadbeef) out[1] = 1;
    out[2 + gw] = clock64() - t0;
  }
}
int main() {
  unsigned long long *ctr, *out;
  cudaMalloc(&ctr, 8 * 16 * 64); cudaMalloc(&out, 8 * 20000);
  for (int ret = 1; ret >= 0; --ret)
  for (int naddr : {1, 8}) for (int nw : {32, 385, 2000, 9472}) {
    cudaMemset(ctr, 0, 8 * 16 * 64); cudaMemset(out, 0, 8 * 20000);
    for (int it = 0; it < 3; ++it) kat<<<296, 512>>>(ctr, out, nw, naddr, ret);
    cudaDeviceSynchronize();
    unsigned long long h[20000]; cudaMemcpy(h, out, 8 * 20000, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0, sum = 0; for (int i = 0; i < nw; ++i) { mx = h[2 + i] > mx ? h[2 + i] : mx; sum += h[2 + i]; }
    printf("%s naddr=%d warps=%5d: max %8llu cyc, mean %8llu cyc\n", ret ? "atom" : "red ", naddr, nw, mx, sum / nw);
  }
  return 0;
}

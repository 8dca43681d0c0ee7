// dsmem_bench.cu — microbenchmarks behind k_narrow's design (16-CTA cluster, DSMEM state):
// remote atomic latency/throughput, remote loads, cluster barrier cost with and without
// outstanding global stores.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int CL = 16, NT = 1024, WORDS = 32768;  // 128 KB slice

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cmap(uint32_t a, uint32_t r) {
  uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o;
}
__device__ __forceinline__ uint32_t datom_or(uint32_t a, uint32_t v) {
  uint32_t o; asm volatile("atom.relaxed.cluster.shared::cluster.or.b32 %0, [%1], %2;" : "=r"(o) : "r"(a), "r"(v) : "memory"); return o;
}
__device__ __forceinline__ uint32_t dld(uint32_t a) {
  uint32_t o; asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(o) : "r"(a) : "memory"); return o;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void csync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t crank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t hash(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

// mode: 0 chain latency (thread 0), 1 remote atomic throughput, 2 remote load throughput,
// 3 local smem atomic throughput, 4 barrier (release), 5 barrier + global store before,
// 6 barrier relaxed, 7 L2-hit ld.global.nc.v4 chain latency, 8 remote atomic, only 256 threads
__global__ void kb(int mode, int reps, unsigned long long *out, uint32_t *gbuf, const uint4 *chase) {
  extern __shared__ uint32_t sm[];
  const uint32_t tid = threadIdx.x, rank = crank();
  for (int i = tid; i < WORDS; i += NT) sm[i] = 0;
  csync();
  const uint32_t base = smem_u32(sm);
  uint32_t acc = 0;
  long long t0 = clock64();
  if (mode == 0) {
    if (tid == 0 && rank == 0) {
      uint32_t x = 0;
      for (int i = 0; i < reps; ++i) x = datom_or(cmap(base + 4 * ((x + i * 97) % WORDS), (i + 1) % CL), 1u);
      acc = x;
    }
  } else if (mode == 1 || mode == 8) {
    if (mode == 1 || tid < 256) {
      for (int i = 0; i < reps; ++i) {
        uint32_t o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t h = hash(tid * 131 + rank * 7919 + i * 4 + k);
          o[k] = datom_or(cmap(base + 4 * (h % WORDS), (h >> 20) % CL), 1u << (h & 31));
        }
        acc += o[0] ^ o[1] ^ o[2] ^ o[3];
      }
    }
  } else if (mode == 2) {
    for (int i = 0; i < reps; ++i) {
      uint32_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t h = hash(tid * 131 + rank * 7919 + i * 4 + k);
        o[k] = dld(cmap(base + 4 * (h % WORDS), (h >> 20) % CL));
      }
      acc += o[0] ^ o[1] ^ o[2] ^ o[3];
    }
  } else if (mode == 3) {
    for (int i = 0; i < reps; ++i) {
      uint32_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t h = hash(tid * 131 + rank * 7919 + i * 4 + k);
        o[k] = atomicOr(sm + (h % WORDS), 1u << (h & 31));
      }
      acc += o[0] ^ o[1] ^ o[2] ^ o[3];
    }
  } else if (mode == 4) {
    for (int i = 0; i < reps; ++i) csync();
  } else if (mode == 5) {
    for (int i = 0; i < reps; ++i) {
      gbuf[(hash(tid + i * NT + rank * 1000003) & ((1u << 24) - 1))] = i;
      csync();
    }
  } else if (mode == 6) {
    for (int i = 0; i < reps; ++i) csync_relaxed();
  } else if (mode == 9) {
    for (int i = 0; i < reps; ++i) {
      gbuf[(hash(tid + i * NT + rank * 1000003) & ((1u << 24) - 1))] = i;
      csync_relaxed();
    }
  } else if (mode == 10) {
    uint32_t x = 0;
    for (int i = 0; i < reps; ++i) {
      if (tid < CL) {
        uint32_t o;
        asm volatile("atom.relaxed.cluster.shared::cluster.exch.b32 %0, [%1], %2;" : "=r"(o) : "r"(cmap(base + 4 * rank, tid)), "r"((uint32_t)i) : "memory");
        x += o;
      }
      asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
      if (x == 0xdeadbeef) sm[0] = 1;
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    }
    acc = x;
  } else if (mode == 11 || mode == 12) {
    // cold 1 GB buffer (big): load latency of line i (stride 1 MB + 4 KB), with (12) or
    // without (11) a prefetch.global.L2 issued ~4000 cycles earlier
    if (tid == 0 && rank == 0) {
      const uint4 *big = reinterpret_cast<const uint4 *>(gbuf);
      uint32_t x = 0;
      long long tot = 0;
      for (int i = 0; i < reps; ++i) {
        const uint4 *a = big + ((size_t)i * ((1 << 16) + 256) + (x & 1)) % ((size_t)1 << 26);
        if (mode == 12) asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
        long long w0 = clock64();
        while (clock64() - w0 < 4000) {
        }
        long long t = clock64();
        uint4 v;
        asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a));
        x += v.x;
        asm volatile("mov.u32 %0, %0;" : "+r"(x));
        tot += clock64() - t;
      }
      acc = x;
      out[100] = tot;
    }
  } else if (mode == 7) {
    if (tid == 0 && rank == 0) {
      uint32_t x = 0;
      for (int i = 0; i < reps; ++i) {
        uint4 v;
        asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(chase + x));
        x = v.x;
      }
      acc = x;
    }
  }
  long long t1 = clock64();
  csync();
  if (tid == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0) + (acc == 0xdeadbeef);
}

int main() {
  const int nb = CL;
  unsigned long long *out; uint32_t *gbuf; uint4 *chase;
  CK(cudaMalloc(&out, 8 * 256));
  CK(cudaMalloc(&gbuf, (size_t)1 << 30));
  CK(cudaMemset(gbuf, 0, (size_t)1 << 30));
  const size_t nch = 1 << 16;  // 1 MB: L2 resident
  CK(cudaMalloc(&chase, 16 * nch));
  uint4 *h = new uint4[nch];
  for (size_t i = 0; i < nch; ++i) h[i] = make_uint4((uint32_t)((i * 40503 + 7777) % nch), 0, 0, 0);
  CK(cudaMemcpy(chase, h, 16 * nch, cudaMemcpyHostToDevice));
  const size_t smb = 4 * WORDS;
  CK(cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
  CK(cudaFuncSetAttribute(kb, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  const char *names[] = {"remote atomic chain latency (cyc/op)", "remote atomic thpt (cyc per op per SM, 1024 thr x4)",
                         "remote load thpt (cyc per op per SM)", "local smem atomic thpt (cyc per op per SM)",
                         "cluster barrier release/acquire (cyc)", "barrier + 1 scattered global store/thread (cyc)",
                         "cluster barrier relaxed (cyc)", "L2-hit ld.global.nc.v4 chain latency (cyc)",
                         "remote atomic thpt, 256 threads (cyc per op per SM)",
                         "relaxed barrier + 1 scattered global store/thread (cyc)",
                         "16 returning remote exch + relaxed barrier (cyc)",
                         "cold 1GB ld.global.nc.v4 latency (cyc)",
                         "same after prefetch.global.L2 4000 cyc earlier (cyc)"};
  for (int mode = 0; mode <= 12; ++mode) {
    const int reps = (mode == 11 || mode == 12) ? 500 : (mode == 0 || mode >= 4) ? 2000 : 200;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(nb); cfg.blockDim = dim3(NT); cfg.dynamicSmemBytes = smb; cfg.attrs = at; cfg.numAttrs = 1;
    for (int w = 0; w < 2; ++w) CK(cudaLaunchKernelEx(&cfg, kb, mode, reps, out, gbuf, (const uint4 *)chase));
    CK(cudaDeviceSynchronize());
    unsigned long long c[CL];
    CK(cudaMemcpy(c, out, 8 * CL, cudaMemcpyDeviceToHost));
    double mx = 0; for (int i = 0; i < CL; ++i) mx = c[i] > mx ? c[i] : mx;
    double per = mx / reps;
    if (mode == 1 || mode == 2 || mode == 3) per = mx / (reps * 4.0 * NT);
    if (mode == 8) per = mx / (reps * 4.0 * 256);
    if (mode == 11 || mode == 12) {
      unsigned long long t; CK(cudaMemcpy(&t, out + 100, 8, cudaMemcpyDeviceToHost)); per = (double)t / reps;
    }
    printf("%-55s %8.2f\n", names[mode], per);
  }
  return 0;
}

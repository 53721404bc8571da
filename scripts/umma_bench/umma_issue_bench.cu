// Issue-cost microbenchmark: tcgen05.mma.cta_group::2 (M=256, N=128) with the B descriptor
// varying per MMA like a pipelined kernel (stage x K-step).  Variants:
//  0: full 64-bit descriptor computed per MMA in C++ (make_desc per instruction)
//  1: 64-bit base + per-MMA constant offset (64-bit add)
//  2: descriptor assembled inside the asm from a 32-bit low word + immediate high word
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// high word of an SW128 K-major descriptor with SBO = 1024: (1024>>4) | version 1<<14 | swizzle 2<<29
constexpr uint32_t kDescHi = (1024 >> 4) | (1u << 14) | (2u << 29);
__device__ __forceinline__ void mma_ts_lo(uint32_t d, uint32_t a, uint32_t blo, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 bd;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "mov.b64 bd, {%2, %5};\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], bd, %3, p;\n\t}" ::"r"(d),
      "r"(a), "r"(blo), "r"(idesc), "r"(acc), "n"(kDescHi));
}
template <int variant>
__global__ void __launch_bounds__(128, 1) bench(int iters, long long* out) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 96 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (tid == 0 && rank == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    const uint32_t sb = smem_u32(smem);
    const uint64_t db = make_desc(sb, 16, 1024);
    const uint32_t dlo = (uint32_t)db;
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
      const uint32_t st = (uint32_t)((i >> 3) % 5) * 16384;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = st + (kk >> 2) * 8192 + (kk & 3) * 32;
        const uint32_t d = tmem + (kk & 1) * 128, a = tmem + 384 + kk * 8;
        if constexpr (variant == 0) {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a),
                       "l"(make_desc(sb + off, 16, 1024)), "r"(idesc), "r"(1));
        } else if constexpr (variant == 1) {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a),
                       "l"(db + (uint64_t)(off >> 4)), "r"(idesc), "r"(1));
        } else if constexpr (variant == 2) {
          mma_ts_lo(d, a, dlo + (off >> 4), idesc, 1);
        } else {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
                       "r"(tmem + 384), "l"(db), "r"(idesc), "r"(1));
        }
      }
      if (variant >= 3 && (i & 15) == 8) {  // after every 16 MMAs: a gap of busy work
        const long long g0 = clock64();
        while (clock64() - g0 < (long long)(variant - 3) * 200) {
        }
      }
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)), "h"((unsigned short)3)
        : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    out[blockIdx.x / 2] = clock64() - t0;
  }
  if (tid == 0 && rank == 1) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (tid < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}
int main() {
  long long* d;
  cudaMalloc(&d, 74 * sizeof(long long));
  cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(bench<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(bench<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(bench<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(bench<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(bench<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(bench<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const char* names[9] = {"make_desc per MMA      ", "64-bit base + offset   ", "lo word + imm hi in asm",
                          "fixed, gap 0/16 MMAs   ", "fixed, gap 200/16 MMAs ", "fixed, gap 400/16 MMAs ",
                          "fixed, gap 600/16 MMAs ", "fixed, gap 800/16 MMAs ", "fixed, gap 1000/16 MMAs"};
  for (int v = 0; v < 9; ++v)
    for (int rep = 0; rep < 2; ++rep) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = 100 * 1024;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const int iters = 4096;
      switch (v) {
        case 0: cudaLaunchKernelEx(&cfg, bench<0>, iters, d); break;
        case 1: cudaLaunchKernelEx(&cfg, bench<1>, iters, d); break;
        case 2: cudaLaunchKernelEx(&cfg, bench<2>, iters, d); break;
        case 3: cudaLaunchKernelEx(&cfg, bench<3>, iters, d); break;
        case 4: cudaLaunchKernelEx(&cfg, bench<4>, iters, d); break;
        case 5: cudaLaunchKernelEx(&cfg, bench<5>, iters, d); break;
        case 6: cudaLaunchKernelEx(&cfg, bench<6>, iters, d); break;
        case 7: cudaLaunchKernelEx(&cfg, bench<7>, iters, d); break;
        default: cudaLaunchKernelEx(&cfg, bench<8>, iters, d); break;
      }
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
      long long h[74];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double cyc = 0;
      for (int i = 0; i < 74; ++i) cyc += h[i];
      printf("TS N=128 pair, %s: %.1f clk/MMA\n", names[v], cyc / 74 / iters);
    }
  return 0;
}

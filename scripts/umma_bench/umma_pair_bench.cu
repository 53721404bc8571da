// Microbenchmark: tcgen05.mma.cta_group::2 kind::f16 issue rate (M=256 = 128 rows per SM, K=16)
// for N in {64,128,256}, SS (A, B from shared memory) and TS (A from TMEM).  Clusters of 2 CTAs,
// one per SM; the leader's single thread issues `iters` MMAs back to back.
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
__global__ void __launch_bounds__(128, 1) bench(int n, int iters, int ts, long long* out, int vary, int warpmode) {
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
  for (int i = tid; i < 100 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (warpmode && tid < 32 && rank == 0) {  // whole warp walks the loop; elect.sync picks the issuer
    uint32_t idesc = (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
    const uint64_t da = make_desc(sa, 16, 1024), db = make_desc(sb, 16, 1024);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t bd = db + (uint64_t)((((i >> 3) % 4) * 16384 + (kk >> 2) * 8192 + (kk & 3) * 32) >> 4);
        if (ts)
          asm volatile(
              "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + (kk & 1) * 128),
              "r"(tmem + 384 + kk * 8), "l"(bd), "r"(idesc), "r"(1));
        else
          asm volatile(
              "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + (kk & 1) * 256),
              "l"(da + (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4)), "l"(bd), "r"(idesc), "r"(1));
      }
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            smem_u32(&bar)), "h"((unsigned short)3)
        : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x / 2] = t1 - t0;
  }
  if (!warpmode && tid == 0 && rank == 0) {
    uint32_t idesc = (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
    long long t0 = clock64();
    if (ts) {
      for (int i = 0; i < iters; ++i) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + (i & 1) * 128),
            "r"(tmem + 384 + (i & 7) * 8), "l"(vary ? make_desc(sb + ((i >> 3) % 4) * 16384 + ((i >> 2) & 1) * 8192 + (i & 3) * 32, 16, 1024) : make_desc(sb, 16, 1024)), "r"(idesc), "r"(1));
      }
    } else {
      for (int i = 0; i < iters; ++i) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + (i & 1) * 256),
            "l"(vary ? make_desc(sa + ((i >> 2) & 1) * 16384 + (i & 3) * 32, 16, 1024) : make_desc(sa, 16, 1024)),
            "l"(vary ? make_desc(sb + ((i >> 3) % 4) * 16384 + ((i >> 2) & 1) * 8192 + (i & 3) * 32, 16, 1024) : make_desc(sb, 16, 1024)), "r"(idesc), "r"(1));
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
    long long t1 = clock64();
    out[blockIdx.x / 2] = t1 - t0;
  }
  if (tid == 0 && rank == 1) {  // wait for the pair's MMAs before teardown
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
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024 + 1024);
  for (int vary = 0; vary < 3; ++vary)
  for (int ts = 0; ts < 2; ++ts)
    for (int n : {128}) {
      if (ts && n > 128) continue;
      const int iters = 4096;
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
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&cfg, bench, n, iters, ts, d, vary & 1, vary == 2);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        if (err != cudaSuccess) { printf("err %s\n", cudaGetErrorString(err)); return 1; }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        long long h[74];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double cyc = 0;
        for (int i = 0; i < 74; ++i) cyc += h[i];
        cyc /= 74;
        const double macs_sm = 128.0 * n * 16;  // per SM per instruction
        printf("%s pair %s N=%d: %.1f clk/MMA, %.0f MAC/clk/SM, event %.3f ms -> %.1f TFLOP/s (all SMs)\n", vary == 2 ? "warp+elect, base+const" : vary ? "varying addr" : "fixed addr  ", ts ? "TS" : "SS", n,
               cyc / iters, macs_sm * iters / cyc, ms, 2 * macs_sm * iters * 148 / (ms * 1e-3) / 1e12);
      }
    }
  return 0;
}

// tcgen05.mma issue/execute rate with operands walking a 5-stage smem ring (as a pipelined
// kernel does), random fp16 data, every SM busy.  cta_group 1 (M=128) or 2 (M=256), N 128/256,
// SS or TS (A from TMEM).  One thread per CTA (or pair) issues `iters` MMAs back to back.
#include <cstdint>
#include <cstdio>
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
template <int CG, int N, int TS, int VARY>
__global__ void __launch_bounds__(128, 1) bench(int iters, long long* out) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (tid < 32) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t x = 0x9E3779B9u * (tid + 1) + blockIdx.x;
  for (int i = tid; i < 200 * 1024 / 4; i += 128) {  // random halves in [-1, 1)
    x ^= x << 13; x ^= x >> 17; x ^= x << 5;
    const uint32_t a = 0x3800u | (x & 0x3ffu) | ((x >> 5) & 0x8000u), b = 0x3800u | ((x >> 10) & 0x3ffu) | ((x >> 16) & 0x8000u);
    reinterpret_cast<uint32_t*>(smem)[i] = a | (b << 16);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (TS) {  // A operand in TMEM columns [384, 448): fill from registers
    uint32_t v = 0x3c00bc00u ^ (tid * 0x00010001u);
    for (int c = 0; c < 64; ++c)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + 384 + c + ((uint32_t)((tid >> 5) * 32) << 16)), "r"(v ^ c));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  const int M = CG == 2 ? 256 : 128;
  if (tid == 0 && rank == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
      const uint32_t st = VARY ? (uint32_t)((i >> 3) % 5) * 32768 : 0;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t bd = make_desc(sb + st + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
        const uint32_t d = tmem + (N <= 128 ? (kk & 1) * N : 0);
        if (TS) {
          if (CG == 2)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(tmem + 384 + kk * 8), "l"(bd), "r"(idesc), "r"(1));
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(tmem + 384 + kk * 8), "l"(bd), "r"(idesc), "r"(1));
        } else {
          const uint64_t ad = make_desc(sa + (VARY ? ((i >> 3) & 1) * 16384 : 0) + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
          if (CG == 2)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(1));
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(1));
        }
      }
    }
    if (CG == 2)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "h"((unsigned short)3) : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    out[blockIdx.x] = clock64() - t0;
  }
  if (CG == 2 && tid == 0 && rank == 1) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (tid < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (CG == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}
template <int CG, int N, int TS, int VARY>
void run(long long* d) {
  auto k = bench<CG, N, TS, VARY>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int iters = 16384;
  for (int rep = 0; rep < 2; ++rep) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k, iters, d);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("err %s\n", cudaGetErrorString(err)); exit(1); }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double clk = 0; int n = 0;
    for (int i = 0; i < 148; i += CG) { clk += h[i]; ++n; }
    clk /= n;
    const int M = CG * 128;
    const double flops = 2.0 * M * N * 16 * iters * (148 / CG);
    printf("cta_group::%d M=%d N=%d %s %s: %.1f clk/MMA (ideal %d), %.1f TFLOP/s, %.2f GHz eff\n", CG, M, N, TS ? "TS" : "SS",
           VARY ? "walking" : "fixed  ", clk / iters, N / 2, flops / ms / 1e9, clk / ms / 1e6);
  }
}
int main(int argc, char**) {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  if (argc > 1) {  // N = 64 shapes only
    run<1, 64, 0, 1>(d); run<1, 64, 1, 1>(d); run<2, 64, 0, 1>(d); run<2, 64, 1, 1>(d); run<2, 128, 0, 1>(d);
    return 0;
  }
  run<1, 128, 0, 1>(d); run<1, 128, 1, 1>(d); run<1, 256, 0, 1>(d); run<1, 256, 1, 1>(d);
  run<2, 128, 0, 1>(d); run<2, 128, 1, 1>(d); run<2, 256, 0, 1>(d); run<2, 256, 1, 1>(d);
  run<2, 128, 1, 0>(d); run<1, 128, 1, 0>(d);
  return 0;
}

// Microbenchmark of the prefill softmax inner loop on one SM (no MMA): per iteration each
// thread tcgen05.ld's `cols` fp32 S values of its TMEM lane, (mode>=1) takes the row max,
// (mode>=2) computes 2^(s*c - m) with ex2.approx, packs f16 pairs and tcgen05.st's them back.
// Prints cycles per iteration for 4 / 8 active warps.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <int COLS>
__global__ void __launch_bounds__(288, 1) bench(int iters, int mode, int nwarps, long long* out, float* sink, int mma) {
  __shared__ uint32_t slot;
  __shared__ __align__(1024) char bsm[16384];
  __shared__ int stop;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = tid; i < 4096; i += blockDim.x) reinterpret_cast<uint32_t*>(bsm)[i] = 0x3c003c00u;
  if (tid == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (warp == 8) {  // concurrent tensor-core traffic: TS MMAs M=128 N=128 into columns 256-383
    if (mma && (tid & 31) == 0) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      uint64_t b = 0;
      const uint32_t sa = smem_u32(bsm);
      b |= (uint64_t)((sa >> 4) & 0x3FFF);
      b |= (uint64_t)1 << 16;
      b |= (uint64_t)64 << 32;
      b |= (uint64_t)1 << 46;
      b |= (uint64_t)2 << 61;
      const long long m0 = clock64();
      for (int n = 0; n < 8192; n += 64) {
        for (int i = 0; i < 64; ++i)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 256),
                       "r"(tmem + 384 + (i & 7) * 8), "l"(b), "r"(idesc), "r"(1));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)) : "memory");
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&mbar)) : "memory");
      out[148 + blockIdx.x] = clock64() - m0;
    }
    __syncwarp();
  }
  float acc = 0.f;
  long long t0 = clock64();
  if (warp < nwarps) {
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + 128 * (warp >> 2) + lane_off;
    float m = 0.f;
    for (int it = 0; it < iters; ++it) {
      float s[COLS];
#pragma unroll
      for (int c = 0; c < COLS; c += 32) {
        uint32_t r[32];
        ld32(tS + c, r);
#pragma unroll
        for (int k = 0; k < 32; ++k) s[c + k] = __uint_as_float(r[k]);
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (mode >= 1) {
        float mx = s[0];
#pragma unroll
        for (int k = 1; k < COLS; ++k) mx = fmaxf(mx, s[k]);
        if (mode >= 3) {  // v10-style row-max exchange between warps w and w+4 (same TMEM lanes)
          __shared__ float xm[2][2][128];
          const int row = (warp & 3) * 32 + (tid & 31), c = (warp >> 2) & 1;
          xm[it & 1][c][row] = mx;
          asm volatile("bar.sync %0, %1;" ::"r"(1 + (warp & 3)), "r"(64) : "memory");
          mx = fmaxf(xm[it & 1][0][row], xm[it & 1][1][row]);
        }
        m = fmaxf(m, mx);
      }
      if (mode >= 4) {  // v10 per-tile protocol: fences, syncwarp, mbarrier arrive + wait (a completed phase)
        if (mode != 5) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        __shared__ __align__(8) uint64_t pb[8];
        const uint32_t ba = smem_u32(&pb[warp]);
        if (it == 0 && (tid & 31) == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ba));
        __syncwarp();
        if (mode != 6 && (tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ba) : "memory");
        uint32_t ok = mode == 6;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                       : "=r"(ok) : "r"(ba), "r"((uint32_t)(it & 1)) : "memory");
      }
      if (mode >= 2) {
#pragma unroll
        for (int c = 0; c < COLS; c += 32) {
          uint32_t pk[16];
#pragma unroll
          for (int k = 0; k < 32; k += 2) {
            const float v0 = ex2(fmaf(s[c + k], 0.1f, -m)), v1 = ex2(fmaf(s[c + k + 1], 0.1f, -m));
            acc += v0 + v1;
            __half2 h = __floats2half2_rn(v0, v1);
            pk[k >> 1] = *reinterpret_cast<uint32_t*>(&h);
          }
          st16(tS + c / 2, pk);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        if (mode >= 4) {
          if (mode != 5) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
        }
      } else {
#pragma unroll
        for (int k = 0; k < COLS; ++k) acc += s[k];
      }
    }
  }
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  if (warp < nwarps) atomicAdd(&stop, 1);
  if (tid < 256) sink[blockIdx.x * 256 + tid] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}
int main() {
  long long* d;
  float* sink;
  cudaMalloc(&d, 2 * 148 * sizeof(long long));
  cudaMalloc(&sink, 148 * 256 * sizeof(float));
  const int iters = 2000;
  for (int mma = 1; mma < 2; ++mma)
  for (int cols : {64})
    for (int mode = 3; mode < 7; ++mode)
      for (int nw : {8}) {
        if (cols == 64) bench<64><<<148, 288>>>(iters, mode, nw, d, sink, mma);
        else bench<128><<<148, 288>>>(iters, mode, nw, d, sink, mma);
        cudaError_t err = cudaDeviceSynchronize();
        if (err != cudaSuccess) { printf("err %s\n", cudaGetErrorString(err)); return 1; }
        long long h[296];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double mc = 0;
        for (int i = 0; i < 148; ++i) mc += h[148 + i];
        printf("  MMA: %.1f clk per 128x128x16 TS MMA; ", mc / 148 / 8192);
        double cyc = 0;
        for (int i = 0; i < 148; ++i) cyc += h[i];
        cyc /= 148;
        const char* mn[7] = {"ld only", "ld+max", "ld+max+exp+st", "ld+max+xchg+exp+st", "+fences+mbarrier round trip", "+mbarrier only", "+fences only"};
        printf("%s cols %d, %d warps, %s: %.0f clk/iter (TMEM read %.1f B/clk/SM)\n", mma ? "with MMA" : "no MMA  ", cols, nw, mn[mode], cyc / iters,
               (double)nw * 32 * cols * 4 * iters / cyc);
      }
  return 0;
}

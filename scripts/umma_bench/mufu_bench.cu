// MUFU throughput on this GPU: ex2.approx.ftz.f32 vs ex2.approx.f16x2 (2 results per lane),
// 8 independent chains per thread, full occupancy; results per clock per SM.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__global__ void f32k(float* out, int iters) {
  float v[8];
  for (int k = 0; k < 8; ++k) v[k] = -0.001f * (threadIdx.x + k);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[k]));
  float s = 0;
  for (int k = 0; k < 8; ++k) s += v[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void f16k(float* out, int iters) {
  unsigned v[8];
  for (int k = 0; k < 8; ++k) {
    __half2 h = __floats2half2_rn(-0.001f * (threadIdx.x + k), -0.002f);
    v[k] = *reinterpret_cast<unsigned*>(&h);
  }
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[k]));
  float s = 0;
  for (int k = 0; k < 8; ++k) s += __half2float(reinterpret_cast<__half2*>(&v[k])->x);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* d;
  cudaMalloc(&d, 148 * 8 * 1024 * sizeof(float));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int iters = 20000;
  for (int which = 0; which < 2; ++which) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      if (which == 0) f32k<<<148 * 8, 1024>>>(d, iters);
      else f16k<<<148 * 8, 1024>>>(d, iters);
      cudaEventRecord(b);
      cudaDeviceSynchronize();
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double results = 148.0 * 8 * 1024 * iters * 8 * (which ? 2 : 1);
      printf("%s: %.3f ms, %.2f Tresults/s, %.1f results/clk/SM at %d MHz nominal\n", which ? "ex2.f16x2" : "ex2.f32",
             ms, results / (ms * 1e-3) / 1e12, results / (ms * 1e-3) / (clk_khz * 1e3) / 148, clk_khz / 1000);
    }
  }
  return 0;
}

// Prints the register <-> (TMEM lane, column) mapping of tcgen05.ld .16x256b and .16x128b
// (warp 0, lanes 0-15 and 16-31), by filling TMEM with value = lane*1000 + column through
// the 32x32b shape (thread i = lane i).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(int* out) {
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (tid < 32) {
    for (int c = 0; c < 16; ++c) {
      uint32_t v = tid * 1000 + c;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + c), "r"(v));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    uint32_t r[8];
    // 16x256b.x1 at lane base 0: 4 regs/thread ; .x2: 8 regs
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 8; ++i) out[tid * 8 + i] = r[i];
    uint32_t q[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7])
                 : "r"(tmem + (16u << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 8; ++i) out[256 + tid * 8 + i] = q[i];
    uint32_t w[4];
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x2.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 4; ++i) out[512 + tid * 4 + i] = w[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
  }
}
int main() {
  int* d;
  cudaMalloc(&d, 1024 * sizeof(int));
  k<<<1, 128>>>(d);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
  int h[1024];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("16x256b.x2 at lane base 0 (value = lane*1000 + col):\n");
  for (int t = 0; t < 32; ++t) {
    printf("t%2d:", t);
    for (int i = 0; i < 8; ++i) printf(" %5d", h[t * 8 + i]);
    printf("\n");
  }
  printf("16x256b.x2 at lane base 16:\n");
  for (int t = 0; t < 8; ++t) {
    printf("t%2d:", t);
    for (int i = 0; i < 8; ++i) printf(" %5d", h[256 + t * 8 + i]);
    printf("\n");
  }
  printf("16x128b.x2 at lane base 0:\n");
  for (int t = 0; t < 32; ++t) {
    printf("t%2d:", t);
    for (int i = 0; i < 4; ++i) printf(" %5d", h[512 + t * 4 + i]);
    printf("\n");
  }
  return 0;
}

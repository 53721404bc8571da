// skv_prefill.cu — causal chunked-prefill attention over the unified pool on the
// 5th-generation tensor cores (tcgen05.mma, accumulators in TMEM), sm_100a.
//
// Each request's last n_new tokens attend causally to every key at or before their own
// position; K/V are read through the request's block table (reference block layout,
// kv_cache.hpp:178-182; per-(layer, kv head) runs of 16 tokens).  GQA query
// rows are folded into M: row i of a 128-row query tile is (token t0 + i/G, q head
// kv_head*G + i%G), so one K/V tile feeds G query heads.
//
// Kernels (SEAKV_PREFILL_V selects; DESIGN.md §5 has the measurements):
//   v10 (default) prefill_kernel_v10: CTA pairs, one 256-row tcgen05.mma.cta_group::2 per
//       K=16 step (N = 128 keys / 128 dims), K/V halves per SM by TMA, S double-buffered
//       in TMEM, persistent with a dynamic work counter;
//   v9  prefill_kernel_v9: one CTA per SM, two 128-row tiles ping-ponging on 64-key tiles;
//   v2  prefill_kernel: one CTA per tile with cp.async staging -- the fallback when the pool
//       has no TMA descriptor.
//
// UMMA operand layouts (cute canonical SW128): a [R rows x 128 d] fp16 tile is two
// 64-element column halves of R x 128 B; row r of a half at (r/8)*1024 + (r%8)*128,
// 16-byte chunk c stored at chunk c ^ (r%8).  Q and K use K-major descriptors (SBO =
// 1024 B, advance 32 B per K=16 step); V uses an MN-major descriptor (SBO = 1024 B,
// advance 2 KiB per 16 keys).  One TMA box {64 elements, 16 rows} = one 2 KiB d-half of a
// native block's K or V run lands directly in this layout.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "skv_internal.h"

namespace skv {

namespace {

constexpr int kD = 128;
constexpr int kTpb = 16;
constexpr int kRows = 128;                  // M (query rows per CTA)
constexpr int kTileBytes = kRows * kD * 2;  // 32 KiB per operand tile
constexpr int kHalf = kRows * 128;          // bytes of one 64-element column half
constexpr int kThreads = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// byte offset of (row, 16B-chunk c in 0..15) in a swizzled [128 x 128] fp16 tile
__device__ __forceinline__ uint32_t sw_off(int row, int c) {
  const int half = c >> 3, cc = c & 7;
  return half * kHalf + (row >> 3) * 1024 + (row & 7) * 128 + ((cc ^ (row & 7)) << 4);
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;  // n = 0: zero-fill (src not read)
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// SW128 UMMA shared-memory descriptor (cute::UMMA::SmemDescriptor, version 1).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (Blackwell)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}


__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// A operand from TMEM (kind::f16, K-major): D[tmem_d] (+)= A[tmem_a] . B[desc_b]
__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Build with `make SKV_EXTRA=-DSKV_WATCHDOG` to turn a protocol hang into a trap that names
// the barrier and phase every stuck warp waits on.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok = 0;
#ifdef SKV_WATCHDOG
  long long spins = 0;
#endif
  while (!ok) {
#ifdef SKV_WATCHDOG
    ++spins;
    if (spins == (1ll << 22) && (threadIdx.x & 31) == 0)
      printf("SKV_WATCHDOG block (%d,%d,%d) warp %d bar_off %u parity %u\n", blockIdx.x, blockIdx.y, blockIdx.z,
             threadIdx.x >> 5, smem_u32(bar) & 0xffff, phase);
    if (spins == (1ll << 25)) __trap();
#endif
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(r[k]);
}

// two 32-column loads in flight, one wait (TMEM load latency is paid once per 64 columns)
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float (&v)[64]) {
  uint32_t r[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]),
        "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]),
        "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]),
        "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]),
        "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr + 32));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < 64; ++k) v[k] = __uint_as_float(r[k]);
}

template <typename T>
__device__ __forceinline__ uint32_t pack2(float a, float b);
template <>
__device__ __forceinline__ uint32_t pack2<__half>(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
template <>
__device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
      "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
      "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
      "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31]));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_st32u(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}


__device__ __forceinline__ float ex2(float x) {
#ifdef SKV_PF_NOMUFU  // diagnostic build only (wrong results): exponentials off the MUFU
  return fmaf(x, 0.0078125f, 0.5f);
#else
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#endif
}

// v2: 64-key tiles (112 KiB smem -> two CTAs per SM overlap each other's MMA and
// softmax phases), O accumulated across tiles by the tensor core in TMEM with a
// lazy (threshold 2^8) softmax-max correction, single-pass softmax, masking only on
// tiles that cross the causal diagonal or the chunk end.
constexpr int kKT = 64;                    // keys per tile
constexpr int kKVHalf = kKT * 128;         // 8 KiB: one 64-element d-half of a K/V tile
constexpr int kKVBytes = 2 * kKVHalf;      // 16 KiB per K or V tile
constexpr int kPBytes = kRows * 128;       // P tile: 128 rows x 64 keys fp16 (one half)
constexpr int kSmem2 = kTileBytes + 4 * kKVBytes + kPBytes + 64;
constexpr float kRescale = 8.0f;           // log2 threshold for the lazy correction

__device__ __forceinline__ uint32_t sw_kv(int row, int c) {  // [64 rows x 128 d] tile
  const int half = c >> 3, cc = c & 7;
  return half * kKVHalf + (row >> 3) * 1024 + (row & 7) * 128 + ((cc ^ (row & 7)) << 4);
}
__device__ __forceinline__ uint32_t sw_p(int row, int c) {  // [128 rows x 64 keys] tile, c in 0..7
  return (row >> 3) * 1024 + (row & 7) * 128 + ((c ^ (row & 7)) << 4);
}

__device__ __forceinline__ uint32_t make_idesc_n(int bf16, int b_mn_major, int n) {
  uint32_t d = 0;
  d |= 1u << 4;
  d |= (uint32_t)bf16 << 7;
  d |= (uint32_t)bf16 << 10;
  d |= (uint32_t)b_mn_major << 16;
  d |= (uint32_t)(n >> 3) << 17;
  d |= (uint32_t)(kRows >> 4) << 24;
  return d;
}

template <typename T>
__global__ void __launch_bounds__(kThreads, 2) prefill_kernel(const __grid_constant__ DataParams p) {
  extern __shared__ __align__(1024) char smem[];
  char* sQ = smem;
  char* sK[2] = {smem + kTileBytes, smem + kTileBytes + kKVBytes};
  char* sV[2] = {smem + kTileBytes + 2 * kKVBytes, smem + kTileBytes + 3 * kKVBytes};
  char* sP = smem + kTileBytes + 4 * kKVBytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + kPBytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sP + kPBytes + 16);

  if (smem_u32(smem) & 1023) __trap();  // SW128 operand tiles need 1 KiB alignment
  const int r = blockIdx.z, h = blockIdx.y, tile = blockIdx.x;
  const int grp = p.req_group[r];
  const DataGroup& g = p.g[grp];
  const int G = g.G;
  const int q_len = p.n_new;
  if (!g.active || h >= g.Hkv || tile * kRows >= q_len * G) return;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int handle = p.handles[r];
  const int ctx = p.req_tokens[handle];
  const int start = ctx - q_len;
  const int tpt = kRows / G;  // tokens per tile
  const int t0 = tile * tpt;
  const int n_keys = min(ctx, start + t0 + tpt);
  const int n_kt = (n_keys + kKT - 1) / kKT;
  const int2* row_tab = p.req_table + (size_t)handle * p.cap;
  const char* kv_base = p.pool + g.layer_off + (long long)h * g.head_stride;
  const int rl = r - g.req_begin;
  const bool tail_rows = t0 + tpt > q_len;  // some rows of this tile are past the chunk end

  if (warp == 0) {  // TMEM: S in columns [0,64), O in [64,192)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  const uint32_t tS = tmem + lane_off, tO = tmem + 64 + lane_off;

  {  // Q tile, coalesced: 8 rows x 256 B per instruction across the CTA
    const int c = tid & 15;
#pragma unroll 4
    for (int i = 0; i < 16; ++i) {
      const int row = (tid >> 4) + 8 * i;
      const int tok = t0 + row / G, gg = row % G;
      const bool ok = tok < q_len;
      const char* src = reinterpret_cast<const char*>(g.q) +
                        (((size_t)rl * q_len + (ok ? tok : 0)) * g.Hq + h * G + gg) * (kD * 2) + c * 16;
      cp_async16(smem_u32(sQ) + sw_off(row, c), src, ok);
    }
  }
  // a 64-key tile spans 4 native blocks; every thread needs the same 4 table entries,
  // fetched one tile ahead so the cp.async address math never waits on a global load
  const int n_blk = (n_keys + kTpb - 1) / kTpb;
  auto fetch_tab = [&](int j, int2 (&e)[4]) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int bi = j * 4 + b;
      e[b] = bi < n_blk ? row_tab[bi] : make_int2(0, 0);
    }
  };
  auto load_kv = [&](int j, int buf, const int2 (&e)[4]) {
    const int c = tid & 15;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int key = (tid >> 4) + 8 * i;
      const int a = j * kKT + key;
      const bool ok = a < n_keys;
      const int2 eb = e[i >> 1];
      const char* src = kv_base + (long long)eb.x * p.merged_stride + (long long)eb.y * g.native_stride +
                        (a % kTpb) * (kD * 2) + c * 16;
      cp_async16(smem_u32(sK[buf]) + sw_kv(key, c), src, ok);
      cp_async16(smem_u32(sV[buf]) + sw_kv(key, c), src + kTpb * kD * 2, ok);
    }
  };
  int2 tab_next[4];
  {
    int2 tab0[4];
    fetch_tab(0, tab0);
    load_kv(0, 0, tab0);
    cp_async_commit();
    fetch_tab(1, tab_next);
  }

  const uint32_t idesc_qk = make_idesc_n(p.dtype, 0, kKT);
  const uint32_t idesc_pv = make_idesc_n(p.dtype, 1, kD);
  const int row = tid;
  const int my_tok = t0 + row / G;
  const bool row_ok = my_tok < q_len;
  const int my_pos = start + my_tok;
  const float c2 = p.scale_log2;
  float m = -INFINITY, l = 0.f;
  uint32_t phase = 0;

  for (int j = 0; j < n_kt; ++j) {
    const int buf = j & 1;
    if (j + 1 < n_kt) {
      load_kv(j + 1, buf ^ 1, tab_next);
      cp_async_commit();
      fetch_tab(j + 2, tab_next);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int k = 0; k < kD / 16; ++k) {
        const uint32_t qoff = (k >> 2) * kHalf + (k & 3) * 32;
        const uint32_t koff = (k >> 2) * kKVHalf + (k & 3) * 32;
        mma_f16(tmem, make_desc(smem_u32(sQ) + qoff, 16, 1024), make_desc(smem_u32(sK[buf]) + koff, 16, 1024),
                idesc_qk, k > 0);
      }
      mma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();

    float s[64];
    {
      float a0[32], a1[32];
      tmem_ld32(tS, a0);
      tmem_ld32(tS + 32, a1);
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        s[k] = a0[k];
        s[32 + k] = a1[k];
      }
    }
    // tiles crossing the causal diagonal / chunk end need per-key masks (CTA-uniform test)
    const bool masked = (j * kKT + kKT - 1 > start + t0) || tail_rows;
    if (masked) {
#pragma unroll
      for (int k = 0; k < 64; ++k)
        if (!(row_ok && j * kKT + k <= my_pos)) s[k] = -INFINITY;
    }
    float mx4[4] = {s[0], s[1], s[2], s[3]};  // 4 independent chains
#pragma unroll
    for (int k = 4; k < 64; ++k) mx4[k & 3] = fmaxf(mx4[k & 3], s[k]);
    const float mt = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * c2;  // tile max, log2 domain
    const bool need = mt > m + kRescale;
    float alpha = 1.f;
    if (need) {
      alpha = ex2(m - mt);  // m = -inf -> 0
      l *= alpha;
      m = mt;
    }
    if (j > 0 && __any_sync(0xffffffffu, need)) {  // correct the TMEM accumulator rows that moved
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        float o[32];
        tmem_ld32(tO + cc * 32, o);
#pragma unroll
        for (int k = 0; k < 32; ++k) o[k] *= alpha;
        tmem_st32(tO + cc * 32, o);
      }
    }
    const float mu = (m == -INFINITY) ? 0.f : m;
    float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      uint32_t pk[4];
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        const float v0 = ex2(fmaf(s[cc * 8 + k], c2, -mu));
        const float v1 = ex2(fmaf(s[cc * 8 + k + 1], c2, -mu));
        ls[k >> 1] += v0 + v1;
        pk[k >> 1] = pack2<T>(v0, v1);
      }
      *reinterpret_cast<uint4*>(sP + sw_p(row, cc)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
    l += (ls[0] + ls[1]) + (ls[2] + ls[3]);
    tc_fence_before();
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
#pragma unroll
      for (int k = 0; k < kKT / 16; ++k)
        mma_f16(tmem + 64, make_desc(smem_u32(sP) + k * 32, 16, 1024),
                make_desc(smem_u32(sV[buf]) + k * 2048, kKVHalf, 1024), idesc_pv, (j > 0 || k > 0) ? 1u : 0u);
      mma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
  }

  {
    const float inv = l > 0.f ? 1.f / l : 0.f;
    char* dst = reinterpret_cast<char*>(g.out) +
                (((size_t)rl * q_len + (row_ok ? my_tok : 0)) * g.Hq + h * G + row % G) * (kD * 2);
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      float o[32];
      tmem_ld32(tO + cc * 32, o);  // warp-collective: every lane loads, valid rows store
      if (row_ok) {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          uint4 v;
          v.x = pack2<T>(o[8 * q4] * inv, o[8 * q4 + 1] * inv);
          v.y = pack2<T>(o[8 * q4 + 2] * inv, o[8 * q4 + 3] * inv);
          v.z = pack2<T>(o[8 * q4 + 4] * inv, o[8 * q4 + 5] * inv);
          v.w = pack2<T>(o[8 * q4 + 6] * inv, o[8 * q4 + 7] * inv);
          *reinterpret_cast<uint4*>(dst + cc * 64 + q4 * 16) = v;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------------------------------
// Warp-specialised kernels (v9, v10; earlier v3/v5/v7 steps are in git history and in
// DESIGN.md): warps 0-7 softmax (two warps per TMEM lane quarter), warp 8 issues every
// tcgen05.mma from one thread, warp 9 streams K/V with TMA, all handshakes on mbarriers.
constexpr int kSoftmaxWarps = 8;             // 4 per query tile, one thread per query row
constexpr int kMmaWarp = kSoftmaxWarps;      // warp 8
constexpr int kLoadWarp = kSoftmaxWarps + 1; // warp 9
constexpr int kThreadsV3 = (kSoftmaxWarps + 2) * 32;

__device__ __forceinline__ void mbar_init_n(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* tmap, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_v3(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

// Build with SKV_EXTRA=-DSKV_PF_TRACE to record, per CTA, clock64 cycles spent in each
// role's waits (16 u64 per CTA in p.trace; see scripts/prefill_trace.py).
#ifdef SKV_PF_TRACE
#define PF_T(slot, stmt)                      \
  do {                                        \
    const long long t0_ = clock64();          \
    stmt;                                     \
    pf_acc[slot] += clock64() - t0_;          \
  } while (0)
#else
#define PF_T(slot, stmt) stmt
#endif

// ---------------------------------------------------------------------------------------
// v9 layout (from v7): Q in TMEM.  With Q and K both read from shared memory, a 128x64x16
// QK^T MMA moves 6 KiB of operands per 32 tensor-core cycles, above the 128 B/clk
// shared-memory read rate, and issues at 48 clk instead of 32 (scripts/umma_bench).  The
// softmax warps write their Q rows into TMEM once per item (tcgen05.st) and QK^T is the TS
// form; the Q buffers' 64 KiB of smem become two more K/V stages (7).  TMEM: Q_A | Q_B (64
// cols each) | S_A | S_B (64) | O_A | O_B (128); S is single-buffered per tile (P written
// over it), so per tile the chain is softmax(j) -> P.V(j) -> QK(j+1) -> softmax(j+1), the
// other tile's softmax running meanwhile.
constexpr int kStagesV7 = 7;
constexpr int kSmemV7 = kStagesV7 * 2 * kKVBytes + 256;

// ---------------------------------------------------------------------------------------
// v9: persistent v7 with dynamic scheduling.  One CTA per SM; the TMA warp draws work
// items (request, kv head, query-tile pair), longest first, from a global counter and
// publishes them through an 8-slot ring in shared memory (item_full[slot] barriers), so
// every role walks the same sequence without per-CTA setup: TMEM, barriers and the CTA
// launch are paid once per SM, and the next item's K/V streams in (and its Q rows are
// written) while the current item drains.  All barrier phases run on CTA-global counters
// (jt: key tiles, it: items).
constexpr int kRing9 = 8;
constexpr int kSmemV9 = kSmemV7 + 128;  // + item ring and its barriers

// item order: (request, kv head) major, query-tile pair descending minor, so the pairs of
// one (request, head) -- which read the same K/V -- run at the same time on different SMs
// (L2 reuse) and each group starts with its longest pair
__device__ __forceinline__ bool prefill_item9(const DataParams& p, int i, int npairs, int hmax, int& r, int& h,
                                              int& pair) {
  pair = npairs - 1 - i % npairs;
  const int rem = i / npairs;
  h = rem % hmax;
  r = rem / hmax;
  const DataGroup& g = p.g[p.req_group[r]];
  return g.active && h < g.Hkv && 2 * pair * kRows < p.n_new * g.G;
}

template <typename T>
__global__ void __launch_bounds__(kThreadsV3, 1) prefill_kernel_v9(const __grid_constant__ DataParams p, int npairs,
                                                                    int hmax) {
  extern __shared__ __align__(1024) char smem[];
  if (smem_u32(smem) & 1023) __trap();
  char* kvbase = smem;
  uint64_t* bars = reinterpret_cast<uint64_t*>(kvbase + kStagesV7 * 2 * kKVBytes);
  uint64_t* kv_full = bars;                       // [stages]
  uint64_t* kv_empty = bars + kStagesV7;          // [stages]
  uint64_t* q_full = bars + 2 * kStagesV7;        // count 256 (per item)
  uint64_t* s_full = bars + 2 * kStagesV7 + 1;    // [tile]
  uint64_t* p_full = bars + 2 * kStagesV7 + 3;    // [tile] count 128
  uint64_t* pv_done = bars + 2 * kStagesV7 + 5;   // [tile]
  uint64_t* item_full = bars + 2 * kStagesV7 + 7; // [kRing9]
  int* ring = reinterpret_cast<int*>(bars + 2 * kStagesV7 + 7 + kRing9);  // [kRing9]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + kRing9);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_items = npairs * hmax * p.nreq;
  const int q_len = p.n_new;

  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < kStagesV7; ++i) {
      mbar_init_n(&kv_full[i], 1);
      mbar_init_n(&kv_empty[i], 1);
    }
    mbar_init_n(q_full, 2 * 128);
    for (int i = 0; i < 2; ++i) {
      mbar_init_n(&s_full[i], 1);
      mbar_init_n(&p_full[i], 128);
      mbar_init_n(&pv_done[i], 1);
    }
    for (int i = 0; i < kRing9; ++i) mbar_init_n(&item_full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  struct Geo {
    int r, h, pair, handle, ctx, start, tpt, t0A, n_keys, n_kt, rl, G;
    const DataGroup* g;
  };
  auto geo = [&](int idx) {
    Geo e;
    prefill_item9(p, idx, npairs, hmax, e.r, e.h, e.pair);
    e.g = &p.g[p.req_group[e.r]];
    e.G = e.g->G;
    e.handle = p.handles[e.r];
    e.ctx = p.req_tokens[e.handle];
    e.start = e.ctx - q_len;
    e.tpt = kRows / e.G;
    e.t0A = 2 * e.pair * e.tpt;
    e.n_keys = min(e.ctx, e.start + e.t0A + 2 * e.tpt);
    e.n_kt = (e.n_keys + kKT - 1) / kKT;
    e.rl = e.r - e.g->req_begin;
    return e;
  };
  // consumers: the k-th item of this CTA (-1 = no more work)
  auto next_item = [&](uint32_t k) {
    mbar_wait(&item_full[k % kRing9], (k / kRing9) & 1);
    return *reinterpret_cast<volatile int*>(&ring[k % kRing9]);
  };

  if (warp == kLoadWarp) {  // ----------------------------------------- scheduler + K/V streaming
    if (lane == 0) {
      uint32_t jt = 0;
      for (uint32_t k = 0;; ++k) {
        int idx = atomicAdd(p.counter, 1);
        while (idx < n_items) {  // skip holes of the (pair, head, request) grid
          int r_, h_, pr_;
          if (prefill_item9(p, idx, npairs, hmax, r_, h_, pr_)) break;
          idx = atomicAdd(p.counter, 1);
        }
        const int pub = idx < n_items ? idx : -1;
        ring[k % kRing9] = pub;
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&item_full[k % kRing9]))
                     : "memory");
        if (pub < 0) break;
        const Geo e = geo(pub);
        const int2* row_tab = p.req_table + (size_t)e.handle * p.cap;
        const long long base_off = e.g->layer_off + (long long)e.h * e.g->head_stride;
        const int n_blk = (e.n_keys + kTpb - 1) / kTpb;
        for (int j = 0; j < e.n_kt; ++j, ++jt) {
          const int st = jt % kStagesV7;
          if (jt >= (uint32_t)kStagesV7) mbar_wait(&kv_empty[st], ((jt / kStagesV7) - 1) & 1);
          int2 eb[4];
          int nb = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int bi = j * 4 + b;
            eb[b] = bi < n_blk ? row_tab[bi] : make_int2(-1, 0);
            nb += bi < n_blk;
          }
          mbar_expect_tx_v3(&kv_full[st], nb * 4 * 2048);
          const uint32_t sK = smem_u32(kvbase + st * 2 * kKVBytes), sV = sK + kKVBytes;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            if (eb[b].x < 0) continue;
            const int row0 = (int)(((long long)eb[b].x * p.merged_stride + (long long)eb[b].y * e.g->native_stride +
                                    base_off) >> 8);
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              tma_load_2d(sK + hh * kKVHalf + b * 2048, &p.kv_tmap, hh * 64, row0, &kv_full[st]);
              tma_load_2d(sV + hh * kKVHalf + b * 2048, &p.kv_tmap, hh * 64, row0 + kTpb, &kv_full[st]);
            }
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {  // -------------------------------------------- MMA issue
    if (lane == 0) {
      const uint32_t idesc_qk = make_idesc_n(p.dtype, 0, kKT);
      const uint32_t idesc_pv = make_idesc_n(p.dtype, 1, kD);
      uint32_t jt = 0;
      for (uint32_t k = 0;; ++k) {
        const int idx = next_item(k);
        if (idx < 0) break;
        const Geo e = geo(idx);
        const uint32_t j0 = jt;
        auto qk = [&](int x, int j) {
          const uint32_t sK = smem_u32(kvbase + ((j0 + j) % kStagesV7) * 2 * kKVBytes);
#pragma unroll
          for (int kk = 0; kk < kD / 16; ++kk) {
            const uint32_t koff = (kk >> 2) * kKVHalf + (kk & 3) * 32;
            mma_f16_ts(tmem + 128 + x * 64, tmem + x * 64 + kk * 8, make_desc(sK + koff, 16, 1024), idesc_qk, kk > 0);
          }
          mma_commit(&s_full[x]);
        };
        auto pv = [&](int x, int j) {
          const uint32_t sV = smem_u32(kvbase + ((j0 + j) % kStagesV7) * 2 * kKVBytes + kKVBytes);
#pragma unroll
          for (int kk = 0; kk < kKT / 16; ++kk)
            mma_f16_ts(tmem + 256 + x * 128, tmem + 128 + x * 64 + kk * 8, make_desc(sV + kk * 2048, kKVHalf, 1024),
                       idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&pv_done[x]);
        };
        auto wait_kv = [&](int j) {
          const uint32_t gj = j0 + j;
          mbar_wait(&kv_full[gj % kStagesV7], (gj / kStagesV7) & 1);
          tc_fence_after();
        };
        mbar_wait(q_full, k & 1);
        tc_fence_after();
        wait_kv(0);
        qk(0, 0);
        qk(1, 0);
        for (int j = 0; j < e.n_kt; ++j) {
          const uint32_t gj = j0 + j;
          mbar_wait(&p_full[0], gj & 1);
          tc_fence_after();
          pv(0, j);
          if (j + 1 < e.n_kt) {
            wait_kv(j + 1);
            qk(0, j + 1);
          }
          mbar_wait(&p_full[1], gj & 1);
          tc_fence_after();
          pv(1, j);
          mma_commit(&kv_empty[gj % kStagesV7]);
          if (j + 1 < e.n_kt) qk(1, j + 1);
        }
        jt += e.n_kt;
      }
    }
    __syncwarp();
  } else {  // ------------------------------------------------------------- softmax warps
    const int x = warp >> 2;
    const int row = tid & 127;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tQ = tmem + x * 64 + lane_off, tS = tmem + 128 + x * 64 + lane_off;
    const uint32_t tO = tmem + 256 + x * 128 + lane_off;
    const float c2 = p.scale_log2;
    uint32_t jt = 0;
    for (uint32_t k = 0;; ++k) {
      const int idx = next_item(k);
      if (idx < 0) break;
      const Geo e = geo(idx);
      const int t0 = e.t0A + x * e.tpt;
      const int my_tok = t0 + row / e.G;
      const bool row_ok = my_tok < q_len;
      const int my_pos = e.start + my_tok;
      const bool tail_rows = t0 + e.tpt > q_len;
      {  // Q rows of this item (the previous item's QK^T all retired: its S tiles were consumed)
        const uint4* src = reinterpret_cast<const uint4*>(
            reinterpret_cast<const char*>(e.g->q) +
            (((size_t)e.rl * q_len + (row_ok ? my_tok : 0)) * e.g->Hq + e.h * e.G + row % e.G) * (kD * 2));
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t qv[32];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const uint4 v = row_ok ? src[hh * 8 + i] : make_uint4(0u, 0u, 0u, 0u);
            qv[4 * i] = v.x;
            qv[4 * i + 1] = v.y;
            qv[4 * i + 2] = v.z;
            qv[4 * i + 3] = v.w;
          }
          tmem_st32u(tQ + hh * 32, qv);
        }
        tc_fence_before();
        mbar_arrive(q_full);
      }
      float m = -INFINITY, l = 0.f;
      const uint32_t j0 = jt;
      for (int j = 0; j < e.n_kt; ++j) {
        const uint32_t gj = j0 + j;
        mbar_wait(&s_full[x], gj & 1);
        tc_fence_after();
        if (x == 0 && j == e.n_kt - 1 && (j + 1) * kKT > e.n_keys) {
          char* sV = kvbase + (gj % kStagesV7) * 2 * kKVBytes + kKVBytes;
          const int c = row & 15;
          for (int key = row >> 4; key < kKT; key += 8)
            if (j * kKT + key >= e.n_keys) *reinterpret_cast<uint4*>(sV + sw_kv(key, c)) = make_uint4(0, 0, 0, 0);
        }
        float s[64];
        tmem_ld64(tS, s);
        const bool masked = (j * kKT + kKT - 1 > e.start + t0) || tail_rows;
        if (masked) {
#pragma unroll
          for (int kk = 0; kk < 64; ++kk)
            if (!(row_ok && j * kKT + kk <= my_pos)) s[kk] = -INFINITY;
        }
        float mx4[4] = {s[0], s[1], s[2], s[3]};
#pragma unroll
        for (int kk = 4; kk < 64; ++kk) mx4[kk & 3] = fmaxf(mx4[kk & 3], s[kk]);
        const float mt = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * c2;
        const bool need = mt > m + kRescale;
        float alpha = 1.f;
        if (need) {
          alpha = ex2(m - mt);
          l *= alpha;
          m = mt;
        }
        if (j > 0 && __any_sync(0xffffffffu, need)) {
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            float o[32];
            tmem_ld32(tO + cc * 32, o);
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) o[kk] *= alpha;
            tmem_st32(tO + cc * 32, o);
          }
        }
        const float mu = (m == -INFINITY) ? 0.f : m;
        float ls[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t pk[32];
#pragma unroll
        for (int kk = 0; kk < 64; kk += 2) {
          const float v0 = ex2(fmaf(s[kk], c2, -mu));
          const float v1 = ex2(fmaf(s[kk + 1], c2, -mu));
          ls[(kk >> 1) & 3] += v0 + v1;
          pk[kk >> 1] = pack2<T>(v0, v1);
        }
        tmem_st32u(tS, pk);
        l += (ls[0] + ls[1]) + (ls[2] + ls[3]);
        fence_async_smem();
        tc_fence_before();
        mbar_arrive(&p_full[x]);
      }
      const uint32_t gl = j0 + e.n_kt - 1;
      mbar_wait(&pv_done[x], gl & 1);
      tc_fence_after();
      jt += e.n_kt;
      const float inv = l > 0.f ? 1.f / l : 0.f;
      char* dst = reinterpret_cast<char*>(e.g->out) +
                  (((size_t)e.rl * q_len + (row_ok ? my_tok : 0)) * e.g->Hq + e.h * e.G + row % e.G) * (kD * 2);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        float o[32];
        tmem_ld32(tO + cc * 32, o);
        if (row_ok) {
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint4 v;
            v.x = pack2<T>(o[8 * q4] * inv, o[8 * q4 + 1] * inv);
            v.y = pack2<T>(o[8 * q4 + 2] * inv, o[8 * q4 + 3] * inv);
            v.z = pack2<T>(o[8 * q4 + 4] * inv, o[8 * q4 + 5] * inv);
            v.w = pack2<T>(o[8 * q4 + 6] * inv, o[8 * q4 + 7] * inv);
            *reinterpret_cast<uint4*>(dst + cc * 64 + q4 * 16) = v;
          }
        }
      }
      tc_fence_before();  // the next item's first P.V (after our p_full arrive) overwrites O
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------------------------------
// v10: CTA pairs (cta_group::2).  A 128x64x16 UMMA issues at 55 clk instead of 32
// (profiles/r01_umma_bench.txt), so v9's 64-key QK^T runs the tensor core at ~58 %, and a
// 128-key QK^T with two query tiles per SM does not fit TMEM (Q 2x64 + S 2x128 + O 2x128
// columns).  Here the two query tiles of a work item sit on the two SMs of a cluster and
// every MMA is one 256-row tcgen05.mma.cta_group::2 issued by the leader CTA: M = 256
// (128 query rows per SM, each SM's TMEM holds its rows), N = 128 keys for S = Q.K^T and
// N = 128 dims for O += P.V, both at the full 64 clk per K=16 step.  The B operands are
// split across the pair: CTA c holds keys [64c, 64c+64) of the K tile (all 128 dims) and
// dims [64c, 64c+64) of the V tile (all 128 keys), each loaded by its own TMA warp and
// signalling the leader's kv_full barrier, so K/V shared-memory traffic per SM halves.
// TMEM per SM: O [0,128) | S0 [128,256) | S1 [256,384) | Q [384,448): S is double
// buffered, so QK^T(j+1) runs while the softmax works on S(j) (P(j) is written over the
// first 64 columns of S(j) and read by the TS-form P.V).  Softmax: 8 warps per SM, warps
// w and w+4 share the TMEM lanes of rows 32(w%4).. and take key columns [0,64) and
// [64,128) resp.; the row max is exchanged through shared memory each tile.
// asynchronous TMEM load: the registers are valid only after tmem_ld32_wait on the same array
// (which takes them as in/out operands so no use can be scheduled above the wait)
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld32_wait(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}


constexpr int kStagesV10 = 6;
constexpr int kKV10 = 2 * kKVHalf * 2;  // per CTA per stage: K half-tile 16 KiB + V half-tile 16 KiB
constexpr int kSmemV10 = kStagesV10 * kKV10 + 4096 + 512;
constexpr int kKT10 = 128;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
  uint32_t d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(saddr), "r"(rank));
  return d;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// default (.release.cta) semantics: the data behind these arrivals is TMEM, ordered by
// tcgen05.fence::before_thread_sync; .release.cluster compiles to MEMBAR.ALL.GPU + ERRBAR
// (27 % of the warp-stall samples of the first v10 build)
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMEM-only handoffs (tcgen05.st -> fence::before_thread_sync -> arrive; the waiter issues
// fence::after_thread_sync before its MMAs): no generic-memory ordering needed, so no MEMBAR
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster_rel(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, uint32_t phase) {
  uint32_t ok = 0;
#ifdef SKV_WATCHDOG
  long long spins = 0;
#endif
  while (!ok) {
#ifdef SKV_WATCHDOG
    ++spins;
    if (spins == (1ll << 22) && (threadIdx.x & 31) == 0)
      printf("SKV_WATCHDOG v10 block %d warp %d bar_off %u parity %u\n", blockIdx.x, threadIdx.x >> 5,
             smem_u32(bar) & 0xffff, phase);
    if (spins == (1ll << 25)) __trap();
#endif
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}
// TMA box into this CTA's shared memory, completion counted on the leader CTA's barrier
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const void* tmap, int x, int y, uint32_t bar_cl) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(bar_cl)
      : "memory");
}
__device__ __forceinline__ void mma_f16_ts_pair(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// arrive on the barrier at this offset in both CTAs of the pair once the issued MMAs retire
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((unsigned short)3)
      : "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ uint32_t make_idesc_pair(int bf16, int b_mn_major) {
  uint32_t d = 0;
  d |= 1u << 4;
  d |= (uint32_t)bf16 << 7;
  d |= (uint32_t)bf16 << 10;
  d |= (uint32_t)b_mn_major << 16;
  d |= (uint32_t)(128 >> 3) << 17;  // N = 128
  d |= (uint32_t)(256 >> 4) << 24;  // M = 256 (128 rows per CTA)
  return d;
}

template <typename T>
__global__ void __launch_bounds__(kThreadsV3, 1) prefill_kernel_v10(const __grid_constant__ DataParams p, int npairs,
                                                                     int hmax) {
  extern __shared__ __align__(1024) char smem[];
  if (smem_u32(smem) & 1023) __trap();
#ifdef SKV_PF_TRACE
  long long pf_acc[5] = {0, 0, 0, 0, 0};
  const long long pf_start = clock64();
  long long pf_tiles = 0;
#endif
  char* kvbase = smem;
  float* xm = reinterpret_cast<float*>(smem + kStagesV10 * kKV10);  // [2 parity][2 half][128 rows]
  float* xl = xm + 512;                                              // [2 half][128 rows]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStagesV10 * kKV10 + 4096);
  uint64_t* kv_full = bars;                         // [stages] leader: both CTAs' bytes
  uint64_t* kv_empty = bars + kStagesV10;           // [stages] both CTAs (multicast commit)
  // Barriers indexed by [tile parity]: a softmax warp can finish S(j+1) before the MMA warp
  // has consumed P(j), and parity waits cannot tell phases two apart.
  uint64_t* q_full = bars + 2 * kStagesV10;         // leader: 16 warp arrivals per item
  uint64_t* p_full = bars + 2 * kStagesV10 + 1;     // [2] leader: 16 warp arrivals
  uint64_t* s_full = bars + 2 * kStagesV10 + 3;     // [2] both CTAs (multicast commit)
  uint64_t* pv_done = bars + 2 * kStagesV10 + 5;    // [2] both CTAs (multicast commit)
  uint64_t* item_full = bars + 2 * kStagesV10 + 7;  // [kRing9] both CTAs
  int* ring = reinterpret_cast<int*>(bars + 2 * kStagesV10 + 7 + kRing9);  // [kRing9]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + kRing9);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
  const int n_items = npairs * hmax * p.nreq;
  const int q_len = p.n_new;

  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < kStagesV10; ++i) {
      mbar_init_n(&kv_full[i], 1);
      mbar_init_n(&kv_empty[i], 1);
    }
    mbar_init_n(q_full, 16);
    for (int i = 0; i < 2; ++i) {
      mbar_init_n(&p_full[i], 16);
      mbar_init_n(&s_full[i], 1);
      mbar_init_n(&pv_done[i], 1);
    }
    for (int i = 0; i < kRing9; ++i) mbar_init_n(&item_full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t q_full_l = mapa_u32(smem_u32(q_full), 0), p_full_l = mapa_u32(smem_u32(p_full), 0);

  struct Geo {
    int r, h, pair, handle, ctx, start, tpt, t0A, n_keys, n_kt, rl, G;
    const DataGroup* g;
  };
  auto geo = [&](int idx) {
    Geo e;
    prefill_item9(p, idx, npairs, hmax, e.r, e.h, e.pair);
    e.g = &p.g[p.req_group[e.r]];
    e.G = e.g->G;
    e.handle = p.handles[e.r];
    e.ctx = p.req_tokens[e.handle];
    e.start = e.ctx - q_len;
    e.tpt = kRows / e.G;
    e.t0A = 2 * e.pair * e.tpt;
    e.n_keys = min(e.ctx, e.start + e.t0A + 2 * e.tpt);
    e.n_kt = (e.n_keys + kKT10 - 1) / kKT10;
    e.rl = e.r - e.g->req_begin;
    return e;
  };
  auto next_item = [&](uint32_t k) {
    mbar_wait_cl(&item_full[k % kRing9], (k / kRing9) & 1);
    return *reinterpret_cast<volatile int*>(&ring[k % kRing9]);
  };

  if (warp == kLoadWarp) {  // --------------------------------- scheduler (leader) + K/V streaming (both)
    // Whole warp: lane i holds block-table entry i of the current 32-entry chunk (4 key tiles)
    // and the next chunk is already in flight, so the table's load latency is off the TMA
    // issue path; the 8 lanes of a tile issue its boxes in parallel.
    uint32_t jt = 0;
    const uint32_t ring_peer = mapa_u32(smem_u32(ring), 1), item_peer = mapa_u32(smem_u32(item_full), 1);
    const uint32_t kv_full_l = mapa_u32(smem_u32(kv_full), 0);
    for (uint32_t k = 0;; ++k) {
      int pub;
      if (rank == 0) {
        if (lane == 0) {
          int idx = atomicAdd(p.counter, 1);
          while (idx < n_items) {
            int r_, h_, pr_;
            if (prefill_item9(p, idx, npairs, hmax, r_, h_, pr_)) break;
            idx = atomicAdd(p.counter, 1);
          }
          pub = idx < n_items ? idx : -1;
          const uint32_t slot = k % kRing9;
          ring[slot] = pub;
          asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(ring_peer + 4 * slot), "r"(pub) : "memory");
          asm volatile("mbarrier.arrive.release.cluster.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&item_full[slot]))
                       : "memory");
          mbar_arrive_cluster_rel(item_peer + 8 * slot);
        }
        pub = __shfl_sync(0xffffffffu, pub, 0);
      } else {
        pub = next_item(k);
      }
      if (pub < 0) break;
      const Geo e = geo(pub);
      const int2* row_tab = p.req_table + (size_t)e.handle * p.cap;
      const long long base_off = e.g->layer_off + (long long)e.h * e.g->head_stride;
      const int n_blk = (e.n_keys + kTpb - 1) / kTpb;
      int2 ent_next = lane < n_blk ? row_tab[lane] : make_int2(-1, 0);
      int row0 = 0;
      bool valid = false;
      for (int j = 0; j < e.n_kt; ++j, ++jt) {
        if ((j & 3) == 0) {
          valid = ent_next.x >= 0;
          row0 = valid ? (int)(((long long)ent_next.x * p.merged_stride + (long long)ent_next.y * e.g->native_stride +
                                base_off) >> 8)
                       : 0;
          const int nx = (j + 4) * 8 + lane;
          ent_next = nx < n_blk ? row_tab[nx] : make_int2(-1, 0);
        }
        const int st = jt % kStagesV10;
        if (jt >= (uint32_t)kStagesV10) {
          if (lane == 0) PF_T(0, mbar_wait(&kv_empty[st], ((jt / kStagesV10) - 1) & 1));
          __syncwarp();
        }
        const int grp = (j & 3) * 8;
        const bool mine = lane >= grp && lane < grp + 8 && valid;
        const int nb = __popc(__ballot_sync(0xffffffffu, mine));
        // leader expects both CTAs' bytes: K 2 halves x 2 KiB and V 2 x 2 KiB per valid block
        if (rank == 0 && lane == 0) mbar_expect_tx_v3(&kv_full[st], nb * 8192);
        __syncwarp();
        if (mine) {
          const int b = lane - grp;
          const uint32_t sK = smem_u32(kvbase + st * kKV10), sV = sK + 2 * kKVHalf;
          const uint32_t bar = kv_full_l + 8 * st;
          if ((b >> 2) == (int)rank) {  // this CTA's 64 keys of K, both d-halves
            tma_load_2d_pair(sK + (b & 3) * 2048, &p.kv_tmap, 0, row0, bar);
            tma_load_2d_pair(sK + kKVHalf + (b & 3) * 2048, &p.kv_tmap, 64, row0, bar);
          }
          tma_load_2d_pair(sV + b * 2048, &p.kv_tmap, (int)rank * 64, row0 + kTpb, bar);  // this CTA's d-half of V
        }
      }
    }
  } else if (warp == kMmaWarp) {  // ------------------------------------- MMA issue (leader only)
    if (lane == 0 && rank == 0) {
      const uint32_t idesc_qk = make_idesc_pair(p.dtype, 0);
      const uint32_t idesc_pv = make_idesc_pair(p.dtype, 1);
      const uint64_t k_desc0 = make_desc(smem_u32(kvbase), 16, 1024);
      const uint64_t v_desc0 = make_desc(smem_u32(kvbase) + 2 * kKVHalf, 2 * kKVHalf, 1024);
      uint32_t jt = 0;
      for (uint32_t k = 0;; ++k) {
        const int idx = next_item(k);
        if (idx < 0) break;
        const Geo e = geo(idx);
        const uint32_t j0 = jt;
        const int J = e.n_kt;
        auto wait_kv = [&](int j) {
          const uint32_t gj = j0 + j;
          PF_T(1, mbar_wait(&kv_full[gj % kStagesV10], (gj / kStagesV10) & 1));
          tc_fence_after();
        };
        // descriptors of a tile's 8 MMAs are materialised before the barrier wait that gates
        // them, so the issue burst after the wait is MMAs only (per-MMA descriptor arithmetic
        // on the issuing thread left the 64-clk MMAs issue-bound, profiles/r01_prefill_v10_diagnostics.txt)
        // descriptor = base descriptor of stage 0 + (byte offset >> 4) in the address field
        // (shared-memory addresses < 256 KiB: the 14-bit field never carries)
        auto k_descs = [&](int j, uint64_t (&d)[8]) {
          const uint64_t b = k_desc0 + (uint64_t)(((j0 + j) % kStagesV10) * (kKV10 >> 4));
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) d[kk] = b + (uint64_t)(((kk >> 2) * kKVHalf + (kk & 3) * 32) >> 4);
        };
        auto v_descs = [&](int j, uint64_t (&d)[8]) {
          const uint64_t b = v_desc0 + (uint64_t)(((j0 + j) % kStagesV10) * (kKV10 >> 4));
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) d[kk] = b + (uint64_t)((kk * 2048) >> 4);
        };
        auto pin = [](const uint64_t (&d)[8]) {  // force the values into registers here
          asm volatile("" ::"l"(d[0]), "l"(d[1]), "l"(d[2]), "l"(d[3]), "l"(d[4]), "l"(d[5]), "l"(d[6]), "l"(d[7]));
        };
        auto qk = [&](int j, const uint64_t (&d)[8]) {
          const uint32_t gj = j0 + j;
          const uint32_t tS = tmem + 128 + (gj & 1) * 128;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) mma_f16_ts_pair(tS, tmem + 384 + kk * 8, d[kk], idesc_qk, kk > 0);
          mma_commit_pair(&s_full[gj & 1]);
        };
        auto pv = [&](int j, const uint64_t (&d)[8]) {
          const uint32_t gj = j0 + j;
          const uint32_t tP = tmem + 128 + (gj & 1) * 128;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) mma_f16_ts_pair(tmem, tP + kk * 8, d[kk], idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
          mma_commit_pair(&pv_done[gj & 1]);
          mma_commit_pair(&kv_empty[gj % kStagesV10]);
        };
        {
          uint64_t d0[8], d1[8];
          k_descs(0, d0);
          if (J > 1) k_descs(1, d1);
          pin(d0);
          pin(d1);
          PF_T(0, mbar_wait(q_full, k & 1));
          tc_fence_after();
          wait_kv(0);
          qk(0, d0);
          if (J > 1) {
            wait_kv(1);
            qk(1, d1);
          }
        }
        for (int j = 0; j < J; ++j) {
          uint64_t vd[8], kd[8];
          PF_T(4, {
            v_descs(j, vd);
            k_descs(j + 2, kd);
            pin(vd);
            pin(kd);
          });
          PF_T(2, mbar_wait(&p_full[(j0 + j) & 1], ((j0 + j) >> 1) & 1));
          tc_fence_after();
          PF_T(3, pv(j, vd));
          if (j + 2 < J) {
            wait_kv(j + 2);
            PF_T(3, qk(j + 2, kd));
          }
        }
        jt += J;
      }
    }
    __syncwarp();
  } else {  // ------------------------------------------------------------- softmax warps
    const int c = warp >> 2;  // key-column half of S / dim half of Q and O
    const int row = (warp & 3) * 32 + lane;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tQ = tmem + 384 + 32 * c + lane_off;
    const uint32_t tO = tmem + 64 * c + lane_off;
    const float c2 = p.scale_log2;
    const int nbar = 1 + (warp & 3);  // named barrier of the two warps sharing these rows
    uint32_t jt = 0;
    for (uint32_t k = 0;; ++k) {
      const int idx = next_item(k);
      if (idx < 0) break;
      const Geo e = geo(idx);
      const int t0 = e.t0A + (int)rank * e.tpt;
      const int my_tok = t0 + row / e.G;
      const bool row_ok = my_tok < q_len;
      const int my_pos = e.start + my_tok;
      const bool tail_rows = t0 + e.tpt > q_len;
      {  // this thread's half of its Q row (all QK^T of the previous item retired)
        const uint4* src = reinterpret_cast<const uint4*>(
            reinterpret_cast<const char*>(e.g->q) +
            (((size_t)e.rl * q_len + (row_ok ? my_tok : 0)) * e.g->Hq + e.h * e.G + row % e.G) * (kD * 2) + c * 128);
        uint32_t qv[32];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint4 v = row_ok ? src[i] : make_uint4(0u, 0u, 0u, 0u);
          qv[4 * i] = v.x;
          qv[4 * i + 1] = v.y;
          qv[4 * i + 2] = v.z;
          qv[4 * i + 3] = v.w;
        }
        tmem_st32u(tQ, qv);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster_relaxed(q_full_l);
      }
      float m = -INFINITY, l = 0.f;
      const uint32_t j0 = jt;
      for (int j = 0; j < e.n_kt; ++j) {
        const uint32_t gj = j0 + j;
        const uint32_t tS = tmem + 128 + (gj & 1) * 128 + lane_off;
        PF_T(0, mbar_wait(&s_full[gj & 1], (gj >> 1) & 1));
        tc_fence_after();
        const bool last_partial = j == e.n_kt - 1 && (j + 1) * kKT10 > e.n_keys;
        if (last_partial) {  // V rows past the keys (stale or another owner's bytes) -> 0
          char* sV = kvbase + (gj % kStagesV10) * kKV10 + 2 * kKVHalf;
          const int first = e.n_keys - j * kKT10;
          for (int i = tid; i < kKT10 * 8; i += 256) {
            const int key = i >> 3, ch = i & 7;
            if (key >= first)
              *reinterpret_cast<uint4*>(sV + (key >> 3) * 1024 + (key & 7) * 128 + ((ch ^ (key & 7)) << 4)) =
                  make_uint4(0, 0, 0, 0);
          }
        }
        const int kbase = j * kKT10 + 64 * c;
        const bool masked = (kbase + 63 > e.start + t0) || tail_rows;
        // path decision shared by the two warps of a row pair (same rows, same tile)
        const bool tile_masked = (j * kKT10 + kKT10 - 1 > e.start + t0) || tail_rows;
        float* xmb = xm + (gj & 1) * 256;
        float ls[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t pk[32];
#ifdef SKV_PF_NOSOFTMAX  // diagnostic build only (wrong results): protocol without the tile math
        if (true) {
#pragma unroll
          for (int kk = 0; kk < 32; ++kk) pk[kk] = 0x3c003c00u;
          PF_T(3, named_bar(nbar, 64));
        } else
#endif
        if (j > 0 && !tile_masked && !(p.dbg & 4) && __all_sync(0xffffffffu, m != -INFINITY)) {
          // Speculative path: exponentials against the running max m while the second 32-column
          // TMEM load is in flight, the row max exchanged only after them; valid unless the tile
          // raises a row max by more than 2^kRescale (rare: then the tile is recomputed from the
          // S values still in registers).  Keeps the TMEM-load latency and the max reduction off
          // the path between the tile barrier and the MUFU work.
          uint32_t ra[32], rb[32];
          float mxa = -INFINITY, mxb = -INFINITY;
          const float2 c2v = make_float2(c2, c2), nmv = make_float2(-m, -m);  // packed (FFMA2 / FADD2)
          float2 ls2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
          tmem_ld32_issue(tS + 64 * c, ra);
          tmem_ld32_wait(ra);
          tmem_ld32_issue(tS + 64 * c + 32, rb);
#pragma unroll
          for (int kk = 0; kk < 32; kk += 2) {
            const float x0 = __uint_as_float(ra[kk]), x1 = __uint_as_float(ra[kk + 1]);
            mxa = fmaxf(mxa, x0);
            mxb = fmaxf(mxb, x1);
            const float2 a = __ffma2_rn(make_float2(x0, x1), c2v, nmv);
            const float v0 = ex2(a.x), v1 = ex2(a.y);
            ls2[(kk >> 1) & 1] = __fadd2_rn(ls2[(kk >> 1) & 1], make_float2(v0, v1));
            pk[kk >> 1] = pack2<T>(v0, v1);
          }
          tmem_ld32_wait(rb);
#pragma unroll
          for (int kk = 0; kk < 32; kk += 2) {
            const float x0 = __uint_as_float(rb[kk]), x1 = __uint_as_float(rb[kk + 1]);
            mxa = fmaxf(mxa, x0);
            mxb = fmaxf(mxb, x1);
            const float2 a = __ffma2_rn(make_float2(x0, x1), c2v, nmv);
            const float v0 = ex2(a.x), v1 = ex2(a.y);
            ls2[(kk >> 1) & 1] = __fadd2_rn(ls2[(kk >> 1) & 1], make_float2(v0, v1));
            pk[16 + (kk >> 1)] = pack2<T>(v0, v1);
          }
          ls[0] = ls2[0].x;
          ls[1] = ls2[0].y;
          ls[2] = ls2[1].x;
          ls[3] = ls2[1].y;
          xmb[c * 128 + row] = fmaxf(mxa, mxb);
          PF_T(3, named_bar(nbar, 64));
          const float mt = fmaxf(xmb[row], xmb[128 + row]) * c2;
          const bool need = mt > m + kRescale;
          if (__any_sync(0xffffffffu, need)) {  // redo the tile with the new max
            float alpha = 1.f;
            if (need) {
              alpha = ex2(m - mt);
              l *= alpha;
              m = mt;
            }
            PF_T(1, mbar_wait(&pv_done[(gj - 1) & 1], ((gj - 1) >> 1) & 1));  // O holds P.V through tile j-1
            tc_fence_after();
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
              float o[32];
              tmem_ld32(tO + cc * 32, o);
#pragma unroll
              for (int kk = 0; kk < 32; ++kk) o[kk] *= alpha;
              tmem_st32(tO + cc * 32, o);
            }
            ls[0] = ls[1] = ls[2] = ls[3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < 64; kk += 2) {
              const uint32_t* src = kk < 32 ? ra : rb;
              const float v0 = ex2(fmaf(__uint_as_float(src[kk & 31]), c2, -m));
              const float v1 = ex2(fmaf(__uint_as_float(src[(kk & 31) + 1]), c2, -m));
              ls[(kk >> 1) & 3] += v0 + v1;
              pk[kk >> 1] = pack2<T>(v0, v1);
            }
          }
        } else {
          float s[64];
          tmem_ld64(tS + 64 * c, s);
          if (masked) {
#pragma unroll
            for (int kk = 0; kk < 64; ++kk)
              if (!(row_ok && kbase + kk <= my_pos)) s[kk] = -INFINITY;
          }
          float mx4[4] = {s[0], s[1], s[2], s[3]};
#pragma unroll
          for (int kk = 4; kk < 64; kk += 4) {
            mx4[0] = fmaxf(mx4[0], s[kk]);
            mx4[1] = fmaxf(mx4[1], s[kk + 1]);
            mx4[2] = fmaxf(mx4[2], s[kk + 2]);
            mx4[3] = fmaxf(mx4[3], s[kk + 3]);
          }
          xmb[c * 128 + row] = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
          PF_T(3, named_bar(nbar, 64));
          const float mt = fmaxf(xmb[row], xmb[128 + row]) * c2;
          const bool need = mt > m + kRescale;
          float alpha = 1.f;
          if (need) {
            alpha = ex2(m - mt);
            l *= alpha;
            m = mt;
          }
          if (j > 0 && __any_sync(0xffffffffu, need)) {
            PF_T(1, mbar_wait(&pv_done[(gj - 1) & 1], ((gj - 1) >> 1) & 1));  // O holds P.V through tile j-1
            tc_fence_after();
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
              float o[32];
              tmem_ld32(tO + cc * 32, o);
#pragma unroll
              for (int kk = 0; kk < 32; ++kk) o[kk] *= alpha;
              tmem_st32(tO + cc * 32, o);
            }
          }
          const float mu = (m == -INFINITY) ? 0.f : m;
#pragma unroll
          for (int kk = 0; kk < 64; kk += 2) {
            const float v0 = ex2(fmaf(s[kk], c2, -mu));
            const float v1 = ex2(fmaf(s[kk + 1], c2, -mu));
            ls[(kk >> 1) & 3] += v0 + v1;
            pk[kk >> 1] = pack2<T>(v0, v1);
          }
        }
        tmem_st32u(tS + 32 * c, pk);
        l += (ls[0] + ls[1]) + (ls[2] + ls[3]);
        if (last_partial) fence_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (last_partial) mbar_arrive_cluster(p_full_l + 8 * (gj & 1));  // orders the V-row zeroing
          else mbar_arrive_cluster_relaxed(p_full_l + 8 * (gj & 1));
        }
      }
      const uint32_t gl = j0 + e.n_kt - 1;
      xl[c * 128 + row] = l;
      PF_T(2, mbar_wait(&pv_done[gl & 1], (gl >> 1) & 1));
      tc_fence_after();
      named_bar(nbar, 64);
      const float lt = xl[row] + xl[128 + row];
      jt += e.n_kt;
#ifdef SKV_PF_TRACE
      pf_tiles += e.n_kt;
#endif
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      char* dst = reinterpret_cast<char*>(e.g->out) +
                  (((size_t)e.rl * q_len + (row_ok ? my_tok : 0)) * e.g->Hq + e.h * e.G + row % e.G) * (kD * 2) +
                  c * 128;
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        float o[32];
        tmem_ld32(tO + cc * 32, o);
        if (row_ok) {
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint4 v;
            v.x = pack2<T>(o[8 * q4] * inv, o[8 * q4 + 1] * inv);
            v.y = pack2<T>(o[8 * q4 + 2] * inv, o[8 * q4 + 3] * inv);
            v.z = pack2<T>(o[8 * q4 + 4] * inv, o[8 * q4 + 5] * inv);
            v.w = pack2<T>(o[8 * q4 + 6] * inv, o[8 * q4 + 7] * inv);
            *reinterpret_cast<uint4*>(dst + cc * 64 + q4 * 16) = v;
          }
        }
      }
      named_bar(nbar, 64);  // xl reused by the next item
      tc_fence_before();    // the next item's first P.V (after our p_full arrive) overwrites O
    }
  }
#ifdef SKV_PF_TRACE
  if (p.trace) {  // [cta][16]: loader 0, mma 1-3, softmax c=0 5-8, c=1 9-12, cta cycles 13, tiles 14
    unsigned long long* t = p.trace + (size_t)blockIdx.x * 16;
    if (warp == kLoadWarp && lane == 0) t[0] = pf_acc[0];
    if (warp == kMmaWarp && lane == 0)
      for (int i = 0; i < 4; ++i) t[1 + i] = pf_acc[i];
    if (warp < kSoftmaxWarps && (tid & 127) == 0)
      for (int i = 0; i < 4; ++i) t[5 + 4 * (warp >> 2) + i] = pf_acc[i];
    if (warp == kMmaWarp && lane == 0) t[15] = pf_acc[4];
    if (tid == 0) {
      t[13] = clock64() - pf_start;
      t[14] = pf_tiles;
    }
  }
#endif
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <typename T>
void launch_prefill_t(const DataParams& p, cudaStream_t s) {
  static std::atomic<uint64_t> attr2{0}, attr9{0}, attr10{0};
  ensure_smem_attr(prefill_kernel<T>, kSmem2, attr2);
  ensure_smem_attr(prefill_kernel_v9<T>, kSmemV9, attr9);
  ensure_smem_attr(prefill_kernel_v10<T>, kSmemV10, attr10);
  int tiles = 1, heads = 1;
  for (int i = 0; i < p.ngroups; ++i) {
    tiles = max(tiles, (p.n_new * p.g[i].G + kRows - 1) / kRows);
    heads = max(heads, p.g[i].Hkv);
  }
  static const int version = [] {
    const char* e = getenv("SEAKV_PREFILL_V");
    return e ? atoi(e) : 10;  // v10 measured fastest (profiles/r01_prefill_probe_v10_final.txt); 2, 9 selectable
  }();
  if (version == 2 || !p.has_tmap) {
    dim3 grid(tiles, heads, p.nreq);
    prefill_kernel<T><<<grid, kThreads, kSmem2, s>>>(p);
  } else if (version == 9) {
    const int npairs = (tiles + 1) / 2;
    const int nsm = num_sms();
    const long long items = (long long)npairs * heads * p.nreq;
    const int grid = (int)std::min<long long>(items, nsm);
    cudaMemsetAsync(p.counter, 0, sizeof(int), s);
    prefill_kernel_v9<T><<<grid, kThreadsV3, kSmemV9, s>>>(p, npairs, heads);
  } else if (version == 10) {
    const int npairs = (tiles + 1) / 2;
    const int nsm = num_sms();
    const long long items = (long long)npairs * heads * p.nreq;
    const int clusters = (int)std::min<long long>(items, nsm / 2);
    cudaMemsetAsync(p.counter, 0, sizeof(int), s);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * clusters, 1, 1);
    cfg.blockDim = dim3(kThreadsV3, 1, 1);
    cfg.dynamicSmemBytes = kSmemV10;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, prefill_kernel_v10<T>, p, npairs, heads);
  } else {
    std::fprintf(stderr, "SEAKV_PREFILL_V=%d: unknown prefill variant (2, 9, 10)\n", version);
    std::abort();
  }
}

}  // namespace

void launch_prefill(const DataParams& p, cudaStream_t s) {
  if (p.nreq <= 0) return;
  if (p.dtype == 0) launch_prefill_t<__half>(p, s);
  else launch_prefill_t<__nv_bfloat16>(p, s);
}

}  // namespace skv

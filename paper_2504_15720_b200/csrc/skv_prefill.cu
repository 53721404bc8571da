// skv_prefill.cu — causal chunked-prefill attention over the unified pool on the
// 5th-generation tensor cores (tcgen05.mma, accumulators in TMEM), sm_100a.
//
// Each request's last q_len tokens (per request) attend causally to every key at or before
// their own position; K/V are read through the request's block table (reference block
// layout, kv_cache.hpp:178-182; per-(layer, kv head) runs of 16 tokens).  GQA
// query rows are folded into M: row i of a 128-row query tile is (token t0 + i/G, q head
// kv_head*G + i%G), so one K/V tile feeds G query heads.
//
// prefill_kernel<T, D> (head dim D = 64, 128, 256): CTA pairs, one 256-row
// tcgen05.mma.cta_group::2 per K=16 step (N = 128 keys for S = Q.K^T, N = D dims for
// O += P.V), K/V halves per SM by TMA, S double-buffered in TMEM, persistent with a dynamic
// work counter.  prefill_pp_kernel<T> (head dim 128, the default for it): the same pairs with
// two query tiles per CTA and one softmax warpgroup each (ping-pong, see below).  (Earlier
// single-CTA variants v2-v9 are in git history; DESIGN.md §5.2 has the measurements.)
//
// UMMA operand layouts (cute canonical): K-major SW128 atoms of [8 rows x 64 elements]
// (128 B rows, 16-byte chunk c of row r at chunk c ^ (r%8)) for Q and K — a [R x D] tile is
// D/64 atom columns of R x 128 B, advance 32 B per K=16 step; V is MN-major: SW128 atoms of
// 64 dims (D = 128, 256: each CTA holds D/2 dims = 1 or 2 atom columns, SBO 1 KiB, advance
// 2 KiB per 16 keys) or, for D = 64 (32 dims per CTA), SW64 atoms of 32 dims (64 B rows,
// SBO 512 B, advance 1 KiB per 16 keys).  One TMA box {64 (or 32) elements, 16 rows} = one
// native block's K or V run (or a 64-dim slice of it) lands directly in this layout.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "skv_internal.h"

namespace skv {

namespace {

constexpr int kTpb = 16;
constexpr int kRows = 128;  // query rows per CTA (M = 256 per CTA pair)
constexpr int kKT = 128;    // keys per tile (N of S = Q.K^T across the pair)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
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

// UMMA shared-memory descriptor (cute::UMMA::SmemDescriptor, version 1); layout 2 = SWIZZLE_128B,
// 4 = SWIZZLE_64B (bits 61-63).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (Blackwell)
  d |= (uint64_t)layout << 61;
  return d;
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
// ---------------------------------------------------------------------------------------
// Warp-specialised kernel (earlier v2-v9 steps are in git history and in DESIGN.md):
// warps 0-7 softmax (two warps per TMEM lane quarter), warp 8 issues every
// tcgen05.mma from one thread, warp 9 streams K/V with TMA, all handshakes on mbarriers.
constexpr int kSoftmaxWarps = 8;             // 4 per query tile, one thread per query row
constexpr int kMmaWarp = kSoftmaxWarps;      // warp 8
constexpr int kLoadWarp = kSoftmaxWarps + 1; // warp 9
constexpr int kThreadsV3 = (kSoftmaxWarps + 2) * 32;

__device__ __forceinline__ void mbar_init_n(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
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
// CTA pairs (cta_group::2).  A 128x64x16 UMMA issues at 55 clk instead of 32
// (profiles/r01_umma_bench.txt), so single-CTA 64-key QK^T tiles ran the tensor core at ~58 %, and a
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
__device__ __forceinline__ uint32_t make_idesc_pair(int bf16, int b_mn_major, int n) {
  uint32_t d = 0;
  d |= 1u << 4;                     // fp32 accumulate
  d |= (uint32_t)bf16 << 7;         // A type
  d |= (uint32_t)bf16 << 10;        // B type
  d |= (uint32_t)b_mn_major << 16;  // B MN-major (V)
  d |= (uint32_t)(n >> 3) << 17;    // N
  d |= (uint32_t)(256 >> 4) << 24;  // M = 256 (128 rows per CTA)
  return d;
}
// both operands from shared memory (D = 256: Q in smem), cta_group::2
__device__ __forceinline__ void mma_f16_ss_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tmem_st16u(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}


constexpr float kRescale = 8.0f;  // log2 threshold for the lazy O correction
constexpr int kRing = 8;          // work-item ring (scheduler -> roles)

// Per-head-dim geometry of the CTA-pair kernel.  Per stage and CTA: K = this CTA's 64 keys
// of the 128-key tile x D dims (D/64 SW128 atom columns of 64 rows x 128 B), V = all 128
// keys x this CTA's D/2 dims (SW128 atom columns of 128 rows x 128 B; D = 64: one SW64 atom
// of 128 rows x 64 B).  TMEM (512 columns per SM): O [0, D) | S0 | S1 (128 each) | Q (D/4,
// D <= 128); D = 256 keeps Q in shared memory (SS-form QK^T) since O alone takes 256 columns.
template <int D>
struct PF {
  static constexpr int KATOMS = D / 64 > 0 ? D / 64 : 1;
  static constexpr int K_ATOM = 64 * 128;
  static constexpr int K_BYTES = KATOMS * K_ATOM;
  static constexpr bool V_SW64 = D == 64;
  static constexpr int V_ROW = V_SW64 ? 64 : 128;  // bytes of one key row of a V atom
  static constexpr int V_ATOMS = V_SW64 ? 1 : D / 128;
  static constexpr int V_ATOM = kKT * V_ROW;
  static constexpr int V_BYTES = V_ATOMS * V_ATOM;
  static constexpr int STAGE = K_BYTES + V_BYTES;
  static constexpr bool Q_SMEM = D == 256;
  static constexpr int Q_BYTES = Q_SMEM ? kRows * D * 2 : 0;
  static constexpr int STAGES = D == 256 ? 2 : 6;
  static constexpr int S0 = D > 128 ? D : 128;  // TMEM column of S(0); S(1) at S0 + 128
  static constexpr int QCOL = S0 + 256;         // TMEM column of Q (D <= 128)
  static constexpr int NQK = D / 16;            // K=16 MMAs of a QK^T tile
  static constexpr int OHALF = D / 2;           // O columns per softmax warp half
  static constexpr int XM_OFF = Q_BYTES + STAGES * STAGE;
  static constexpr int BAR_OFF = XM_OFF + 4096;
  static constexpr int SMEM = BAR_OFF + 512;
  static_assert(SMEM <= 227 * 1024, "shared memory");
  static_assert(S0 + 256 + (Q_SMEM ? 0 : D / 4) <= 512, "TMEM columns");
};

// per-request chunk length and the request's first row in its group's q / out tensor
__device__ __forceinline__ int qlen_of(const DataParams& p, int r) { return p.q_lens ? p.q_lens[r] : p.n_new; }
__device__ __forceinline__ int qoff_of(const DataParams& p, int r, int rl) {
  return p.q_offs ? p.q_offs[r] : rl * p.n_new;
}

// Work items are numbered densely group by group (pf_base / pf_npairs set per launch): a
// group's items are (request, kv head) major, query-tile pair descending minor, so the pairs of
// one (request, head) -- which read the same K/V -- run at the same time on different SMs (L2
// reuse) and each (request, head) starts with its longest pair.  Only pairs past a ragged
// request's own chunk are skipped.
__device__ __forceinline__ bool prefill_item(const DataParams& p, int i, int& r, int& h, int& pair,
                                             int item_rows = 2 * kRows) {
  int gi = 0;
  while (gi + 1 < p.ngroups && i >= p.g[gi + 1].pf_base) ++gi;
  const DataGroup& g = p.g[gi];
  const int rem = i - g.pf_base;
  pair = g.pf_npairs - 1 - rem % g.pf_npairs;
  const int rh = rem / g.pf_npairs;
  h = rh % g.Hkv;
  r = g.req_begin + rh / g.Hkv;
  return pair * item_rows < qlen_of(p, r) * g.G;
}

template <typename T, int D>
__global__ void __launch_bounds__(kThreadsV3, 1) prefill_kernel(const __grid_constant__ DataParams p, int n_items) {
  using F = PF<D>;
  extern __shared__ __align__(1024) char smem[];
  if (smem_u32(smem) & 1023) __trap();
#ifdef SKV_PF_TRACE
  long long pf_acc[5] = {0, 0, 0, 0, 0};
  const long long pf_start = clock64();
  long long pf_tiles = 0;
#endif
  char* qbase = smem;                  // D = 256: [128 rows x 256 d] K-major SW128 (4 atom columns)
  char* kvbase = smem + F::Q_BYTES;    // [stages][K | V]
  float* xm = reinterpret_cast<float*>(smem + F::XM_OFF);  // [2 parity][2 half][128 rows]
  float* xl = xm + 512;                                     // [2 half][128 rows]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + F::BAR_OFF);
  constexpr int ST = F::STAGES;
  uint64_t* kv_full = bars;                 // [stages] leader: both CTAs' bytes
  uint64_t* kv_empty = bars + ST;           // [stages] both CTAs (multicast commit)
  // Barriers indexed by [tile parity]: a softmax warp can finish S(j+1) before the MMA warp
  // has consumed P(j), and parity waits cannot tell phases two apart.
  uint64_t* q_full = bars + 2 * ST;         // leader: 16 warp arrivals per item
  uint64_t* p_full = bars + 2 * ST + 1;     // [2] leader: 16 warp arrivals
  uint64_t* s_full = bars + 2 * ST + 3;     // [2] both CTAs (multicast commit)
  uint64_t* pv_done = bars + 2 * ST + 5;    // [2] both CTAs (multicast commit)
  uint64_t* item_full = bars + 2 * ST + 7;  // [kRing] both CTAs
  int* ring = reinterpret_cast<int*>(bars + 2 * ST + 7 + kRing);  // [kRing]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + kRing);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();

  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init_n(&kv_full[i], 1);
      mbar_init_n(&kv_empty[i], 1);
    }
    mbar_init_n(q_full, 16);
    for (int i = 0; i < 2; ++i) {
      mbar_init_n(&p_full[i], 16);
      mbar_init_n(&s_full[i], 1);
      mbar_init_n(&pv_done[i], 1);
    }
    for (int i = 0; i < kRing; ++i) mbar_init_n(&item_full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t q_full_l = mapa_u32(smem_u32(q_full), 0), p_full_l = mapa_u32(smem_u32(p_full), 0);

  struct Geo {
    int r, h, pair, handle, ctx, start, tpt, t0A, n_keys, n_kt, rl, G, q_len, q_off;
    const DataGroup* g;
  };
  auto geo = [&](int idx) {
    Geo e;
    prefill_item(p, idx, e.r, e.h, e.pair);
    e.g = &p.g[p.req_group[e.r]];
    e.G = e.g->G;
    e.handle = p.handles[e.r];
    e.ctx = p.req_tokens[e.handle];
    e.rl = e.r - e.g->req_begin;
    e.q_len = qlen_of(p, e.r);
    e.q_off = qoff_of(p, e.r, e.rl);
    e.start = e.ctx - e.q_len;
    e.tpt = kRows / e.G;
    e.t0A = 2 * e.pair * e.tpt;
    e.n_keys = min(e.ctx, e.start + e.t0A + 2 * e.tpt);
    e.n_kt = (e.n_keys + kKT - 1) / kKT;
    return e;
  };
  auto next_item = [&](uint32_t k) {
    mbar_wait_cl(&item_full[k % kRing], (k / kRing) & 1);
    return *reinterpret_cast<volatile int*>(&ring[k % kRing]);
  };

  if (warp == kLoadWarp) {  // --------------------------------- scheduler (leader) + K/V streaming (both)
    // Whole warp: lane i holds block-table entry i of the current 32-entry chunk (4 key tiles)
    // and the next chunk is already in flight, so the table's load latency is off the TMA
    // issue path; the 8 lanes of a tile issue its boxes in parallel.
    const void* kmap = D == 64 ? &p.kv_tmap64 : D == 128 ? &p.kv_tmap : &p.kv_tmap256;
    const void* vmap = D == 64 ? &p.kv_tmap64v : kmap;
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
            if (prefill_item(p, idx, r_, h_, pr_)) break;
            idx = atomicAdd(p.counter, 1);
          }
          pub = idx < n_items ? idx : -1;
          const uint32_t slot = k % kRing;
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
      {  // this CTA's Q rows of the item -> L2 (the softmax warps install them one item ahead)
        const int t0 = e.t0A + (int)rank * e.tpt, ntok = min(e.tpt, e.q_len - t0);
        const char* qb = reinterpret_cast<const char*>(e.g->q) +
                         (((size_t)e.q_off + t0) * e.g->Hq + (size_t)e.h * e.G) * (D * 2);
        for (int t = lane; t < ntok; t += 32)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(qb + (size_t)t * e.g->Hq * (D * 2)),
                       "r"(e.G * D * 2)
                       : "memory");
      }
      const int2* row_tab = p.req_table + (size_t)e.handle * p.cap;
      const long long base_off = e.g->layer_off + (long long)e.h * e.g->head_stride;
      const int n_blk = (e.n_keys + kTpb - 1) / kTpb;
      int2 ent_next = lane < n_blk ? row_tab[lane] : make_int2(-1, 0);
      int row0 = 0;
      bool valid = false;
      for (int j = 0; j < e.n_kt; ++j, ++jt) {
        if ((j & 3) == 0) {
          valid = ent_next.x >= 0;
          // TMA row = one token's 2*D-byte K or V row
          row0 = valid ? (int)(((long long)ent_next.x * p.merged_stride + (long long)ent_next.y * e.g->native_stride +
                                base_off) / (2 * D))
                       : 0;
          const int nx = (j + 4) * 8 + lane;
          ent_next = nx < n_blk ? row_tab[nx] : make_int2(-1, 0);
        }
        const int st = jt % ST;
        if (jt >= (uint32_t)ST) {
          if (lane == 0) PF_T(0, mbar_wait(&kv_empty[st], ((jt / ST) - 1) & 1));
          __syncwarp();
        }
        const int grp = (j & 3) * 8;
        const bool mine = lane >= grp && lane < grp + 8 && valid;
        const int nb = __popc(__ballot_sync(0xffffffffu, mine));
        // leader expects both CTAs' bytes: the block's K run (one CTA) + its V run (both halves)
        if (rank == 0 && lane == 0) mbar_expect_tx_v3(&kv_full[st], nb * (64 * D));
        __syncwarp();
        if (mine) {
          const int b = lane - grp;
          const uint32_t sK = smem_u32(kvbase + st * F::STAGE), sV = sK + F::K_BYTES;
          const uint32_t bar = kv_full_l + 8 * st;
          if ((b >> 2) == (int)rank) {  // this CTA's 64 keys of K, every 64-dim atom column
#pragma unroll
            for (int a = 0; a < F::KATOMS; ++a) tma_load_2d_pair(sK + a * F::K_ATOM + (b & 3) * 2048, kmap, 64 * a, row0, bar);
          }
          // this CTA's D/2 dims of V, all 8 blocks of the tile
#pragma unroll
          for (int a = 0; a < F::V_ATOMS; ++a)
            tma_load_2d_pair(sV + a * F::V_ATOM + b * (kTpb * F::V_ROW), vmap, (int)rank * (D / 2) + 64 * a,
                             row0 + kTpb, bar);
        }
      }
    }
  } else if (warp == kMmaWarp) {  // ------------------------------------- MMA issue (leader only)
    if (lane == 0 && rank == 0) {
      const uint32_t idesc_qk = make_idesc_pair(p.dtype, 0, kKT);
      const uint32_t idesc_pv = make_idesc_pair(p.dtype, 1, D);
      const uint64_t k_desc0 = make_desc(smem_u32(kvbase), 16, 1024);
      const uint64_t v_desc0 = F::V_SW64 ? make_desc(smem_u32(kvbase) + F::K_BYTES, F::V_ATOM, 512, 4)
                                         : make_desc(smem_u32(kvbase) + F::K_BYTES, F::V_ATOM, 1024);
      const uint64_t q_desc0 = make_desc(smem_u32(qbase), 16, 1024);
      uint32_t jt = 0;
      for (uint32_t k = 0;; ++k) {
        const int idx = next_item(k);
        if (idx < 0) break;
        const Geo e = geo(idx);
        const uint32_t j0 = jt;
        const int J = e.n_kt;
        auto wait_kv = [&](int j) {
          const uint32_t gj = j0 + j;
          PF_T(1, mbar_wait(&kv_full[gj % ST], (gj / ST) & 1));
          tc_fence_after();
        };
        // descriptors of a tile's MMAs are materialised before the barrier wait that gates
        // them, so the issue burst after the wait is MMAs only (per-MMA descriptor arithmetic
        // on the issuing thread left the 64-clk MMAs issue-bound, profiles/r01_prefill_v10_diagnostics.txt)
        // descriptor = base descriptor of stage 0 + (byte offset >> 4) in the address field
        // (shared-memory addresses < 256 KiB: the 14-bit field never carries)
        auto k_descs = [&](int j, uint64_t (&d)[F::NQK]) {
          const uint64_t b = k_desc0 + (uint64_t)(((j0 + j) % ST) * (F::STAGE >> 4));
#pragma unroll
          for (int kk = 0; kk < F::NQK; ++kk) d[kk] = b + (uint64_t)(((kk >> 2) * F::K_ATOM + (kk & 3) * 32) >> 4);
        };
        auto v_descs = [&](int j, uint64_t (&d)[8]) {
          const uint64_t b = v_desc0 + (uint64_t)(((j0 + j) % ST) * (F::STAGE >> 4));
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) d[kk] = b + (uint64_t)((kk * kTpb * F::V_ROW) >> 4);
        };
        auto pin = [](const uint64_t* d, int n) {  // force the values into registers here
#pragma unroll
          for (int i = 0; i < n; ++i) asm volatile("" ::"l"(d[i]));
        };
        auto qk = [&](int j, const uint64_t (&d)[F::NQK]) {
          const uint32_t gj = j0 + j;
          const uint32_t tS = tmem + F::S0 + (gj & 1) * 128;
#pragma unroll
          for (int kk = 0; kk < F::NQK; ++kk) {
            if constexpr (F::Q_SMEM)
              mma_f16_ss_pair(tS, q_desc0 + (uint64_t)(((kk >> 2) * (kRows * 128) + (kk & 3) * 32) >> 4), d[kk],
                              idesc_qk, kk > 0);
            else
              mma_f16_ts_pair(tS, tmem + F::QCOL + kk * 8, d[kk], idesc_qk, kk > 0);
          }
          mma_commit_pair(&s_full[gj & 1]);
        };
        auto pv = [&](int j, const uint64_t (&d)[8]) {
          const uint32_t gj = j0 + j;
          const uint32_t tP = tmem + F::S0 + (gj & 1) * 128;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) mma_f16_ts_pair(tmem, tP + kk * 8, d[kk], idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
          mma_commit_pair(&pv_done[gj & 1]);
          mma_commit_pair(&kv_empty[gj % ST]);
        };
        {
          uint64_t d0[F::NQK], d1[F::NQK];
          k_descs(0, d0);
          if (J > 1) k_descs(1, d1);
          pin(d0, F::NQK);
          pin(d1, F::NQK);
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
          uint64_t vd[8], kd[F::NQK];
          PF_T(4, {
            v_descs(j, vd);
            k_descs(j + 2, kd);
            pin(vd, 8);
            pin(kd, F::NQK);
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
    const uint32_t tO = tmem + F::OHALF * c + lane_off;
    const int nbar = 1 + (warp & 3);  // named barrier of the two warps sharing these rows
    constexpr int OCH = F::OHALF / 32;  // 32-column O chunks per half (1, 2, 4)
    // Q of an item is installed as soon as the previous item's last S tile has been consumed
    // (all of its QK^T retired), before that item's epilogue, so the next item's first QK^T
    // runs while the epilogue drains O (the loader prefetched the rows into L2)
    auto install_q = [&](const Geo& e) {
      const int t0 = e.t0A + (int)rank * e.tpt;
      const int my_tok = t0 + row / e.G;
      const bool row_ok = my_tok < e.q_len;
      {  // this thread's half of its Q row
        const uint4* src = reinterpret_cast<const uint4*>(
            reinterpret_cast<const char*>(e.g->q) +
            (((size_t)e.q_off + (row_ok ? my_tok : 0)) * e.g->Hq + e.h * e.G + row % e.G) * (D * 2) + c * D);
        if constexpr (F::Q_SMEM) {  // 128 dims = 2 SW128 atom columns of the [128 x 256] Q tile
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const uint4 v = row_ok ? src[i] : make_uint4(0u, 0u, 0u, 0u);
            const int a = 2 * c + (i >> 3), ch = i & 7;
            *reinterpret_cast<uint4*>(qbase + a * (kRows * 128) + (row >> 3) * 1024 + (row & 7) * 128 +
                                      ((ch ^ (row & 7)) << 4)) = v;
          }
          fence_async_smem();  // generic-proxy writes read by the (leader's) tensor core
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster_rel(q_full_l);
        } else {
          constexpr int NW = D / 4;  // packed 32-bit words of this thread's half row (16 or 32)
          uint32_t qv[NW];
#pragma unroll
          for (int i = 0; i < NW / 4; ++i) {
            const uint4 v = row_ok ? src[i] : make_uint4(0u, 0u, 0u, 0u);
            qv[4 * i] = v.x;
            qv[4 * i + 1] = v.y;
            qv[4 * i + 2] = v.z;
            qv[4 * i + 3] = v.w;
          }
          const uint32_t tQ = tmem + F::QCOL + (D / 4) * c + lane_off;
          if constexpr (NW == 32) tmem_st32u(tQ, *reinterpret_cast<const uint32_t(*)[32]>(qv));
          else tmem_st16u(tQ, qv);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster_relaxed(q_full_l);
        }
      }
    };
    uint32_t jt = 0;
    int idx = next_item(0);
    if (idx >= 0) install_q(geo(idx));
    for (uint32_t k = 0; idx >= 0; ++k) {
      const Geo e = geo(idx);
      const float c2 = e.g->scale_log2;
      const int t0 = e.t0A + (int)rank * e.tpt;
      const int my_tok = t0 + row / e.G;
      const bool row_ok = my_tok < e.q_len;
      const int my_pos = e.start + my_tok;
      const bool tail_rows = t0 + e.tpt > e.q_len;
      float m = -INFINITY, l = 0.f;
      const uint32_t j0 = jt;
      for (int j = 0; j < e.n_kt; ++j) {
        const uint32_t gj = j0 + j;
        const uint32_t tS = tmem + F::S0 + (gj & 1) * 128 + lane_off;
        PF_T(0, mbar_wait(&s_full[gj & 1], (gj >> 1) & 1));
        tc_fence_after();
        const bool last_partial = j == e.n_kt - 1 && (j + 1) * kKT > e.n_keys;
        if (last_partial) {  // V rows past the keys (stale or another owner's bytes) -> 0
          char* sV = kvbase + (gj % ST) * F::STAGE + F::K_BYTES;
          const int first = e.n_keys - j * kKT;
          constexpr int CPRV = F::V_ROW / 16;  // 16-B chunks of a V atom row (whole rows: swizzle-agnostic)
          for (int i = tid; i < kKT * CPRV * F::V_ATOMS; i += 256) {
            const int a = i / (kKT * CPRV), rem = i % (kKT * CPRV), key = rem / CPRV, ch = rem % CPRV;
            if (key >= first) *reinterpret_cast<uint4*>(sV + a * F::V_ATOM + key * F::V_ROW + ch * 16) = make_uint4(0, 0, 0, 0);
          }
        }
        const int kbase = j * kKT + 64 * c;
        const bool masked = (kbase + 63 > e.start + t0) || tail_rows;
        // path decision shared by the two warps of a row pair (same rows, same tile)
        const bool tile_masked = (j * kKT + kKT - 1 > e.start + t0) || tail_rows;
        float* xmb = xm + (gj & 1) * 256;
        float ls[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t pk[32];
        auto rescale_o = [&](float alpha) {  // O holds P.V through tile j-1: scale it in TMEM
#pragma unroll
          for (int cc = 0; cc < OCH; ++cc) {
            float o[32];
            tmem_ld32(tO + cc * 32, o);
#pragma unroll
            for (int kk = 0; kk < 32; ++kk) o[kk] *= alpha;
            tmem_st32(tO + cc * 32, o);
          }
        };
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
            rescale_o(alpha);
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
            rescale_o(alpha);
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
      const int nidx = next_item(k + 1);
      if (nidx >= 0) install_q(geo(nidx));
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
                  (((size_t)e.q_off + (row_ok ? my_tok : 0)) * e.g->Hq + e.h * e.G + row % e.G) * (D * 2) + c * D;
#pragma unroll
      for (int cc = 0; cc < OCH; ++cc) {
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
      idx = nidx;
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

// ---------------------------------------------------------------------------------------
// Ping-pong variant for head dim 128 (prefill_pp_kernel): every CTA of a pair holds TWO
// 128-row query tiles, A and B, each with its own softmax warpgroup (warps 0-3: A, 4-7: B,
// one thread per query row, all 128 key columns), so a TMEM lane quarter -- and an SM
// sub-partition -- carries one A warp and one B warp whose tile phases are offset by half a
// period: softmax(A, j) runs while the tensor core computes P.V(B, j-1) and S(B, j), and
// vice versa.  No row-max exchange between warps; the running max is speculative (a 32-key
// chunk is exponentiated against it and it is raised -- rescaling O, l and the chunks
// already stored -- only when the chunk's max exceeds it by 2^kRescale).
//   TMEM: O_A [0,128) | O_B [128,256) | S_A [256,384) | S_B [384,512); P_X over S_X [0,64).
//   SMEM: Q_A | Q_B (K-major SW128, SS-form Q.K^T) | 5 K/V stages (same halves as above).
// An item is four query tiles of a (request, kv head): A = tiles 0 (rank 0) and 1 (rank 1),
// B = tiles 2 and 3; the K/V stream is shared by both.
namespace pp {
constexpr int kWarps = 12;  // 0-3 softmax A, 4-7 softmax B, 8 MMA, 9 scheduler + TMA, 10-11 idle
// registers: launched at 168 per thread (12 warps), then setmaxnreg moves 80 per thread from
// warpgroup 2 (MMA, loader) to the two softmax warpgroups
constexpr int kRegSoftmax = 208, kRegOther = 88;  // 2*208 + 88 = 3*168
constexpr int kThreads = kWarps * 32;
constexpr int kD = 128;
constexpr int kQTile = kRows * kD * 2;  // 32 KiB: 2 SW128 atom columns of 128 rows x 128 B
constexpr int kKBytes = 2 * 64 * 128;   // this CTA's 64 keys x 128 dims
constexpr int kVAtom = kKT * 128;       // all 128 keys x this CTA's 64 dims
constexpr int kStage = kKBytes + kVAtom;
constexpr int kStages = 5;
constexpr int kKvOff = 2 * kQTile;
constexpr int kBarOff = kKvOff + kStages * kStage;
constexpr int kSmem = kBarOff + 512;
constexpr int kOCol = 0, kSCol = 256;  // + 128 * X
constexpr int kItemRows = 4 * kRows;
static_assert(kSmem <= 227 * 1024, "shared memory");
}  // namespace pp

__device__ __forceinline__ void tmem_st16_nowait(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// Rare path of the ping-pong softmax (a tile raised a row's running max by more than
// 2^kRescale): O (through the previous tile; that P.V has retired) is rescaled by alpha in
// TMEM.  Out of line to keep the hot loop small (instruction cache).
__device__ __noinline__ void pp_rescale_o(uint32_t tO, float alpha) {
  for (int cc = 0; cc < 4; ++cc) {
    float o[32];
    tmem_ld32(tO + cc * 32, o);
#pragma unroll
    for (int kk = 0; kk < 32; ++kk) o[kk] *= alpha;
    tmem_st32(tO + cc * 32, o);
  }
}

// 2^x for two values on the FMA/ALU pipes (FA4-style MUFU offload): x clamped to -125, split
// x = j + f (round-to-nearest through the 1.5*2^23 magic add), 2^f by a degree-3 minimax
// polynomial on [-0.5, 0.5] (max rel. error 1.3e-4, below fp16's half ulp), 2^j added into
// the exponent field (LEA).  Packed FADD2/FFMA2: 10 instructions per pair.
__device__ __forceinline__ float2 ex2_emu2(float2 x) {
  x.x = fmaxf(x.x, -125.f);
  x.y = fmaxf(x.y, -125.f);
  const float2 t = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
  const float2 jf = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 fr = __fadd2_rn(x, make_float2(-jf.x, -jf.y));
  float2 q = __ffma2_rn(fr, make_float2(0.05504561f, 0.05504561f), make_float2(0.24229777f, 0.24229777f));
  q = __ffma2_rn(q, fr, make_float2(0.69325471f, 0.69325471f));
  q = __ffma2_rn(q, fr, make_float2(0.99994976f, 0.99994976f));
  return make_float2(__uint_as_float(__float_as_uint(q.x) + (__float_as_uint(t.x) << 23)),
                     __uint_as_float(__float_as_uint(q.y) + (__float_as_uint(t.y) << 23)));
}
#ifndef SKV_PP_EMU
#define SKV_PP_EMU 6  // exponential pairs of every 16 (per 32 keys) computed by ex2_emu2 (swept: 0-10, 6 best)
#endif

// warp-wide issue: the whole (converged) warp runs the MMA loop, one elected lane issues
// eight K=16 steps of one tile in one asm block: one elect, only the descriptors' low words
// move (immediate steps: Q atom column 16 KiB / K atom column 8 KiB per 4 steps, 32 B per step;
// V 2 KiB and P 8 TMEM columns per step), high words are compile-time constants; `acc0` =
// accumulate on the first step
template <uint32_t AHI, uint32_t BHI>
__device__ __forceinline__ void qk8_pair(uint32_t tmem_d, uint32_t alo, uint32_t blo, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      ".reg .b32 al<8>, bl<8>, ah, bh;\n\t.reg .b64 a<8>, b<8>;\n\t"
      "mov.b32 ah, %5;\n\tmov.b32 bh, %6;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "add.u32 al0, %1, 0;\n\tmov.b64 a0, {al0, ah};\n\t"
      "add.u32 bl0, %2, 0;\n\tmov.b64 b0, {bl0, bh};\n\t"
      "add.u32 al1, %1, 2;\n\tmov.b64 a1, {al1, ah};\n\t"
      "add.u32 bl1, %2, 2;\n\tmov.b64 b1, {bl1, bh};\n\t"
      "add.u32 al2, %1, 4;\n\tmov.b64 a2, {al2, ah};\n\t"
      "add.u32 bl2, %2, 4;\n\tmov.b64 b2, {bl2, bh};\n\t"
      "add.u32 al3, %1, 6;\n\tmov.b64 a3, {al3, ah};\n\t"
      "add.u32 bl3, %2, 6;\n\tmov.b64 b3, {bl3, bh};\n\t"
      "add.u32 al4, %1, 1024;\n\tmov.b64 a4, {al4, ah};\n\t"
      "add.u32 bl4, %2, 512;\n\tmov.b64 b4, {bl4, bh};\n\t"
      "add.u32 al5, %1, 1026;\n\tmov.b64 a5, {al5, ah};\n\t"
      "add.u32 bl5, %2, 514;\n\tmov.b64 b5, {bl5, bh};\n\t"
      "add.u32 al6, %1, 1028;\n\tmov.b64 a6, {al6, ah};\n\t"
      "add.u32 bl6, %2, 516;\n\tmov.b64 b6, {bl6, bh};\n\t"
      "add.u32 al7, %1, 1030;\n\tmov.b64 a7, {al7, ah};\n\t"
      "add.u32 bl7, %2, 518;\n\tmov.b64 b7, {bl7, bh};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a0, b0, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a3, b3, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a4, b4, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a5, b5, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a6, b6, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a7, b7, %3, 1;\n\t"
      "}"
      ::"r"(tmem_d), "r"(alo), "r"(blo), "r"(idesc), "r"(acc0), "n"(AHI), "n"(BHI));
}
template <uint32_t BHI>
__device__ __forceinline__ void pv8_pair(uint32_t tmem_d, uint32_t tmem_a, uint32_t blo, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\t"
      ".reg .b32 a<8>, bl<8>, bh;\n\t.reg .b64 b<8>;\n\t"
      "mov.b32 bh, %5;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "add.u32 a0, %1, 0;\n\t"
      "add.u32 bl0, %2, 0;\n\tmov.b64 b0, {bl0, bh};\n\t"
      "add.u32 a1, %1, 8;\n\t"
      "add.u32 bl1, %2, 128;\n\tmov.b64 b1, {bl1, bh};\n\t"
      "add.u32 a2, %1, 16;\n\t"
      "add.u32 bl2, %2, 256;\n\tmov.b64 b2, {bl2, bh};\n\t"
      "add.u32 a3, %1, 24;\n\t"
      "add.u32 bl3, %2, 384;\n\tmov.b64 b3, {bl3, bh};\n\t"
      "add.u32 a4, %1, 32;\n\t"
      "add.u32 bl4, %2, 512;\n\tmov.b64 b4, {bl4, bh};\n\t"
      "add.u32 a5, %1, 40;\n\t"
      "add.u32 bl5, %2, 640;\n\tmov.b64 b5, {bl5, bh};\n\t"
      "add.u32 a6, %1, 48;\n\t"
      "add.u32 bl6, %2, 768;\n\tmov.b64 b6, {bl6, bh};\n\t"
      "add.u32 a7, %1, 56;\n\t"
      "add.u32 bl7, %2, 896;\n\tmov.b64 b7, {bl7, bh};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a0], b0, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a1], b1, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a2], b2, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a3], b3, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a4], b4, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a5], b5, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a6], b6, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a7], b7, %3, 1;\n\t"
      "}"
      ::"r"(tmem_d), "r"(tmem_a), "r"(blo), "r"(idesc), "r"(acc0), "n"(BHI));
}
// a quarter of a P.V tile (K-steps [2Q, 2Q+2), keys 32Q..32Q+31)
template <uint32_t BHI, int Q>
__device__ __forceinline__ void pv2_pair(uint32_t tmem_d, uint32_t tmem_a, uint32_t blo, uint32_t idesc, uint32_t acc0) {
  if constexpr (Q == 0)
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
      ".reg .b32 a<2>, bl<2>, bh;\n\t.reg .b64 b<2>;\n\t"
      "mov.b32 bh, %5;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "add.u32 a0, %1, 0;\n\t"
      "add.u32 bl0, %2, 0;\n\tmov.b64 b0, {bl0, bh};\n\t"
      "add.u32 a1, %1, 8;\n\t"
      "add.u32 bl1, %2, 128;\n\tmov.b64 b1, {bl1, bh};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a0], b0, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a1], b1, %3, 1;\n\t"
      "}"
        ::"r"(tmem_d), "r"(tmem_a), "r"(blo), "r"(idesc), "r"(acc0), "n"(BHI));
  else if constexpr (Q == 1)
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
      ".reg .b32 a<2>, bl<2>, bh;\n\t.reg .b64 b<2>;\n\t"
      "mov.b32 bh, %5;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "add.u32 a0, %1, 16;\n\t"
      "add.u32 bl0, %2, 256;\n\tmov.b64 b0, {bl0, bh};\n\t"
      "add.u32 a1, %1, 24;\n\t"
      "add.u32 bl1, %2, 384;\n\tmov.b64 b1, {bl1, bh};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a0], b0, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a1], b1, %3, 1;\n\t"
      "}"
        ::"r"(tmem_d), "r"(tmem_a), "r"(blo), "r"(idesc), "r"(acc0), "n"(BHI));
  else if constexpr (Q == 2)
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
      ".reg .b32 a<2>, bl<2>, bh;\n\t.reg .b64 b<2>;\n\t"
      "mov.b32 bh, %5;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "add.u32 a0, %1, 32;\n\t"
      "add.u32 bl0, %2, 512;\n\tmov.b64 b0, {bl0, bh};\n\t"
      "add.u32 a1, %1, 40;\n\t"
      "add.u32 bl1, %2, 640;\n\tmov.b64 b1, {bl1, bh};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a0], b0, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a1], b1, %3, 1;\n\t"
      "}"
        ::"r"(tmem_d), "r"(tmem_a), "r"(blo), "r"(idesc), "r"(acc0), "n"(BHI));
  else if constexpr (Q == 3)
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
      ".reg .b32 a<2>, bl<2>, bh;\n\t.reg .b64 b<2>;\n\t"
      "mov.b32 bh, %5;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "add.u32 a0, %1, 48;\n\t"
      "add.u32 bl0, %2, 768;\n\tmov.b64 b0, {bl0, bh};\n\t"
      "add.u32 a1, %1, 56;\n\t"
      "add.u32 bl1, %2, 896;\n\tmov.b64 b1, {bl1, bh};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a0], b0, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a1], b1, %3, 1;\n\t"
      "}"
        ::"r"(tmem_d), "r"(tmem_a), "r"(blo), "r"(idesc), "r"(acc0), "n"(BHI));
}
__device__ __forceinline__ void commit_pair_e(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"((unsigned short)3)
      : "memory");
}

template <typename T>
__global__ void __launch_bounds__(pp::kThreads, 1) prefill_pp_kernel(const __grid_constant__ DataParams p, int n_items) {
  using namespace pp;
  extern __shared__ __align__(1024) char smem[];
  if (smem_u32(smem) & 1023) __trap();
  char* qbase = smem;  // [X][128 rows x 128 d]
  char* kvbase = smem + kKvOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kBarOff);
  constexpr int ST = kStages;
  uint64_t* kv_full = bars;                 // [stages] leader: both CTAs' bytes
  uint64_t* kv_empty = bars + ST;           // [stages] both CTAs (multicast commit)
  uint64_t* q_full = bars + 2 * ST;         // [X] leader: 8 warp arrivals per item
  uint64_t* p_full = bars + 2 * ST + 2;     // [X] leader: 8 warp arrivals per tile
  uint64_t* s_full = bars + 2 * ST + 4;     // [X] both CTAs (multicast commit)
  uint64_t* o_done = bars + 2 * ST + 6;     // [X] both CTAs: the item's last P.V retired
  uint64_t* p_part = bars + 2 * ST + 8;     // [3][X] leader: 8 warp arrivals per tile (P keys < 32, 64, 96 stored)
  uint64_t* item_full = bars + 2 * ST + 14; // [kRing] both CTAs
  int* ring = reinterpret_cast<int*>(bars + 2 * ST + 14 + kRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + kRing);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_rank();
#ifdef SKV_PF_TRACE
  long long pf_acc[5] = {0, 0, 0, 0, 0};
  const long long pf_start = clock64();
  long long pf_tiles = 0;
#endif

  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init_n(&kv_full[i], 1);
      mbar_init_n(&kv_empty[i], 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init_n(&q_full[x], 8);
      mbar_init_n(&p_full[x], 8);
      for (int q = 0; q < 3; ++q) mbar_init_n(&p_part[2 * q + x], 8);
      mbar_init_n(&s_full[x], 1);
      mbar_init_n(&o_done[x], 1);
    }
    for (int i = 0; i < kRing; ++i) mbar_init_n(&item_full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  struct Geo {
    int r, h, quad, handle, ctx, start, tpt, t0Q, n_keys, n_kt, rl, G, q_len, q_off;
    const DataGroup* g;
  };
  auto geo = [&](int idx) {
    Geo e;
    prefill_item(p, idx, e.r, e.h, e.quad, kItemRows);
    e.g = &p.g[p.req_group[e.r]];
    e.G = e.g->G;
    e.handle = p.handles[e.r];
    e.ctx = p.req_tokens[e.handle];
    e.rl = e.r - e.g->req_begin;
    e.q_len = qlen_of(p, e.r);
    e.q_off = qoff_of(p, e.r, e.rl);
    e.start = e.ctx - e.q_len;
    e.tpt = kRows / e.G;
    e.t0Q = 4 * e.quad * e.tpt;
    e.n_keys = min(e.ctx, e.start + e.t0Q + 4 * e.tpt);
    e.n_kt = (e.n_keys + kKT - 1) / kKT;
    return e;
  };
  auto next_item = [&](uint32_t k) {
    mbar_wait_cl(&item_full[k % kRing], (k / kRing) & 1);
    return *reinterpret_cast<volatile int*>(&ring[k % kRing]);
  };

  if (warp >= 8) {  // warpgroup 2: one setmaxnreg for all four warps (.aligned), then the roles
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegOther));
  if (warp >= 10) {  // idle
  } else if (warp == 9) {  // ------------------------------- scheduler (leader) + K/V streaming (both)
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
            if (prefill_item(p, idx, r_, h_, pr_, kItemRows)) break;
            idx = atomicAdd(p.counter, 1);
          }
          pub = idx < n_items ? idx : -1;
          const uint32_t slot = k % kRing;
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
#pragma unroll
      for (int x = 0; x < 2; ++x) {  // this CTA's Q rows of both tiles -> L2
        const int t0 = e.t0Q + (2 * x + (int)rank) * e.tpt, ntok = min(e.tpt, e.q_len - t0);
        const char* qb = reinterpret_cast<const char*>(e.g->q) +
                         (((size_t)e.q_off + t0) * e.g->Hq + (size_t)e.h * e.G) * (kD * 2);
        for (int t = lane; t < ntok; t += 32)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(qb + (size_t)t * e.g->Hq * (kD * 2)),
                       "r"(e.G * kD * 2)
                       : "memory");
      }
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
                                base_off) / (2 * kD))
                       : 0;
          const int nx = (j + 4) * 8 + lane;
          ent_next = nx < n_blk ? row_tab[nx] : make_int2(-1, 0);
        }
        const int st = jt % ST;
        if (jt >= (uint32_t)ST) {
          if (lane == 0) PF_T(0, mbar_wait(&kv_empty[st], ((jt / ST) - 1) & 1));
          __syncwarp();
        }
        const int grp = (j & 3) * 8;
        const bool mine = lane >= grp && lane < grp + 8 && valid;
        const int nb = __popc(__ballot_sync(0xffffffffu, mine));
        if (rank == 0 && lane == 0) mbar_expect_tx_v3(&kv_full[st], nb * (64 * kD));
        __syncwarp();
        if (mine) {
          const int b = lane - grp;
          const uint32_t sK = smem_u32(kvbase + st * kStage), sV = sK + kKBytes;
          const uint32_t bar = kv_full_l + 8 * st;
          if ((b >> 2) == (int)rank) {
            tma_load_2d_pair(sK + (b & 3) * 2048, &p.kv_tmap, 0, row0, bar);
            tma_load_2d_pair(sK + 8192 + (b & 3) * 2048, &p.kv_tmap, 64, row0, bar);
          }
          tma_load_2d_pair(sV + b * (kTpb * 128), &p.kv_tmap, (int)rank * 64, row0 + kTpb, bar);
        }
      }
    }
  } else {  // warp 8 --------------------------------------- MMA issue (leader; whole warp, elected lane)
    if (rank == 0) {
      const uint32_t idesc_qk = make_idesc_pair(p.dtype, 0, kKT);
      const uint32_t idesc_pv = make_idesc_pair(p.dtype, 1, kD);
      const uint64_t k_desc0 = make_desc(smem_u32(kvbase), 16, 1024);
      const uint64_t v_desc0 = make_desc(smem_u32(kvbase) + kKBytes, kVAtom, 1024);
      const uint64_t q_desc0 = make_desc(smem_u32(qbase), 16, 1024);
      uint32_t jt = 0;
      const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);  // warp-uniform (uniform datapath)
      for (uint32_t k = 0;; ++k) {
        const int idx = __shfl_sync(0xffffffffu, next_item(k), 0);
        if (idx < 0) break;
        const Geo e = geo(idx);
        const uint32_t j0 = jt;
        const int J = __shfl_sync(0xffffffffu, e.n_kt, 0);
        auto wait_kv = [&](int j) {
          const uint32_t gj = j0 + j;
          PF_T(1, mbar_wait(&kv_full[gj % ST], (gj / ST) & 1));
          tc_fence_after();
        };
        auto k_descs = [&](int j, uint64_t (&d)[8]) {
          const uint64_t b = k_desc0 + (uint64_t)(((j0 + j) % ST) * (kStage >> 4));
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) d[kk] = b + (uint64_t)(((kk >> 2) * 8192 + (kk & 3) * 32) >> 4);
        };
        auto v_descs = [&](int j, uint64_t (&d)[8]) {
          const uint64_t b = v_desc0 + (uint64_t)(((j0 + j) % ST) * (kStage >> 4));
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) d[kk] = b + (uint64_t)((kk * kTpb * 128) >> 4);
        };
        auto pin = [](const uint64_t* d, int n) {
#pragma unroll
          for (int i = 0; i < n; ++i) asm volatile("" ::"l"(d[i]));
        };
        // descriptor high words: SBO 1024 B, version 1, SWIZZLE_128B (K-major Q/K and MN-major V)
        constexpr uint32_t kHi = (1024u >> 4) | (1u << 14) | (2u << 29);
        auto qk = [&](int x, const uint64_t (&d)[8]) {
          qk8_pair<kHi, kHi>(tm + kSCol + 128 * x, (uint32_t)q_desc0 + (uint32_t)((x * kQTile) >> 4), (uint32_t)d[0],
                             idesc_qk, 0u);
          commit_pair_e(&s_full[x]);
        };
        auto pv = [&](int x, int j, const uint64_t (&d)[8]) {  // waits for the two P halves itself
          const uint32_t gj = j0 + j;
          const uint32_t tO_ = tm + kOCol + 128 * x, tP_ = tm + kSCol + 128 * x, vlo = (uint32_t)d[0];
          PF_T(2 + x, mbar_wait(&p_part[x], gj & 1));
          tc_fence_after();
          pv2_pair<kHi, 0>(tO_, tP_, vlo, idesc_pv, j > 0 ? 1u : 0u);
          PF_T(2 + x, mbar_wait(&p_part[2 + x], gj & 1));
          tc_fence_after();
          pv2_pair<kHi, 1>(tO_, tP_, vlo, idesc_pv, 1u);
          PF_T(2 + x, mbar_wait(&p_part[4 + x], gj & 1));
          tc_fence_after();
          pv2_pair<kHi, 2>(tO_, tP_, vlo, idesc_pv, 1u);
          PF_T(2 + x, mbar_wait(&p_full[x], gj & 1));
          tc_fence_after();
          pv2_pair<kHi, 3>(tO_, tP_, vlo, idesc_pv, 1u);
          if (j == J - 1) commit_pair_e(&o_done[x]);
        };
        {
          uint64_t kd[8];
          k_descs(0, kd);
          pin(kd, 8);
          PF_T(0, mbar_wait(&q_full[0], k & 1));
          tc_fence_after();
          wait_kv(0);
          qk(0, kd);
          PF_T(0, mbar_wait(&q_full[1], k & 1));
          tc_fence_after();
          qk(1, kd);
        }
        for (int j = 0; j < J; ++j) {
          const uint32_t gj = j0 + j;
          uint64_t vd[8], kd[8];
          v_descs(j, vd);
          k_descs(j + 1, kd);
          pin(vd, 8);
          pin(kd, 8);
          pv(0, j, vd);
          if (j + 1 < J) {
            wait_kv(j + 1);
            PF_T(4, qk(0, kd));
          }
          pv(1, j, vd);
          commit_pair_e(&kv_empty[gj % ST]);
          if (j + 1 < J) PF_T(4, qk(1, kd));
        }
        jt += J;
      }
    }
    __syncwarp();
  }
  } else {  // ---------------------------------------------------------------- softmax warps
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegSoftmax));
    const int x = warp >> 2;  // query tile (A = 0, B = 1)
    const int row = (warp & 3) * 32 + lane;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + kSCol + 128 * x + lane_off;
    const uint32_t tO = tmem + kOCol + 128 * x + lane_off;
    const uint32_t q_full_l = mapa_u32(smem_u32(&q_full[x]), 0), p_full_l = mapa_u32(smem_u32(&p_full[x]), 0),
                   p_part_l = mapa_u32(smem_u32(&p_part[x]), 0);  // + 16 * q: quarter q's barrier
    char* qtile = qbase + x * kQTile;
    auto install_q = [&](const Geo& e) {  // this thread's Q row into the tile's SW128 K-major layout
      const int t0 = e.t0Q + (2 * x + (int)rank) * e.tpt;
      const int my_tok = t0 + row / e.G;
      const bool row_ok = my_tok < e.q_len;
      const uint4* src = reinterpret_cast<const uint4*>(
          reinterpret_cast<const char*>(e.g->q) +
          (((size_t)e.q_off + (row_ok ? my_tok : 0)) * e.g->Hq + e.h * e.G + row % e.G) * (kD * 2));
      uint4 v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = row_ok ? src[i] : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int a = i >> 3, ch = i & 7;
        *reinterpret_cast<uint4*>(qtile + a * (kRows * 128) + (row >> 3) * 1024 + (row & 7) * 128 +
                                  ((ch ^ (row & 7)) << 4)) = v[i];
      }
      fence_async_smem();  // generic-proxy writes read by the (leader's) tensor core
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster_rel(q_full_l);
    };
    uint32_t tc = 0;
    int idx = next_item(0);
    if (idx >= 0) install_q(geo(idx));
    for (uint32_t k = 0; idx >= 0; ++k) {
      const Geo e = geo(idx);
      const float c2 = e.g->scale_log2;
      const int t0 = e.t0Q + (2 * x + (int)rank) * e.tpt;
      const int my_tok = t0 + row / e.G;
      const bool row_ok = my_tok < e.q_len;
      const int my_pos = e.start + my_tok;
      const bool tail_rows = t0 + e.tpt > e.q_len;
      float m = -INFINITY;  // reference max (log2 domain) of the row's P values
      float2 lsum = make_float2(0.f, 0.f);
      for (int j = 0; j < e.n_kt; ++j) {
        const uint32_t gj = tc + j;
        PF_T(0, mbar_wait(&s_full[x], gj & 1));  // CTA scope: an acquire.cluster wait invalidates L1 (CCTL.IVALL)
        tc_fence_after();
        const bool last_partial = j == e.n_kt - 1 && (j + 1) * kKT > e.n_keys;
        if (x == 0 && last_partial) {  // V rows past the keys (stale or another owner's bytes) -> 0
          char* sV = kvbase + (gj % ST) * kStage + kKBytes;
          const int first = e.n_keys - j * kKT;
          for (int i = tid; i < kKT * 8; i += 128)
            if ((i >> 3) >= first) *reinterpret_cast<uint4*>(sV + (i >> 3) * 128 + (i & 7) * 16) = make_uint4(0, 0, 0, 0);
        }
        const bool masked = (j * kKT + kKT - 1 > e.start + t0) || tail_rows;
        const int kb = j * kKT;
        {  // both 64-key halves loaded, one exact tile max and vote, then P handed over per half
          uint32_t ra[64], rb[64];
#pragma unroll
          for (int q = 0; q < 2; ++q) tmem_ld32_issue(tS + 32 * q, *reinterpret_cast<uint32_t(*)[32]>(ra + 32 * q));
#pragma unroll
          for (int q = 0; q < 2; ++q) tmem_ld32_issue(tS + 64 + 32 * q, *reinterpret_cast<uint32_t(*)[32]>(rb + 32 * q));
#pragma unroll
          for (int q = 0; q < 2; ++q) tmem_ld32_wait(*reinterpret_cast<uint32_t(*)[32]>(ra + 32 * q));
#pragma unroll
          for (int q = 0; q < 2; ++q) tmem_ld32_wait(*reinterpret_cast<uint32_t(*)[32]>(rb + 32 * q));
          if (masked) {
#pragma unroll
            for (int kk = 0; kk < 64; ++kk) {
              if (!(row_ok && kb + kk <= my_pos)) ra[kk] = __float_as_uint(-INFINITY);
              if (!(row_ok && kb + 64 + kk <= my_pos)) rb[kk] = __float_as_uint(-INFINITY);
            }
          }
          float mx4[4] = {__uint_as_float(ra[0]), __uint_as_float(ra[1]), __uint_as_float(rb[0]), __uint_as_float(rb[1])};
#pragma unroll
          for (int kk = 2; kk < 64; kk += 4) {
            mx4[0] = fmax3(mx4[0], __uint_as_float(ra[kk]), __uint_as_float(ra[kk + 1]));
            mx4[1] = fmax3(mx4[1], __uint_as_float(ra[kk + 2]), __uint_as_float(ra[kk + 3]));
            mx4[2] = fmax3(mx4[2], __uint_as_float(rb[kk]), __uint_as_float(rb[kk + 1]));
            mx4[3] = fmax3(mx4[3], __uint_as_float(rb[kk + 2]), __uint_as_float(rb[kk + 3]));
          }
          const float mt = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * c2;
          if (j == 0) {
            m = mt;
          } else {
            const bool need = mt > m + kRescale;
            if (__any_sync(0xffffffffu, need)) {  // raise the max: rescale O and l (no P of this tile yet)
              const float mn = need ? mt : m;
              const float alpha = need ? ex2(m - mn) : 1.f;
              m = mn;
              lsum.x *= alpha;
              lsum.y *= alpha;
              pp_rescale_o(tO, alpha);
            }
          }
          const float mu = m == -INFINITY ? 0.f : m;
          const float2 c2v = make_float2(c2, c2), nmv = make_float2(-mu, -mu);
          auto exps32 = [&](const uint32_t* r, uint32_t col) {  // 32 keys -> 16 packed P columns at col
            uint32_t pk[16];
            float2 v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float2 a = __ffma2_rn(make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])), c2v, nmv);
              if (i >= 16 - SKV_PP_EMU) v[i] = ex2_emu2(a);
              else v[i] = make_float2(ex2(a.x), ex2(a.y));
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) pk[i] = pack2<T>(v[i].x, v[i].y);
#pragma unroll
            for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
              for (int i = 0; i < w; ++i) v[i] = __fadd2_rn(v[i], v[i + w]);
            lsum = __fadd2_rn(lsum, v[0]);
            tmem_st16_nowait(tS + col, pk);
          };
          auto hand_over = [&](uint32_t bar, bool zeroed) {  // P columns stored so far -> MMA warp
            tmem_wait_st();
            if (zeroed) fence_async_smem();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (zeroed) mbar_arrive_cluster(bar);  // orders the V-row zeroing
              else mbar_arrive_cluster_relaxed(bar);
            }
          };
          exps32(ra, 0);
          hand_over(p_part_l, x == 0 && last_partial);
          exps32(ra + 32, 16);
          hand_over(p_part_l + 16, false);
          exps32(rb, 32);
          hand_over(p_part_l + 32, false);
          exps32(rb + 32, 48);
          hand_over(p_full_l, false);
        }
      }
      tc += e.n_kt;
#ifdef SKV_PF_TRACE
      pf_tiles += e.n_kt;
#endif
      const int nidx = next_item(k + 1);
      if (nidx >= 0) install_q(geo(nidx));  // all Q.K^T of this item retired
      PF_T(1, mbar_wait(&o_done[x], k & 1));
      tc_fence_after();
      const float lt = lsum.x + lsum.y;
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      char* dst = reinterpret_cast<char*>(e.g->out) +
                  (((size_t)e.q_off + (row_ok ? my_tok : 0)) * e.g->Hq + e.h * e.G + row % e.G) * (kD * 2);
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
      idx = nidx;
    }
  }
#ifdef SKV_PF_TRACE
  if (p.trace) {  // [cta][16]: loader kv_empty 0; mma q_full 1, kv_full 2, p_full A 3, B 4; softmax A
                  // (warp 0) s_full 5, o_done 6; B (warp 4) s_full 9, o_done 10; cycles 13, tiles 14
    unsigned long long* t = p.trace + (size_t)blockIdx.x * 16;
    if (warp == 9 && lane == 0) t[0] = pf_acc[0];
    if (warp == 8 && lane == 0) {
      for (int i = 0; i < 4; ++i) t[1 + i] = pf_acc[i];
      t[15] = pf_acc[4];
    }
    if (warp < 8 && (tid & 127) == 0)
      for (int i = 0; i < 2; ++i) t[5 + 4 * (warp >> 2) + i] = pf_acc[i];
    if (tid == 0) {
      t[13] = clock64() - pf_start;
      t[14] = pf_tiles;
    }
  }
#endif
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 8) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <typename T, int D>
void launch_prefill_d(const DataParams& p, cudaStream_t s) {
  static std::atomic<uint64_t> attr{0};
  ensure_smem_attr(prefill_kernel<T, D>, PF<D>::SMEM, attr);
  DataParams q = p;  // dense work-item numbering, group by group (prefill_item)
  long long items = 0;
  for (int i = 0; i < q.ngroups; ++i) {
    DataGroup& g = q.g[i];
    g.pf_base = (int)items;
    g.pf_npairs = ((p.max_q_len * g.G + kRows - 1) / kRows + 1) / 2;
    if (g.active) items += (long long)g.nreq * g.Hkv * g.pf_npairs;
  }
  if (items <= 0) return;
  const int clusters = (int)std::min<long long>(items, num_sms() / 2);
  cudaMemsetAsync(p.counter, 0, sizeof(int), s);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters, 1, 1);
  cfg.blockDim = dim3(kThreadsV3, 1, 1);
  cfg.dynamicSmemBytes = PF<D>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, prefill_kernel<T, D>, q, (int)items);
}

template <typename T>
void launch_prefill_pp(const DataParams& p, cudaStream_t s) {
  static std::atomic<uint64_t> attr{0};
  ensure_smem_attr(prefill_pp_kernel<T>, pp::kSmem, attr);
  DataParams q = p;
  long long items = 0;
  for (int i = 0; i < q.ngroups; ++i) {
    DataGroup& g = q.g[i];
    g.pf_base = (int)items;
    g.pf_npairs = (p.max_q_len * g.G + pp::kItemRows - 1) / pp::kItemRows;  // items per (request, kv head)
    if (g.active) items += (long long)g.nreq * g.Hkv * g.pf_npairs;
  }
  if (items <= 0) return;
  const int clusters = (int)std::min<long long>(items, num_sms() / 2);
  cudaMemsetAsync(p.counter, 0, sizeof(int), s);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * clusters, 1, 1);
  cfg.blockDim = dim3(pp::kThreads, 1, 1);
  cfg.dynamicSmemBytes = pp::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, prefill_pp_kernel<T>, q, (int)items);
}

// SKV_PREFILL_PP=0 selects the one-tile-per-CTA kernel for head dim 128 as well
bool use_pp() {
  static const bool on = [] {
    const char* e = getenv("SKV_PREFILL_PP");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace

// One launch per head dim present: the groups of other head dims are marked inactive in the
// copy each launch receives, so every (request, kv head) is computed exactly once.
void launch_prefill(const DataParams& p, cudaStream_t s) {
  if (p.nreq <= 0) return;
  for (int D : {128, 64, 256}) {
    bool any = false;
    DataParams q = p;
    for (int i = 0; i < q.ngroups; ++i) {
      if (q.g[i].D != D) q.g[i].active = 0;
      any |= q.g[i].active != 0 && q.g[i].D == D;
    }
    if (!any) continue;
    q.scale_log2 = 0.f;
    for (int i = 0; i < q.ngroups; ++i)
      if (q.g[i].D == D) q.scale_log2 = q.g[i].scale_log2;
    if (p.dtype == 0) {
      if (D == 64) launch_prefill_d<__half, 64>(q, s);
      else if (D == 128) use_pp() ? launch_prefill_pp<__half>(q, s) : launch_prefill_d<__half, 128>(q, s);
      else launch_prefill_d<__half, 256>(q, s);
    } else {
      if (D == 64) launch_prefill_d<__nv_bfloat16, 64>(q, s);
      else if (D == 128) use_pp() ? launch_prefill_pp<__nv_bfloat16>(q, s) : launch_prefill_d<__nv_bfloat16, 128>(q, s);
      else launch_prefill_d<__nv_bfloat16, 256>(q, s);
    }
  }
}

}  // namespace skv

// skv_attn.cu — data-path kernels of the unified KV pool (sm_100a).
//
// Layout: sub-slot s of merged block b of model m starts at
//   pool + b*merged_stride + s*native_stride[m];
// inside a native block: [phys_layer][kv_head][K|V][tpb=16][head_dim], so the K
// and V tiles of one (layer, head) are one contiguous 2*16*d*2 = 8 KiB run.
//
// Decode attention is HBM-bound (AI = Hq/Hkv flop/B): a persistent kernel, one
// CTA per SM, 8 independent warps; each warp owns a ring of STAGES 8 KiB smem
// tiles filled by cp.async.bulk (1-D TMA, mbarrier complete_tx) from
// block-table-indirected addresses, and computes softmax(q·Kᵀ)·V for all G query
// heads of a KV head from each tile (K/V read once per GQA group).  Work items
// (request, kv head, split) are fetched dynamically; the ring runs ahead across
// item boundaries; the work list is ordered by decreasing piece size (plan_kernel).
// Pieces of a cut (request, kv head) are merged (LSE combine) by the piece that
// finishes last, inside the same launch.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdlib>
#include <utility>

#include "skv_internal.h"

namespace skv {

namespace {

constexpr int kTpb = 16;                      // tokens per native block
constexpr int kTile = 8192;                   // ring slot: a d=128 K|V run, a d=64 run, or half a d=256 run
constexpr int kWsRow = 256;                   // floats per partial-output slot (any head_dim <= 256)
#ifndef SKV_DEC_WARPS
#define SKV_DEC_WARPS 8
#endif
#ifndef SKV_DEC_STAGES
#define SKV_DEC_STAGES 3
#endif
constexpr int kWarps = SKV_DEC_WARPS;    // independent warps per CTA (one CTA per SM)
constexpr int kStages = SKV_DEC_STAGES;  // 8 KiB tiles in flight per warp
constexpr int kRing = 16;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  while (!mbar_try_wait(bar, phase)) {
  }
}

// Programmatic dependent launch: kernels launched with the PDL attribute may start
// while the previous kernel on the stream drains; pdl_wait() blocks until that kernel
// has completed and its memory is visible, pdl_trigger() lets the next one launch.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename T>
struct Cvt;
template <>
struct Cvt<__half> {
  __device__ __forceinline__ static void to_f32(const uint4& r, float* f) {
    const __half2* h = reinterpret_cast<const __half2*>(&r);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 v = __half22float2(h[k]);
      f[2 * k] = v.x;
      f[2 * k + 1] = v.y;
    }
  }
  __device__ __forceinline__ static uint4 from_f32(const float* f) {
    uint4 r;
    __half2* h = reinterpret_cast<__half2*>(&r);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __floats2half2_rn(f[2 * k], f[2 * k + 1]);
    return r;
  }
  __device__ __forceinline__ static uint16_t one(float x) { return __half_as_ushort(__float2half_rn(x)); }
};
template <>
struct Cvt<__nv_bfloat16> {
  __device__ __forceinline__ static void to_f32(const uint4& r, float* f) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&r);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      f[2 * k] = __uint_as_float(w[k] << 16);
      f[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
    }
  }
  __device__ __forceinline__ static uint4 from_f32(const float* f) {
    uint4 r;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(f[2 * k], f[2 * k + 1]);
    return r;
  }
  __device__ __forceinline__ static uint16_t one(float x) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(x));
  }
};

// fp32 += 16-bit x 16-bit (one FHFMA: the half/bf16 operands are read straight from the
// packed register halves, no conversion instructions; the product is exact in fp32)
template <typename T>
struct MixFma;
template <>
struct MixFma<__half> {
  __device__ __forceinline__ static float f(float c, unsigned short a, unsigned short b) {
    asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(c) : "h"(a), "h"(b));
    return c;
  }
};
template <>
struct MixFma<__nv_bfloat16> {
  __device__ __forceinline__ static float f(float c, unsigned short a, unsigned short b) {
    asm("fma.rn.f32.bf16 %0, %1, %2, %0;" : "+f"(c) : "h"(a), "h"(b));
    return c;
  }
};

// Lane geometry of a 16-token K/V tile for head dim D.  A lane always holds 8 dims (16 B) of a
// token row: CPR = D/8 lanes cover one row, so a warp pass reads TPP = 32/CPR tokens and a
// tile takes NP = 16/TPP passes.  D = 64, 128: one ring unit = the native block's whole K|V
// run of this (layer, kv head) (64*D B: 4 / 8 KiB).  D = 256: the 16 KiB run is two ring
// units of 8 KiB (K, then V), each read by all 32 lanes, one token per pass.
template <int D>
struct Lanes {
  static constexpr int CPR = D / 8;
  static constexpr int TPP = CPR >= 32 ? 1 : 32 / CPR;
  static constexpr int NP = kTpb / TPP;
  static constexpr int ROW = 2 * D;                                    // bytes of one token row
  static constexpr int USH = D == 256 ? 1 : 0;                         // log2(ring units per block)
  static constexpr int UNIT = D == 256 ? kTpb * ROW : 2 * kTpb * ROW;  // bytes of one ring unit
  static_assert(D == 64 || D == 128 || D == 256, "head_dim 64, 128 or 256");
  static_assert(UNIT <= kTile, "a ring unit must fit a ring slot");
};

// Sum of W per-lane partials over 2W lanes (xor distances W .. 1), scattered so lane c ends
// up with the total of index (c >> 1) & (W - 1) (2W - 1 shuffles, not W * log2(2W)).
template <int W>
__device__ __forceinline__ float reduce_scatter(float (&v)[W], int lane) {
#pragma unroll
  for (int w = W; w >= 2; w >>= 1) {
    const bool hi = lane & w;
#pragma unroll
    for (int k = 0; k < w / 2; ++k) {
      const float send = hi ? v[k] : v[k + w / 2];
      const float keep = hi ? v[k + w / 2] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, w);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

// max over the warp (lanes c and c^1 hold the same value)
__device__ __forceinline__ float warp_max_pairs(float x) {
  x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 2));
  x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 4));
  x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 8));
  return fmaxf(x, __shfl_xor_sync(0xffffffffu, x, 16));
}

// q . k over this lane's 8 dims for G heads: packed fp32 FMA (FFMA2), 4 + 1 instructions
template <int G>
__device__ __forceinline__ void dot8(const float (&q)[G][8], const float (&kf)[8], float (&out)[G]) {
#pragma unroll
  for (int g = 0; g < G; ++g) {
    float2 a = __fmul2_rn(make_float2(q[g][0], q[g][1]), make_float2(kf[0], kf[1]));
#pragma unroll
    for (int j = 2; j < 8; j += 2) a = __ffma2_rn(make_float2(q[g][j], q[g][j + 1]), make_float2(kf[j], kf[j + 1]), a);
    out[g] = a.x + a.y;
  }
}

// o += p * v over this lane's 8 dims (FFMA2)
__device__ __forceinline__ void axpy8(float pt, const float (&vf)[8], float (&o)[8]) {
  const float2 pt2 = make_float2(pt, pt);
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    const float2 r = __ffma2_rn(pt2, make_float2(vf[j], vf[j + 1]), make_float2(o[j], o[j + 1]));
    o[j] = r.x;
    o[j + 1] = r.y;
  }
}

__device__ __forceinline__ void scale8(float alpha, float (&o)[8]) {
  const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    const float2 r = __fmul2_rn(make_float2(o[j], o[j + 1]), a2);
    o[j] = r.x;
    o[j + 1] = r.y;
  }
}

// One 16-token K/V tile (D = 64 / 128) for G query heads sharing a KV head (GQA path: K/V
// converted once, reused for the G heads).  Lane (c = lane % CPR, hf = lane / CPR) reads
// dims [8c, 8c+8) of tokens TPP*i + hf.
template <typename T, int G, int D, bool PARTIAL>
__device__ __forceinline__ void consume_tile(const char* tile, int lane, int valid,
                                             const float (&q)[G][8], float (&o)[G][8],
                                             float (&mx)[G], float (&l)[G]) {
  using LG = Lanes<D>;
  const int c = lane % LG::CPR, hf = lane / LG::CPR;
  float part[G][LG::NP];
#pragma unroll
  for (int i = 0; i < LG::NP; ++i) {
    const uint4 raw = *reinterpret_cast<const uint4*>(tile + (LG::TPP * i + hf) * LG::ROW + c * 16);
    float kf[8];
    Cvt<T>::to_f32(raw, kf);
    float d[G];
    dot8<G>(q, kf, d);
#pragma unroll
    for (int g = 0; g < G; ++g) part[g][i] = d[g];
  }
  const int tok = LG::TPP * ((c >> 1) & (LG::NP - 1)) + hf;
  float p[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    float s = reduce_scatter<LG::NP>(part[g], lane);
    if (tok >= valid) s = -INFINITY;
    const float mnew = fmaxf(mx[g], warp_max_pairs(s));
    const float alpha = exp2f(mx[g] - mnew);
    p[g] = exp2f(s - mnew);
    l[g] = l[g] * alpha + p[g];
    scale8(alpha, o[g]);
    mx[g] = mnew;
  }
  const char* vt = tile + kTpb * LG::ROW;
#pragma unroll
  for (int i = 0; i < LG::NP; ++i) {
    uint4 raw = *reinterpret_cast<const uint4*>(vt + (LG::TPP * i + hf) * LG::ROW + c * 16);
    if (PARTIAL && LG::TPP * i + hf >= valid) raw = make_uint4(0u, 0u, 0u, 0u);  // unwritten slots may hold NaN
    float vf[8];
    Cvt<T>::to_f32(raw, vf);
    const int src = hf * LG::CPR + 2 * i;
#pragma unroll
    for (int g = 0; g < G; ++g) axpy8(__shfl_sync(0xffffffffu, p[g], src), vf, o[g]);
  }
}

// Block-table row of (request handle, kv head) at the launch's layer: one row per request
// in the merged scheme, one per (request, layer, kv head) in the split scheme.
__device__ __forceinline__ const int2* table_row(const DataParams& p, int handle, int head) {
  return p.split_L ? p.req_table + (((size_t)handle * p.split_L + p.layer) * p.split_H + head) * p.cap
                   : p.req_table + (size_t)handle * p.cap;
}

// G = 1 (MHA) variant of consume_tile: q stays in 16-bit (qraw, this lane's 8 raw dims) and
// both dot products run as mixed-precision FMAs (fp32 accumulate, 16-bit operands), so
// neither K nor V is converted; P is rounded to the 16-bit type for P.V, as the tensor-core
// prefill does.  About 30 % fewer instructions per tile than the converting path.
template <typename T, int D, bool PARTIAL>
__device__ __forceinline__ void consume_tile_mha(const char* tile, int lane, int valid, const uint4& qraw,
                                                 float scale_log2, float (&o)[8], float& mx, float& l) {
  using LG = Lanes<D>;
  const int c = lane % LG::CPR, hf = lane / LG::CPR;
  const unsigned short* qh = reinterpret_cast<const unsigned short*>(&qraw);
  float part[LG::NP];
#pragma unroll
  for (int i = 0; i < LG::NP; ++i) {
    const uint4 raw = *reinterpret_cast<const uint4*>(tile + (LG::TPP * i + hf) * LG::ROW + c * 16);
    const unsigned short* kh = reinterpret_cast<const unsigned short*>(&raw);
    float a = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) a = MixFma<T>::f(a, qh[j], kh[j]);
    part[i] = a;
  }
  const int tok = LG::TPP * ((c >> 1) & (LG::NP - 1)) + hf;
  float sc = reduce_scatter<LG::NP>(part, lane) * scale_log2;
  if (tok >= valid) sc = -INFINITY;
  const float mnew = fmaxf(mx, warp_max_pairs(sc));
  const float alpha = exp2f(mx - mnew);
  const float pr = exp2f(sc - mnew);
  l = l * alpha + pr;
  scale8(alpha, o);
  mx = mnew;
  const char* vt = tile + kTpb * LG::ROW;
#pragma unroll
  for (int i = 0; i < LG::NP; ++i) {
    uint4 raw = *reinterpret_cast<const uint4*>(vt + (LG::TPP * i + hf) * LG::ROW + c * 16);
    if (PARTIAL && LG::TPP * i + hf >= valid) raw = make_uint4(0u, 0u, 0u, 0u);  // unwritten slots may hold NaN
    const unsigned short* vh = reinterpret_cast<const unsigned short*>(&raw);
    const unsigned short ph = Cvt<T>::one(__shfl_sync(0xffffffffu, pr, hf * LG::CPR + 2 * i));
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = MixFma<T>::f(o[j], ph, vh[j]);
  }
}

// D = 256, K unit (16 tokens x 512 B, one token per pass, lane = dims [8*lane, 8*lane+8)):
// scores of tokens 0-7 and 8-15 as two reduce-scatters of 8 values over 16 lanes plus the
// other 16 lanes' dims (xor 16), so a lane holds tokens (lane>>1)&7 and 8 + that; then the
// online-softmax update.  p0 / p1 are the lane's two probabilities.
template <typename T, int G>
__device__ __forceinline__ void scores_256(const char* kt, int lane, int valid, const float (&q)[G][8],
                                           float (&o)[G][8], float (&mx)[G], float (&l)[G], float (&p0)[G],
                                           float (&p1)[G]) {
  float s[2][G];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float part[G][8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 raw = *reinterpret_cast<const uint4*>(kt + (8 * h + i) * 512 + lane * 16);
      float kf[8];
      Cvt<T>::to_f32(raw, kf);
      float d[G];
      dot8<G>(q, kf, d);
#pragma unroll
      for (int g = 0; g < G; ++g) part[g][i] = d[g];
    }
    const int tok = 8 * h + ((lane >> 1) & 7);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float x = reduce_scatter<8>(part[g], lane);
      x += __shfl_xor_sync(0xffffffffu, x, 16);
      s[h][g] = tok >= valid ? -INFINITY : x;
    }
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const float mnew = fmaxf(mx[g], warp_max_pairs(fmaxf(s[0][g], s[1][g])));
    const float alpha = exp2f(mx[g] - mnew);
    p0[g] = exp2f(s[0][g] - mnew);
    p1[g] = exp2f(s[1][g] - mnew);
    l[g] = l[g] * alpha + (p0[g] + p1[g]);
    scale8(alpha, o[g]);
    mx[g] = mnew;
  }
}

// D = 256, V unit: o += p . V; token i's probability sits in lane 2*(i&7) (p0 for i < 8, p1 after)
template <typename T, int G, bool PARTIAL>
__device__ __forceinline__ void pv_256(const char* vt, int lane, int valid, const float (&p0)[G],
                                       const float (&p1)[G], float (&o)[G][8]) {
#pragma unroll
  for (int i = 0; i < kTpb; ++i) {
    uint4 raw = *reinterpret_cast<const uint4*>(vt + i * 512 + lane * 16);
    if (PARTIAL && i >= valid) raw = make_uint4(0u, 0u, 0u, 0u);  // unwritten slots may hold NaN
    float vf[8];
    Cvt<T>::to_f32(raw, vf);
#pragma unroll
    for (int g = 0; g < G; ++g) axpy8(__shfl_sync(0xffffffffu, i < 8 ? p0[g] : p1[g], 2 * (i & 7)), vf, o[g]);
  }
}

// D = 256 MHA variants (16-bit q, mixed-precision FMAs, P rounded to 16 bits for P.V)
template <typename T>
__device__ __forceinline__ void scores_256_mha(const char* kt, int lane, int valid, const uint4& qraw,
                                               float scale_log2, float (&o)[8], float& mx, float& l, float& p0,
                                               float& p1) {
  const unsigned short* qh = reinterpret_cast<const unsigned short*>(&qraw);
  float s[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float part[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint4 raw = *reinterpret_cast<const uint4*>(kt + (8 * h + i) * 512 + lane * 16);
      const unsigned short* kh = reinterpret_cast<const unsigned short*>(&raw);
      float a = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) a = MixFma<T>::f(a, qh[j], kh[j]);
      part[i] = a;
    }
    float x = reduce_scatter<8>(part, lane);
    x = (x + __shfl_xor_sync(0xffffffffu, x, 16)) * scale_log2;
    s[h] = 8 * h + ((lane >> 1) & 7) >= valid ? -INFINITY : x;
  }
  const float mnew = fmaxf(mx, warp_max_pairs(fmaxf(s[0], s[1])));
  const float alpha = exp2f(mx - mnew);
  p0 = exp2f(s[0] - mnew);
  p1 = exp2f(s[1] - mnew);
  l = l * alpha + (p0 + p1);
  scale8(alpha, o);
  mx = mnew;
}

template <typename T, bool PARTIAL>
__device__ __forceinline__ void pv_256_mha(const char* vt, int lane, int valid, float p0, float p1, float (&o)[8]) {
#pragma unroll
  for (int i = 0; i < kTpb; ++i) {
    uint4 raw = *reinterpret_cast<const uint4*>(vt + i * 512 + lane * 16);
    if (PARTIAL && i >= valid) raw = make_uint4(0u, 0u, 0u, 0u);  // unwritten slots may hold NaN
    const unsigned short* vh = reinterpret_cast<const unsigned short*>(&raw);
    const unsigned short ph = Cvt<T>::one(__shfl_sync(0xffffffffu, i < 8 ? p0 : p1, 2 * (i & 7)));
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = MixFma<T>::f(o[j], ph, vh[j]);
  }
}

// Per-warp producer: walks the same item sequence as the consumer, kStages ring units ahead.
struct Producer {
  int idx;         // current item, -1 before the first
  int blk, bend;   // next ring unit to issue / end (unit = native block << ush, + K/V half)
  int ush;         // log2(ring units per native block) of the current item (1 for D = 256)
  int ubytes;      // bytes of one ring unit of the current item
  int cbase;       // first native block of the cached table chunk (-1 = none)
  int2 tc;         // lane-held table chunk entry
  const int2* row;
  const char* base;  // pool + layer/head offset of the current item
  long long nstride;
  int done;
  int pushed, popped;  // ring counters
  uint32_t issued, consumed;
};

struct WarpCtx {
  char* tiles;
  uint64_t* bars;
  int* ring;
  int lane;
  int n_items;
  uint64_t policy;
};

__device__ __forceinline__ bool produce_one(const DataParams& p, Producer& P, const WarpCtx& w) {
  while (!P.done && P.blk >= P.bend) {
    if (P.pushed - P.popped >= kRing) return false;
    int idx = 0;
    if (w.lane == 0) idx = atomicAdd(p.counter, 1);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= w.n_items) {
      P.done = 1;
      break;
    }
    const int4 it = p.items[idx];
    const DataGroup& g = p.g[it.y >> 16];
    if (!g.active) continue;
    if (w.lane == 0) w.ring[P.pushed % kRing] = idx;
    __syncwarp();
    P.pushed++;
    P.idx = idx;
    P.ush = g.D == 256 ? 1 : 0;
    P.ubytes = g.D == 256 ? kTpb * 512 : 64 * g.D;
    P.blk = (it.z / kTpb) << P.ush;
    P.bend = ((it.w + kTpb - 1) / kTpb) << P.ush;
    P.row = table_row(p, p.handles[it.x], it.y & 0xffff);
    P.base = p.pool + g.layer_off + (long long)(it.y & 0xffff) * g.head_stride;
    P.nstride = g.native_stride;
    P.cbase = -1;
  }
  if (P.done || P.blk >= P.bend) return false;
  const int blk = P.blk >> P.ush;
  if (P.cbase < 0 || blk - P.cbase >= 32) {
    P.cbase = blk;
    const int b = blk + w.lane;
    P.tc = b < (P.bend >> P.ush) ? P.row[b] : make_int2(0, 0);
  }
  const int rel = blk - P.cbase;
  const int bx = __shfl_sync(0xffffffffu, P.tc.x, rel);
  const int by = __shfl_sync(0xffffffffu, P.tc.y, rel);
  const int stage = P.issued % kStages;
  if (w.lane == 0) {
    const char* src = P.base + (long long)bx * p.merged_stride + (long long)by * P.nstride + (P.blk & P.ush) * (kTpb * 512);
    mbar_expect_tx(&w.bars[stage], P.ubytes);
    bulk_g2s(w.tiles + stage * kTile, src, P.ubytes, &w.bars[stage], w.policy);
  }
  P.issued++;
  P.blk++;
  return true;
}

__device__ __forceinline__ void fill(const DataParams& p, Producer& P, const WarpCtx& w) {
  while (P.issued - P.consumed < (uint32_t)kStages) {
    if (!produce_one(p, P, w)) break;
  }
}

// Waits for the next ring unit of the current item; returns its shared-memory tile.
__device__ __forceinline__ char* next_unit(const DataParams& p, Producer& P, const WarpCtx& w) {
  if (P.issued == P.consumed) fill(p, P, w);
  const int stage = P.consumed % kStages;
  mbar_wait(&w.bars[stage], (P.consumed / kStages) & 1u);
  return w.tiles + stage * kTile;
}

__device__ __forceinline__ void release_unit(const DataParams& p, Producer& P, const WarpCtx& w) {
  __syncwarp();
  P.consumed++;
  fill(p, P, w);
}

// Fused append (n_new == 1): writes the step's new K (kv 0) and/or V (kv 1) row of token apos
// into the pool and patches it into the staged unit, which holds the K|V run (D <= 128) or just
// the K or V half (D = 256).  16 B per lane, as append_kernel.
template <int D>
__device__ __forceinline__ void patch_new_token(const DataParams& p, const DataGroup& g, int handle, int head, int rl,
                                                int b, int apos, char* unit, int kv_first, int kv_last, int lane) {
  using LG = Lanes<D>;
  const int2 e = table_row(p, handle, head)[b];
  char* run = p.pool + g.layer_off + (long long)head * g.head_stride + (long long)e.x * p.merged_stride +
              (long long)e.y * g.native_stride;
  for (int ch = lane + kv_first * LG::CPR; ch < (kv_last + 1) * LG::CPR; ch += 32) {
    const int kv = ch / LG::CPR, c = ch % LG::CPR;
    const uint4 val = *reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(kv ? g.v : g.k) +
                                                      ((size_t)rl * g.Hkv + head) * LG::ROW + c * 16);
    const int off = (apos % kTpb) * LG::ROW + c * 16;
    *reinterpret_cast<uint4*>(run + kv * (kTpb * LG::ROW) + off) = val;
    *reinterpret_cast<uint4*>(unit + (D == 256 ? 0 : kv * (kTpb * LG::ROW)) + off) = val;
  }
  // the slot is refilled by TMA (async proxy) later: order this generic write first
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
}

template <typename T, int G, int D>
__device__ __forceinline__ void process_item(const DataParams& p, Producer& P, const WarpCtx& w,
                                             const int4 it, int idx) {
  using LG = Lanes<D>;
  const int lane = w.lane, c = lane % LG::CPR, hf = lane / LG::CPR;
  const int grp = it.y >> 16, head = it.y & 0xffff;
  const DataGroup& g = p.g[grp];
  const int rl = it.x - g.req_begin;
  float q[G][8], o[G][8], mx[G], l[G];
  uint4 qraw = make_uint4(0u, 0u, 0u, 0u);  // G = 1: this lane's 8 raw query dims
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    const T* qp = reinterpret_cast<const T*>(g.q) + ((size_t)rl * g.Hq + head * G + gg) * D;
    const uint4 raw = *reinterpret_cast<const uint4*>(qp + c * 8);
    if (G == 1) qraw = raw;
    Cvt<T>::to_f32(raw, q[gg]);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      q[gg][j] *= g.scale_log2;
      o[gg][j] = 0.f;
    }
    mx[gg] = -INFINITY;
    l[gg] = 0.f;
  }
  // fused append (n_new == 1): the item holding position ctx-1 writes the step's new K/V
  // token into the pool and patches it into the staged unit(s) before attending
  int apos = -1;
  const int handle = p.handles[it.x];
  if (p.n_new == 1 && g.k != nullptr) {
    const int pos = p.req_tokens[handle] - 1;
    if (pos >= it.z && pos < it.w) apos = pos;
  }
  const int b0 = it.z / kTpb, b1 = (it.w + kTpb - 1) / kTpb;
  for (int b = b0; b < b1; ++b) {
    const int valid = min(kTpb, it.w - b * kTpb);
    const bool patch = apos >= 0 && b == apos / kTpb;
    char* unit = next_unit(p, P, w);
    if constexpr (D != 256) {
      if (patch) patch_new_token<D>(p, g, handle, head, rl, b, apos, unit, 0, 1, lane);
      if constexpr (G == 1) {
        if (valid == kTpb) consume_tile_mha<T, D, false>(unit, lane, valid, qraw, g.scale_log2, o[0], mx[0], l[0]);
        else consume_tile_mha<T, D, true>(unit, lane, valid, qraw, g.scale_log2, o[0], mx[0], l[0]);
      } else {
        if (valid == kTpb) consume_tile<T, G, D, false>(unit, lane, valid, q, o, mx, l);
        else consume_tile<T, G, D, true>(unit, lane, valid, q, o, mx, l);
      }
      release_unit(p, P, w);
    } else {
      float p0[G], p1[G];
      if (patch) patch_new_token<D>(p, g, handle, head, rl, b, apos, unit, 0, 0, lane);
      if constexpr (G == 1) scores_256_mha<T>(unit, lane, valid, qraw, g.scale_log2, o[0], mx[0], l[0], p0[0], p1[0]);
      else scores_256<T, G>(unit, lane, valid, q, o, mx, l, p0, p1);
      release_unit(p, P, w);
      unit = next_unit(p, P, w);
      if (patch) patch_new_token<D>(p, g, handle, head, rl, b, apos, unit, 1, 1, lane);
      if constexpr (G == 1) {
        if (valid == kTpb) pv_256_mha<T, false>(unit, lane, valid, p0[0], p1[0], o[0]);
        else pv_256_mha<T, true>(unit, lane, valid, p0[0], p1[0], o[0]);
      } else {
        if (valid == kTpb) pv_256<T, G, false>(unit, lane, valid, p0, p1, o);
        else pv_256<T, G, true>(unit, lane, valid, p0, p1, o);
      }
      release_unit(p, P, w);
    }
  }
  // finalize: l over the lanes holding distinct tokens, o over the TPP token lanes
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    float s = l[gg];
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 8);
    if (D != 256) s += __shfl_xor_sync(0xffffffffu, s, 16);  // D = 256: lanes c, c^16 hold the same tokens
    l[gg] = s;
#pragma unroll
    for (int x = LG::CPR; x < 32; x <<= 1)
#pragma unroll
      for (int j = 0; j < 8; ++j) o[gg][j] += __shfl_xor_sync(0xffffffffu, o[gg][j], x);
  }
  const int4 x = p.itemx[idx];  // {pieces, partial-slot base, piece, arrival index}
  const int ns = x.x;
  if (ns <= 1) {
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      if (hf == 0) {
        const float inv = l[gg] > 0.f ? 1.f / l[gg] : 0.f;
        float r[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = o[gg][j] * inv;
        T* op = reinterpret_cast<T*>(g.out) + ((size_t)rl * g.Hq + head * G + gg) * D + c * 8;
        *reinterpret_cast<uint4*>(op) = Cvt<T>::from_f32(r);
      }
    }
    return;
  }
  // piece of a cut (request, kv head): publish (m, l, o); the piece that finishes last
  // merges all of them (LSE combine) and writes the output, inside this launch
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    const size_t slot = (size_t)x.y + (size_t)x.z * G + gg;
    if (hf == 0) {
      float4* dst = reinterpret_cast<float4*>(p.ws_o + slot * kWsRow + c * 8);
      __stcg(dst, make_float4(o[gg][0], o[gg][1], o[gg][2], o[gg][3]));
      __stcg(dst + 1, make_float4(o[gg][4], o[gg][5], o[gg][6], o[gg][7]));
    }
    if (lane == 0) __stcg(p.ws_ml + slot, make_float2(mx[gg], l[gg]));
  }
  __syncwarp();
  int last = 0;
  if (lane == 0) {
    __threadfence();
    last = atomicAdd(p.arrive + x.w, 1) == ns - 1;
    if (last) __threadfence();
  }
  last = __shfl_sync(0xffffffffu, last, 0);
  if (!last) return;
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    float M = -INFINITY;
    for (int s = lane; s < ns; s += 32) M = fmaxf(M, __ldcg(p.ws_ml + x.y + (size_t)s * G + gg).x);
#pragma unroll
    for (int o2 = 16; o2 >= 1; o2 >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o2));
    // lane (c, hf): dims [8c, 8c+8) over pieces hf, hf + TPP, ...
    float L = 0.f, acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
#pragma unroll 2
    for (int s = hf; s < ns; s += LG::TPP) {
      const size_t slot = (size_t)x.y + (size_t)s * G + gg;
      const float2 ml = __ldcg(p.ws_ml + slot);
      const float4* src = reinterpret_cast<const float4*>(p.ws_o + slot * kWsRow + c * 8);
      const float4 a = __ldcg(src), bb = __ldcg(src + 1);
      const float wgt = ml.y > 0.f ? exp2f(ml.x - M) : 0.f;
      L += ml.y * wgt;
      acc[0] += a.x * wgt;
      acc[1] += a.y * wgt;
      acc[2] += a.z * wgt;
      acc[3] += a.w * wgt;
      acc[4] += bb.x * wgt;
      acc[5] += bb.y * wgt;
      acc[6] += bb.z * wgt;
      acc[7] += bb.w * wgt;
    }
#pragma unroll
    for (int xo = LG::CPR; xo < 32; xo <<= 1) {
      L += __shfl_xor_sync(0xffffffffu, L, xo);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], xo);
    }
    if (hf == 0) {
      const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] *= inv;
      T* op = reinterpret_cast<T*>(g.out) + ((size_t)rl * g.Hq + head * G + gg) * D + c * 8;
      *reinterpret_cast<uint4*>(op) = Cvt<T>::from_f32(acc);
    }
  }
  if (lane == 0) p.arrive[x.w] = 0;  // ready for the launch after next (same counter set)
}

template <typename T, int MAXG, int D>
__device__ __forceinline__ void run_item(const DataParams& p, Producer& P, const WarpCtx& w, const int4 it, int idx,
                                         int G) {
  if (G == 1) process_item<T, 1, D>(p, P, w, it, idx);
  else if (MAXG >= 2 && G == 2) process_item<T, (MAXG >= 2 ? 2 : 1), D>(p, P, w, it, idx);
  else if (MAXG >= 4 && G == 4) process_item<T, (MAXG >= 4 ? 4 : 1), D>(p, P, w, it, idx);
  else if (MAXG >= 8 && G == 8) process_item<T, (MAXG >= 8 ? 8 : 1), D>(p, P, w, it, idx);
}

// DMASK: head dims present in the launch (1: 64, 2: 128, 4: 256); a d = 128-only launch
// compiles just that path.
template <typename T, int MAXG, int DMASK>
__global__ void __launch_bounds__(kWarps * 32, 1) decode_kernel(const __grid_constant__ DataParams p) {
  extern __shared__ __align__(128) char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned long long t_start = p.trace ? global_ns() : 0ull;
  unsigned long long t_wait = 0ull;
  int n_done = 0;
  WarpCtx w;
  w.tiles = smem + wid * kStages * kTile;
  w.bars = reinterpret_cast<uint64_t*>(smem + kWarps * kStages * kTile) + wid * kStages;
  w.ring = reinterpret_cast<int*>(smem + kWarps * kStages * kTile + kWarps * kStages * 8) + wid * kRing;
  w.lane = lane;
  w.policy = evict_first_policy();
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(&w.bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  Producer P;
  P.idx = -1;
  P.blk = P.bend = 0;
  P.ush = 0;
  P.ubytes = kTile;
  P.cbase = -1;
  P.tc = make_int2(0, 0);
  P.row = nullptr;
  P.base = nullptr;
  P.nstride = 0;
  P.done = 0;
  P.pushed = P.popped = 0;
  P.issued = P.consumed = 0;
  // Everything before pdl_wait() overlaps the previous launch's tail.  With prefetch the
  // first kStages K/V units of this warp are already in flight: the cache bytes of this
  // layer do not depend on the previous launch (see DataParams::prefetch).
  if (p.prefetch) {
    w.n_items = *p.n_items;
    fill(p, P, w);
  }
  pdl_wait();
  if (p.trace) t_wait = global_ns();
  // the next launch may queue its CTAs now (they become resident as this grid's CTAs exit)
  pdl_trigger();
  if (!p.prefetch) w.n_items = *p.n_items;
  for (;;) {
    fill(p, P, w);
    if (P.pushed == P.popped) {
      // ring empty: either finished or only zero-block items were skipped
      if (P.done) break;
      continue;
    }
    const int idx = w.ring[P.popped % kRing];
    P.popped++;
    ++n_done;
    const int4 it = p.items[idx];
    const DataGroup& gi = p.g[it.y >> 16];
    const int G = gi.G;
    if constexpr ((DMASK & 2) != 0) {
      if (DMASK == 2 || gi.D == 128) {
        run_item<T, MAXG, 128>(p, P, w, it, idx, G);
        continue;
      }
    }
    if constexpr ((DMASK & 1) != 0) {
      if (gi.D == 64) {
        run_item<T, MAXG, 64>(p, P, w, it, idx, G);
        continue;
      }
    }
    if constexpr ((DMASK & 4) != 0) {
      if (gi.D == 256) run_item<T, MAXG, 256>(p, P, w, it, idx, G);
    }
  }
  if (p.trace && lane == 0) {
    unsigned long long* t = p.trace + ((size_t)blockIdx.x * kWarps + wid) * 4;
    t[0] = t_start;
    t[1] = t_wait;
    t[2] = global_ns();
    t[3] = ((unsigned long long)P.consumed << 32) | (unsigned)n_done;
  }
  // the last CTA to finish resets the work counter for the next launch (no memset node)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(p.counter + 1, 1) == (int)gridDim.x - 1) {
      p.counter[0] = 0;
      p.counter[1] = 0;
      __threadfence();
    }
  }
}

// Work list for the dynamically scheduled decode.  A (request, kv head) of nt K/V
// tiles is one piece, or — for the last n_cut (request, kv head)s of the batch — a
// leading part plus two trailing pieces of ~3/16 and ~1/16 of a base piece.  The list
// holds all leading pieces, then all middle ones, then all small ones; warps fetch in
// list order, so the launch ends on small pieces: its tail (warps idling while others
// finish) stays short even though per-warp HBM bandwidth is uneven, while the piece
// count (per-piece q loads, partial writes, merges) grows only by ~2*n_cut.  Leading
// parts longer than split_tokens are cut further into balanced chunks.  Pieces of a cut
// (request, kv head) are merged in-kernel by the piece that finishes last.
struct PieceShape {
  int s1, s2, s3;  // leading / middle / small tiles
  int k1, c1;      // leading chunks and their size
  int ns;          // pieces
};
__device__ __forceinline__ PieceShape piece_shape(int nt, int maxt, bool cut) {
  PieceShape q;
  const int base = min(nt, maxt);
  if (cut && nt >= 4) {
    q.s3 = max(1, base / 16);
    q.s2 = max(1, (3 * base) / 16);
  } else {
    q.s2 = q.s3 = 0;
  }
  q.s1 = nt - q.s2 - q.s3;
  q.k1 = q.s1 > 0 ? (q.s1 + maxt - 1) / maxt : 1;  // empty context: one (empty) piece -> zeros
  q.c1 = q.s1 > 0 ? (q.s1 + q.k1 - 1) / q.k1 : 0;
  q.ns = q.k1 + (q.s2 > 0) + (q.s3 > 0);
  return q;
}

__global__ void __launch_bounds__(1024) plan_kernel(DataParams p) {
  __shared__ int sm_warp[33];
  __shared__ int carry[5];  // (request, kv head)s, leading, middle, small pieces, partial slots
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  pdl_wait();  // the previous decode may still be reading the work list
  pdl_trigger();
  if (tid < 5) carry[tid] = 0;
  __syncthreads();
  auto scan = [&](int v, int* total) {
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) sm_warp[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const int x = sm_warp[lane];
      int xi = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, xi, o);
        if (lane >= o) xi += t;
      }
      sm_warp[lane] = xi - x;
      if (lane == 31) sm_warp[32] = xi;
    }
    __syncthreads();
    const int ex = sm_warp[wid] + incl - v;
    *total = sm_warp[32];
    __syncthreads();
    return ex;
  };
  // Every group is planned (the plan is reused across layers); pieces of groups inactive
  // at a layer are skipped when fetched.
  const int n = p.nreq, maxt = max(1, p.split_tokens / kTpb);
  int* rh_off = p.rscr;           // (request, kv head) offset of request r
  int* o1 = p.rscr + n;           // leading-piece offset
  int* o2 = p.rscr + 2 * n;       // middle-piece offset
  int* o3 = p.rscr + 3 * n;       // small-piece offset
  int* os = p.rscr + 4 * n;       // partial-slot offset
  // pass 0: (request, kv head) offsets
  for (int r0 = 0; r0 < n; r0 += 1024) {
    const int r = r0 + tid;
    int t;
    const int e = scan(r < n ? p.g[p.req_group[r]].Hkv : 0, &t);
    if (r < n) rh_off[r] = carry[0] + e;
    __syncthreads();
    if (tid == 0) carry[0] += t;
    __syncthreads();
  }
  const int NRH = carry[0];
  const int first_cut = NRH - min(NRH, p.n_cut);
  // pass A: piece and slot offsets per request
  for (int r0 = 0; r0 < n; r0 += 1024) {
    const int r = r0 + tid;
    int v1 = 0, v2 = 0, v3 = 0, vs = 0;
    if (r < n) {
      const DataGroup& g = p.g[p.req_group[r]];
      const int nt = (p.req_tokens[p.handles[r]] + kTpb - 1) / kTpb;
      const int nc = min(g.Hkv, max(0, rh_off[r] + g.Hkv - first_cut));  // its last nc heads are cut
      const PieceShape u = piece_shape(nt, maxt, false), c = piece_shape(nt, maxt, true);
      v1 = (g.Hkv - nc) * u.k1 + nc * c.k1;
      v2 = c.s2 > 0 ? nc : 0;
      v3 = c.s3 > 0 ? nc : 0;
      vs = (u.ns > 1 ? (g.Hkv - nc) * u.ns : 0) * g.G + (c.ns > 1 ? nc * c.ns : 0) * g.G;
    }
    int t1, t2, t3, ts;
    const int e1 = scan(v1, &t1), e2 = scan(v2, &t2), e3 = scan(v3, &t3), es = scan(vs, &ts);
    if (r < n) {
      o1[r] = carry[1] + e1;
      o2[r] = carry[2] + e2;
      o3[r] = carry[3] + e3;
      os[r] = carry[4] + es;
    }
    __syncthreads();
    if (tid == 0) {
      carry[1] += t1;
      carry[2] += t2;
      carry[3] += t3;
      carry[4] += ts;
    }
    __syncthreads();
  }
  const int N1 = carry[1], N2 = carry[2];
  // Capacity guard: a CUDA graph replays this plan with the token counts of the replay, which
  // may need more pieces than the host sized the buffers for at capture time.  Never write
  // past them: flag the pool (skv_synchronize reports it) and run an empty launch instead.
  if ((long long)N1 + N2 + carry[3] > p.items_cap || carry[4] > p.slots_cap) {
    if (tid == 0) {
      *p.n_items = 0;
      p.counter[0] = 0;
      p.counter[1] = 0;
      if (p.status) atomicExch(p.status, 3);
    }
    return;
  }
  // pass B: one warp per request, lanes over its kv heads
  for (int r = wid; r < n; r += 32) {
    const int grp = p.req_group[r];
    const DataGroup& g = p.g[grp];
    const int ctx = p.req_tokens[p.handles[r]];
    const int nt = (ctx + kTpb - 1) / kTpb;
    const int nc = min(g.Hkv, max(0, rh_off[r] + g.Hkv - first_cut));
    const int hcut = g.Hkv - nc;  // heads >= hcut are cut
    const PieceShape u = piece_shape(nt, maxt, false), c = piece_shape(nt, maxt, true);
    for (int h = lane; h < g.Hkv; h += 32) {
      const bool cut = h >= hcut;
      const PieceShape& q = cut ? c : u;
      const int i1 = o1[r] + (cut ? hcut * u.k1 + (h - hcut) * c.k1 : h * u.k1);  // also the arrival index
      const int sb = os[r] + (cut ? (u.ns > 1 ? hcut * u.ns : 0) + (h - hcut) * c.ns : h * u.ns) * g.G;
      const int hy = (grp << 16) | h;
      for (int j = 0; j < q.k1; ++j) {
        const int tb = j * q.c1, te = min(q.s1, tb + q.c1);
        p.items[i1 + j] = make_int4(r, hy, tb * kTpb, min(ctx, te * kTpb));
        p.itemx[i1 + j] = make_int4(q.ns, sb, j, i1);
      }
      if (q.s2 > 0) {
        const int i = N1 + o2[r] + (h - hcut);
        p.items[i] = make_int4(r, hy, q.s1 * kTpb, min(ctx, (q.s1 + q.s2) * kTpb));
        p.itemx[i] = make_int4(q.ns, sb, q.k1, i1);
      }
      if (q.s3 > 0) {
        const int i = N1 + N2 + o3[r] + (h - hcut);
        p.items[i] = make_int4(r, hy, (q.s1 + q.s2) * kTpb, ctx);
        p.itemx[i] = make_int4(q.ns, sb, q.k1 + (q.s2 > 0), i1);
      }
    }
  }
  if (tid == 0) {
    *p.n_items = N1 + N2 + carry[3];
    p.counter[0] = 0;  // this launch's counter set (each decode launch also self-resets its set)
    p.counter[1] = 0;
  }
}

// KV append: one warp per (request, new token, kv head); lanes 0-15 move the K row
// (256 B), lanes 16-31 the V row, 16 B each.
__global__ void append_kernel(const __grid_constant__ DataParams p) {
  pdl_wait();
  pdl_trigger();
  const int r = blockIdx.y;
  const DataGroup& g = p.g[p.req_group[r]];
  if (!g.active) return;
  const int lane = threadIdx.x & 31;
  const int wglob = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int n_new = p.q_lens ? p.q_lens[r] : p.n_new;  // ragged: this request's own count
  const int total = n_new * g.Hkv;
  if (wglob >= total) return;
  const int i = wglob / g.Hkv, h = wglob % g.Hkv;
  const int handle = p.handles[r];
  const int pos = p.req_tokens[handle] - n_new + i;
  if (pos < 0) return;
  const int2 e = table_row(p, handle, h)[pos / kTpb];
  const int row = 2 * g.D, cpr = g.D / 8;  // bytes of a token row, 16-B chunks per row
  char* run = p.pool + (long long)e.x * p.merged_stride + (long long)e.y * g.native_stride + g.layer_off +
              (long long)h * g.head_stride + (pos % kTpb) * row;
  const int rl = r - g.req_begin;
  const size_t first = p.q_offs ? (size_t)p.q_offs[r] : (size_t)rl * p.n_new;  // request's first packed token
  const size_t src_row = ((first + i) * g.Hkv + h) * row;
  for (int ch = lane; ch < 2 * cpr; ch += 32) {  // K row then V row, 16 B per lane
    const int kv = ch >= cpr, c = ch - kv * cpr;
    const char* src = reinterpret_cast<const char*>(kv ? g.v : g.k) + src_row + c * 16;
    *reinterpret_cast<uint4*>(run + kv * (kTpb * row) + c * 16) = *reinterpret_cast<const uint4*>(src);
  }
}

__device__ __forceinline__ float synth_u(unsigned long long seed, unsigned long long i) {
  unsigned long long z = seed + (i + 1ull) * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  z ^= z >> 31;
  return (float)(z >> 40) * (1.0f / 16777216.0f);
}

template <typename T>
__global__ void synth_kernel(uint4* pool, size_t n16, unsigned long long seed, float amp) {
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n16; v += (size_t)gridDim.x * blockDim.x) {
    float f[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = (2.f * synth_u(seed, v * 8 + k) - 1.f) * amp;
    pool[v] = Cvt<T>::from_f32(f);
  }
}

bool pdl_enabled() {
  static const bool on = [] {  // environment read once (thread-safe static init)
    const char* e = getenv("SKV_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

// Launch with the programmatic-stream-serialization attribute (see pdl_wait).
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <typename T, int MAXG, int DMASK>
void launch_decode_t(const DataParams& p, int grid, cudaStream_t s) {
  const int smem = kWarps * kStages * kTile + kWarps * kStages * 8 + kWarps * kRing * 4;
  static std::atomic<uint64_t> attr{0};
  ensure_smem_attr(decode_kernel<T, MAXG, DMASK>, smem, attr);
  launch_pdl(decode_kernel<T, MAXG, DMASK>, dim3(grid), dim3(kWarps * 32), smem, s, p);
}

template <typename T, int DMASK>
void launch_decode_g(const DataParams& p, int max_g, int grid, cudaStream_t s) {
  if (max_g <= 1) launch_decode_t<T, 1, DMASK>(p, grid, s);
  else if (max_g <= 2) launch_decode_t<T, 2, DMASK>(p, grid, s);
  else if (max_g <= 4) launch_decode_t<T, 4, DMASK>(p, grid, s);
  else launch_decode_t<T, 8, DMASK>(p, grid, s);
}

}  // namespace

int num_sms() {
  static std::atomic<int> cached[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& c = cached[dev & 63];
  int n = c.load(std::memory_order_relaxed);
  if (n <= 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    c.store(n, std::memory_order_relaxed);
  }
  return n;
}

int decode_ctas_per_sm() { return 1; }
int decode_warps_per_cta() { return kWarps; }

void launch_decode_plan(const DataParams& p, cudaStream_t s) {
  launch_pdl(plan_kernel, dim3(1), dim3(1024), 0, s, p);
}

void launch_decode(const DataParams& p, int max_g, int grid, cudaStream_t s) {
  if (grid <= 0) grid = num_sms() * decode_ctas_per_sm();
  int dmask = 0;
  for (int i = 0; i < p.ngroups; ++i) dmask |= p.g[i].D == 64 ? 1 : p.g[i].D == 128 ? 2 : 4;
  if (p.dtype == 0) {
    if (dmask == 2) launch_decode_g<__half, 2>(p, max_g, grid, s);
    else launch_decode_g<__half, 7>(p, max_g, grid, s);
  } else {
    if (dmask == 2) launch_decode_g<__nv_bfloat16, 2>(p, max_g, grid, s);
    else launch_decode_g<__nv_bfloat16, 7>(p, max_g, grid, s);
  }
}

void launch_append(const DataParams& p, cudaStream_t s) {
  int maxh = 1;
  for (int i = 0; i < p.ngroups; ++i) maxh = max(maxh, p.g[i].Hkv);
  const int warps = (p.q_lens ? p.max_q_len : p.n_new) * maxh;
  dim3 grid((warps + 7) / 8, p.nreq);
  launch_pdl(append_kernel, grid, dim3(256), 0, s, p);
}

void launch_synth_fill(void* pool, size_t bytes, int dtype, unsigned long long seed, float amp,
                       cudaStream_t s) {
  const size_t n16 = bytes / 16;
  const int grid = num_sms() * 8;
  if (dtype == 0) synth_kernel<__half><<<grid, 256, 0, s>>>(reinterpret_cast<uint4*>(pool), n16, seed, amp);
  else synth_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(reinterpret_cast<uint4*>(pool), n16, seed, amp);
}

}  // namespace skv

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

constexpr int kD = 128;                       // head_dim handled by the kernels
constexpr int kTpb = 16;                      // tokens per native block
constexpr int kTile = 2 * kTpb * kD * 2;      // K + V tile bytes (8 KiB)
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

// Sum of 8 per-lane partials over the 16 lanes of a half-warp, scattered so lane
// (c = lane&15) ends up with the total of index (c>>1)&7 (8 shuffles, not 32).
__device__ __forceinline__ float reduce_scatter16(const float (&v)[8], int lane) {
  const bool b3 = lane & 8, b2 = lane & 4, b1 = lane & 2;
  float v4[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float send = b3 ? v[k] : v[k + 4];
    const float keep = b3 ? v[k + 4] : v[k];
    v4[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  float v2[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float send = b2 ? v4[k] : v4[k + 2];
    const float keep = b2 ? v4[k + 2] : v4[k];
    v2[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  const float send = b1 ? v2[0] : v2[1];
  const float keep = b1 ? v2[1] : v2[0];
  float s = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  return s;
}

// One 16-token K/V tile for G query heads sharing a KV head.
// Lane (c = lane&15, hf = lane>>4) reads dims [8c, 8c+8) of tokens 2i+hf.
template <typename T, int G, bool PARTIAL>
__device__ __forceinline__ void consume_tile(const char* tile, int lane, int valid,
                                             const float (&q)[G][8], float (&o)[G][8],
                                             float (&mx)[G], float (&l)[G]) {
  const int c = lane & 15, hf = lane >> 4;
  float part[G][8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint4 raw = *reinterpret_cast<const uint4*>(tile + (2 * i + hf) * (kD * 2) + c * 16);
    float kf[8];
    Cvt<T>::to_f32(raw, kf);
#pragma unroll
    for (int g = 0; g < G; ++g) {  // packed fp32 FMA (FFMA2): 4 + 1 instructions per 8 dims
      float2 a = __fmul2_rn(make_float2(q[g][0], q[g][1]), make_float2(kf[0], kf[1]));
#pragma unroll
      for (int j = 2; j < 8; j += 2) a = __ffma2_rn(make_float2(q[g][j], q[g][j + 1]), make_float2(kf[j], kf[j + 1]), a);
      part[g][i] = a.x + a.y;
    }
  }
  const int tok = 2 * ((c >> 1) & 7) + hf;
  float p[G];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    float s = reduce_scatter16(part[g], lane);
    if (tok >= valid) s = -INFINITY;
    float bm = s;
    bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 2));
    bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 4));
    bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 8));
    bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 16));
    const float mnew = fmaxf(mx[g], bm);
    const float alpha = exp2f(mx[g] - mnew);
    p[g] = exp2f(s - mnew);
    l[g] = l[g] * alpha + p[g];
    const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      const float2 r = __fmul2_rn(make_float2(o[g][j], o[g][j + 1]), a2);
      o[g][j] = r.x;
      o[g][j + 1] = r.y;
    }
    mx[g] = mnew;
  }
  const char* vt = tile + kTpb * kD * 2;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint4 raw = *reinterpret_cast<const uint4*>(vt + (2 * i + hf) * (kD * 2) + c * 16);
    if (PARTIAL && 2 * i + hf >= valid) raw = make_uint4(0u, 0u, 0u, 0u);  // unwritten slots may hold NaN
    float vf[8];
    Cvt<T>::to_f32(raw, vf);
    const int src = (hf << 4) | (i << 1);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const float pt = __shfl_sync(0xffffffffu, p[g], src);
      const float2 pt2 = make_float2(pt, pt);
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        const float2 r = __ffma2_rn(pt2, make_float2(vf[j], vf[j + 1]), make_float2(o[g][j], o[g][j + 1]));
        o[g][j] = r.x;
        o[g][j + 1] = r.y;
      }
    }
  }
}

// Block-table row of (request handle, kv head) at the launch's layer: one row per request
// in the merged scheme, one per (request, layer, kv head) in the split scheme.
__device__ __forceinline__ const int2* table_row(const DataParams& p, int handle, int head) {
  return p.split_L ? p.req_table + (((size_t)handle * p.split_L + p.layer) * p.split_H + head) * p.cap
                   : p.req_table + (size_t)handle * p.cap;
}

// G = 1 (MHA) variant of consume_tile: q stays in 16-bit (qraw, this lane's 8 dims) and
// both dot products run as mixed-precision FMAs (fp32 accumulate, 16-bit operands), so
// neither K nor V is converted; P is rounded to the 16-bit type for P.V, as the tensor-core
// prefill does.  About 30 % fewer instructions per tile than the converting path.
template <typename T, bool PARTIAL>
__device__ __forceinline__ void consume_tile_mha(const char* tile, int lane, int valid, const uint4& qraw,
                                                 float scale_log2, float (&o)[8], float& mx, float& l) {
  const int c = lane & 15, hf = lane >> 4;
  const unsigned short* qh = reinterpret_cast<const unsigned short*>(&qraw);
  float part[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint4 raw = *reinterpret_cast<const uint4*>(tile + (2 * i + hf) * (kD * 2) + c * 16);
    const unsigned short* kh = reinterpret_cast<const unsigned short*>(&raw);
    float a = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) a = MixFma<T>::f(a, qh[j], kh[j]);
    part[i] = a;
  }
  const int tok = 2 * ((c >> 1) & 7) + hf;
  float sc = reduce_scatter16(part, lane) * scale_log2;
  if (tok >= valid) sc = -INFINITY;
  float bm = sc;
  bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 2));
  bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 4));
  bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 8));
  bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 16));
  const float mnew = fmaxf(mx, bm);
  const float alpha = exp2f(mx - mnew);
  const float pr = exp2f(sc - mnew);
  l = l * alpha + pr;
  const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    const float2 r = __fmul2_rn(make_float2(o[j], o[j + 1]), a2);
    o[j] = r.x;
    o[j + 1] = r.y;
  }
  mx = mnew;
  const char* vt = tile + kTpb * kD * 2;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint4 raw = *reinterpret_cast<const uint4*>(vt + (2 * i + hf) * (kD * 2) + c * 16);
    if (PARTIAL && 2 * i + hf >= valid) raw = make_uint4(0u, 0u, 0u, 0u);  // unwritten slots may hold NaN
    const unsigned short* vh = reinterpret_cast<const unsigned short*>(&raw);
    const unsigned short ph = Cvt<T>::one(__shfl_sync(0xffffffffu, pr, (hf << 4) | (i << 1)));
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = MixFma<T>::f(o[j], ph, vh[j]);
  }
}

// Per-warp producer: walks the same item sequence as the consumer, kStages tiles ahead.
struct Producer {
  int idx;         // current item, -1 before the first
  int blk, bend;   // next block to issue / end (native block indices)
  int cbase;       // first block of the cached table chunk (-1 = none)
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
    P.blk = it.z / kTpb;
    P.bend = (it.w + kTpb - 1) / kTpb;
    P.row = table_row(p, p.handles[it.x], it.y & 0xffff);
    P.base = p.pool + g.layer_off + (long long)(it.y & 0xffff) * g.head_stride;
    P.nstride = g.native_stride;
    P.cbase = -1;
  }
  if (P.done || P.blk >= P.bend) return false;
  if (P.cbase < 0 || P.blk - P.cbase >= 32) {
    P.cbase = P.blk;
    const int b = P.blk + w.lane;
    P.tc = b < P.bend ? P.row[b] : make_int2(0, 0);
  }
  const int rel = P.blk - P.cbase;
  const int bx = __shfl_sync(0xffffffffu, P.tc.x, rel);
  const int by = __shfl_sync(0xffffffffu, P.tc.y, rel);
  const int stage = P.issued % kStages;
  if (w.lane == 0) {
    const char* src = P.base + (long long)bx * p.merged_stride + (long long)by * P.nstride;
    mbar_expect_tx(&w.bars[stage], kTile);
    bulk_g2s(w.tiles + stage * kTile, src, kTile, &w.bars[stage], w.policy);
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

template <typename T, int G>
__device__ __forceinline__ void process_item(const DataParams& p, Producer& P, const WarpCtx& w,
                                             const int4 it, int idx) {
  const int lane = w.lane, c = lane & 15, hf = lane >> 4;
  const int grp = it.y >> 16, head = it.y & 0xffff;
  const DataGroup& g = p.g[grp];
  const int rl = it.x - g.req_begin;
  float q[G][8], o[G][8], mx[G], l[G];
  uint4 qraw = make_uint4(0u, 0u, 0u, 0u);  // G = 1: this lane's 8 raw query dims
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    const T* qp = reinterpret_cast<const T*>(g.q) + ((size_t)rl * g.Hq + head * G + gg) * kD;
    const uint4 raw = *reinterpret_cast<const uint4*>(qp + c * 8);
    if (G == 1) qraw = raw;
    Cvt<T>::to_f32(raw, q[gg]);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      q[gg][j] *= p.scale_log2;
      o[gg][j] = 0.f;
    }
    mx[gg] = -INFINITY;
    l[gg] = 0.f;
  }
  // fused append (n_new == 1): the item holding position ctx-1 writes the step's new
  // K/V token into the pool and patches it into the staged tile before attending
  int apos = -1;
  if (p.n_new == 1 && g.k != nullptr) {
    const int pos = p.req_tokens[p.handles[it.x]] - 1;
    if (pos >= it.z && pos < it.w) apos = pos;
  }
  const int b0 = it.z / kTpb, b1 = (it.w + kTpb - 1) / kTpb;
  for (int b = b0; b < b1; ++b) {
    if (P.issued == P.consumed) fill(p, P, w);
    const int stage = P.consumed % kStages;
    const uint32_t phase = (P.consumed / kStages) & 1u;
    mbar_wait(&w.bars[stage], phase);
    if (apos >= 0 && b == apos / kTpb) {
      // lanes 0-15 move the K row, 16-31 the V row (16 B each), as append_kernel
      const int kv = lane >> 4;
      const int2 e = table_row(p, p.handles[it.x], head)[b];
      const uint4 val = *reinterpret_cast<const uint4*>(reinterpret_cast<const char*>(kv ? g.v : g.k) +
                                                        ((size_t)rl * g.Hkv + head) * (kD * 2) + c * 16);
      const int off = kv * (kTpb * kD * 2) + (apos % kTpb) * (kD * 2) + c * 16;
      *reinterpret_cast<uint4*>(p.pool + g.layer_off + (long long)head * g.head_stride +
                                (long long)e.x * p.merged_stride + (long long)e.y * g.native_stride + off) = val;
      *reinterpret_cast<uint4*>(w.tiles + stage * kTile + off) = val;
      // the slot is refilled by TMA (async proxy) later: order this generic write first
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
    }
    const int valid = min(kTpb, it.w - b * kTpb);
    if constexpr (G == 1) {
      if (valid == kTpb)
        consume_tile_mha<T, false>(w.tiles + stage * kTile, lane, valid, qraw, p.scale_log2, o[0], mx[0], l[0]);
      else
        consume_tile_mha<T, true>(w.tiles + stage * kTile, lane, valid, qraw, p.scale_log2, o[0], mx[0], l[0]);
    } else {
      if (valid == kTpb) consume_tile<T, G, false>(w.tiles + stage * kTile, lane, valid, q, o, mx, l);
      else consume_tile<T, G, true>(w.tiles + stage * kTile, lane, valid, q, o, mx, l);
    }
    __syncwarp();
    P.consumed++;
    fill(p, P, w);
  }
  // finalize: l over the 16 distinct token lanes, o over the two token halves
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    float s = l[gg];
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 8);
    s += __shfl_xor_sync(0xffffffffu, s, 16);
    l[gg] = s;
#pragma unroll
    for (int j = 0; j < 8; ++j) o[gg][j] += __shfl_xor_sync(0xffffffffu, o[gg][j], 16);
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
        T* op = reinterpret_cast<T*>(g.out) + ((size_t)rl * g.Hq + head * G + gg) * kD + c * 8;
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
      float4* dst = reinterpret_cast<float4*>(p.ws_o + slot * kD + c * 8);
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
    // lane (c, hf): dims [8c, 8c+8) over pieces hf, hf+2, ...
    float L = 0.f, acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
#pragma unroll 2
    for (int s = hf; s < ns; s += 2) {
      const size_t slot = (size_t)x.y + (size_t)s * G + gg;
      const float2 ml = __ldcg(p.ws_ml + slot);
      const float4* src = reinterpret_cast<const float4*>(p.ws_o + slot * kD + c * 8);
      const float4 a = __ldcg(src), b = __ldcg(src + 1);
      const float wgt = ml.y > 0.f ? exp2f(ml.x - M) : 0.f;
      L += ml.y * wgt;
      acc[0] += a.x * wgt;
      acc[1] += a.y * wgt;
      acc[2] += a.z * wgt;
      acc[3] += a.w * wgt;
      acc[4] += b.x * wgt;
      acc[5] += b.y * wgt;
      acc[6] += b.z * wgt;
      acc[7] += b.w * wgt;
    }
    L += __shfl_xor_sync(0xffffffffu, L, 16);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], 16);
    if (hf == 0) {
      const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] *= inv;
      T* op = reinterpret_cast<T*>(g.out) + ((size_t)rl * g.Hq + head * G + gg) * kD + c * 8;
      *reinterpret_cast<uint4*>(op) = Cvt<T>::from_f32(acc);
    }
  }
  if (lane == 0) p.arrive[x.w] = 0;  // ready for the launch after next (same counter set)
}

template <typename T, int MAXG>
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
  P.cbase = -1;
  P.tc = make_int2(0, 0);
  P.row = nullptr;
  P.base = nullptr;
  P.nstride = 0;
  P.done = 0;
  P.pushed = P.popped = 0;
  P.issued = P.consumed = 0;
  // Everything before pdl_wait() overlaps the previous launch's tail.  With prefetch the
  // first kStages K/V tiles of this warp are already in flight: the cache bytes of this
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
    const int G = p.g[it.y >> 16].G;
    if (G == 1) process_item<T, 1>(p, P, w, it, idx);
    else if (MAXG >= 2 && G == 2) process_item<T, (MAXG >= 2 ? 2 : 1)>(p, P, w, it, idx);
    else if (MAXG >= 4 && G == 4) process_item<T, (MAXG >= 4 ? 4 : 1)>(p, P, w, it, idx);
    else if (MAXG >= 8 && G == 8) process_item<T, (MAXG >= 8 ? 8 : 1)>(p, P, w, it, idx);
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
  const int total = p.n_new * g.Hkv;
  if (wglob >= total) return;
  const int i = wglob / g.Hkv, h = wglob % g.Hkv;
  const int handle = p.handles[r];
  const int pos = p.req_tokens[handle] - p.n_new + i;
  if (pos < 0) return;
  const int2 e = table_row(p, handle, h)[pos / kTpb];
  const int kv = lane >> 4, c = lane & 15;
  char* dst = p.pool + (long long)e.x * p.merged_stride + (long long)e.y * g.native_stride + g.layer_off +
              (long long)h * g.head_stride + kv * (kTpb * kD * 2) + (pos % kTpb) * (kD * 2) + c * 16;
  const int rl = r - g.req_begin;
  const char* src = reinterpret_cast<const char*>(kv ? g.v : g.k) +
                    (((size_t)rl * p.n_new + i) * g.Hkv + h) * (kD * 2) + c * 16;
  *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
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

template <typename T, int MAXG>
void launch_decode_t(const DataParams& p, int grid, cudaStream_t s) {
  const int smem = kWarps * kStages * kTile + kWarps * kStages * 8 + kWarps * kRing * 4;
  static std::atomic<uint64_t> attr{0};
  ensure_smem_attr(decode_kernel<T, MAXG>, smem, attr);
  launch_pdl(decode_kernel<T, MAXG>, dim3(grid), dim3(kWarps * 32), smem, s, p);
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
  if (p.dtype == 0) {
    if (max_g <= 1) launch_decode_t<__half, 1>(p, grid, s);
    else if (max_g <= 2) launch_decode_t<__half, 2>(p, grid, s);
    else if (max_g <= 4) launch_decode_t<__half, 4>(p, grid, s);
    else launch_decode_t<__half, 8>(p, grid, s);
  } else {
    if (max_g <= 1) launch_decode_t<__nv_bfloat16, 1>(p, grid, s);
    else if (max_g <= 2) launch_decode_t<__nv_bfloat16, 2>(p, grid, s);
    else if (max_g <= 4) launch_decode_t<__nv_bfloat16, 4>(p, grid, s);
    else launch_decode_t<__nv_bfloat16, 8>(p, grid, s);
  }
}

void launch_append(const DataParams& p, cudaStream_t s) {
  int maxh = 1;
  for (int i = 0; i < p.ngroups; ++i) maxh = max(maxh, p.g[i].Hkv);
  const int warps = p.n_new * maxh;
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

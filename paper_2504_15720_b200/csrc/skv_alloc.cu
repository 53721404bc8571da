// skv_alloc.cu — GPU block allocator for the unified KV pool (sm_100a).
//
// Bit-exact restatement of the reference claim/release policy
// (kv_cache.hpp:191-240) for a whole batch of operations at once:
//
//   claim_slot: a model with partially filled merged blocks takes the lowest-id
//   one and its lowest empty sub-slot (:195-204); otherwise it takes the lowest
//   free merged block (:207-217).
//
// For a run of grows with no frees in between this is equivalent to:
//   * model m consumes its open (block, slot) pairs in lexicographic order, then
//     slots of fresh blocks 0..sub-1 in order;
//   * fresh blocks are handed out across all models in op order as the
//     successive lowest free block ids.
// So a batch needs only (i) a per-model prefix of claims (block-wide scans),
// (ii) the first N set bits of the free bitmap, (iii) the first K open slots of
// each model — all computed by one 1024-thread CTA with warp-aggregated scans.
// Frees are order-independent (set inserts): one warp per request with
// warp-aggregated atomics on the occupancy masks, then an idempotent fix-up pass.
#include <algorithm>

#include "skv_internal.h"

namespace skv {

namespace {

constexpr int kGrowThreads = 1024;

__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Block-wide exclusive scan over kGrowThreads threads; returns (exclusive, total).
__device__ __forceinline__ int block_excl_scan(int v, int* total, int* sm_warp) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int incl = warp_incl_scan(v);
  if (lane == 31) sm_warp[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int w = lane < (int)(blockDim.x >> 5) ? sm_warp[lane] : 0;
    const int wi = warp_incl_scan(w);
    sm_warp[lane] = wi - w;  // exclusive warp offsets
    if (lane == 31) sm_warp[32] = wi;
  }
  __syncthreads();
  const int ex = sm_warp[wid] + incl - v;
  *total = sm_warp[32];
  __syncthreads();
  return ex;
}

__device__ __forceinline__ int ceil_div(int a, int b) { return (a + b - 1) / b; }

__device__ __forceinline__ unsigned long long full_mask(int sub) {
  return sub >= 64 ? ~0ull : ((1ull << sub) - 1ull);
}

// Decode-step ops (STEP): op i = try_allocate(req_id[h], model, tokens + delta) of batch request
// i, from the device's own request state (the host mirror found every one granted).
struct StepArgs {
  const int32_t* handles;
  const int32_t* group;
  StepModels gm;
  int delta, tpb;
};

// SMALL (n <= kSmallOps ops, <= kSmallClaims claims — every decode step): ops and all scratch
// live in shared memory, so the phases exchange data without global-memory round trips.
constexpr int kSmallOps = 1024, kSmallClaims = 2048;
constexpr int kSmallSmem = kSmallOps * (int)sizeof(GrowOp) + 5 * kSmallOps * 4 + kSmallClaims * (4 + 4 + 8);

template <bool STEP, bool SMALL, int NT>
__global__ void __launch_bounds__(NT, 1)
grow_kernel(DevAlloc st, AllocParams pr, const GrowOp* ops_g, int n, GrowScratch sc_g, StepArgs sa) {
  extern __shared__ __align__(16) char gsm[];
  const GrowOp* ops = ops_g;  // no __restrict__: STEP writes them
  GrowScratch sc = sc_g;
  if constexpr (SMALL) {
    GrowOp* o = reinterpret_cast<GrowOp*>(gsm);
    int32_t* a = reinterpret_cast<int32_t*>(gsm + kSmallOps * sizeof(GrowOp));
    sc.S = a;
    sc.cbeg = a + kSmallOps;
    sc.nnew = a + 2 * kSmallOps;
    sc.base = a + 3 * kSmallOps;
    sc.nbfirst = a + 4 * kSmallOps;
    sc.newblk = a + 5 * kSmallOps;
    sc.newrank = a + 5 * kSmallOps + kSmallClaims;
    sc.openlist = reinterpret_cast<int2*>(a + 5 * kSmallOps + 2 * kSmallClaims);
    if constexpr (!STEP)
      for (int i = threadIdx.x; i < n; i += NT) o[i] = ops_g[i];
    ops = o;
  }
  __shared__ int sm_warp[33];
  __shared__ int carryC[kMaxModels];   // claims per model so far
  __shared__ long long O[kMaxModels];  // open slots at batch start
  __shared__ int needOpen[kMaxModels], offOpen[kMaxModels], newcnt[kMaxModels], offNew[kMaxModels];
  __shared__ int carryNew, carryCl, sh_total;
  __shared__ int hint[1 + kMaxModels];  // bitmap scan starts (DevAlloc::hints), updated at the end
  const int tid = threadIdx.x;
  const int M = pr.M;
  if (tid < M) {
    carryC[tid] = 0;
    O[tid] = st.open[tid];
  }
  if (tid <= M) hint[tid] = st.hints[tid];
  if (tid == 0) carryNew = carryCl = 0;
  if constexpr (STEP) {  // phase 0: the ops themselves
    GrowOp* w = const_cast<GrowOp*>(ops);  // shared memory (SMALL) or the batch's buffer
    for (int i = tid; i < n; i += NT) {
      const int h = sa.handles[i];
      const int have = st.req_nslots[h];
      const int tok = st.req_tokens[h] + sa.delta;
      GrowOp op;
      op.handle = h;
      op.model = sa.gm.m[sa.group[i]];
      op.have = have;
      op.claims = max(0, (tok + sa.tpb - 1) / sa.tpb - have);
      op.tokens_after = tok;
      op.pad = 0;
      op.id = st.req_id[h];
      w[i] = op;
    }
    __threadfence_block();
  }
  __syncthreads();
  {  // token-only growth (15 of every 16 decode steps at tpb 16): no placement work at all
    int any = 0;
    for (int i = tid; i < n; i += NT) any |= ops[i].claims > 0;
    if (!__syncthreads_or(any)) {
      for (int i = tid; i < n; i += NT) {
        const GrowOp op = ops[i];
        atomicMax(&st.req_tokens[op.handle], op.tokens_after);
        st.req_model[op.handle] = op.model;
        st.req_id[op.handle] = op.id;
      }
      return;
    }
  }

  // ---- phase 1: per-model claim prefixes and fresh-block counts ------------------
  for (int c0 = 0; c0 < n; c0 += NT) {
    const int i = c0 + tid;
    const bool valid = i < n;
    GrowOp op{};
    if (valid) op = ops[i];
    const int cl = valid ? op.claims : 0;
    int S = 0;
    for (int mm = 0; mm < M; ++mm) {
      int tot;
      const int v = (valid && op.model == mm) ? cl : 0;
      const int ex = block_excl_scan(v, &tot, sm_warp);
      if (valid && op.model == mm) S = carryC[mm] + ex;
      __syncthreads();
      if (tid == 0) carryC[mm] += tot;
      __syncthreads();
    }
    int nn = 0, nbf = 0;
    if (valid && cl > 0) {
      const int sub = pr.sub[op.model];
      const int Om = (int)O[op.model];
      const int a = max(S, Om) - Om, b = S + cl - Om;
      if (b > a) {
        nbf = ceil_div(a, sub);
        nn = ceil_div(b, sub) - nbf;
      }
    }
    int tot;
    const int exn = block_excl_scan(nn, &tot, sm_warp);
    const int base = carryNew + exn;
    int totc;
    const int exc = block_excl_scan(cl, &totc, sm_warp);
    if (valid) {
      sc.S[i] = S;
      sc.nnew[i] = nn;
      sc.base[i] = base;
      sc.nbfirst[i] = nbf;
      sc.cbeg[i] = carryCl + exc;
    }
    __syncthreads();
    if (tid == 0) {
      carryNew += tot;
      carryCl += totc;
    }
    __syncthreads();
  }
  const int Nnew = carryNew, Tcl = carryCl;
  if (tid == 0) {
    int offo = 0, offn = 0;
    for (int m = 0; m < M; ++m) {
      const int claims = carryC[m];
      needOpen[m] = (int)min((long long)claims, O[m]);
      offOpen[m] = offo;
      offo += needOpen[m];
      newcnt[m] = claims > O[m] ? ceil_div(claims - (int)O[m], pr.sub[m]) : 0;
      offNew[m] = offn;
      offn += newcnt[m];
    }
  }
  __syncthreads();

  // ---- phase 2a: the Nnew lowest free block ids (words below hint[0] hold none) --------
  {
    int cum = 0;
    for (int w0 = hint[0]; w0 < pr.W && cum < Nnew; w0 += NT) {
      const int w = w0 + tid;
      uint32_t bits = w < pr.W ? st.free_bits[w] : 0u;
      int tot;
      int r = cum + block_excl_scan(__popc(bits), &tot, sm_warp);
      while (bits && r < Nnew) {
        const int bpos = __ffs(bits) - 1;
        sc.newblk[r++] = w * 32 + bpos;
        bits &= bits - 1;
      }
      cum += tot;
    }
    if (tid == 0 && cum < Nnew) atomicExch(st.status, 1);  // host admitted more than exists
  }
  __syncthreads();
  if (tid == 0 && Nnew > 0) hint[0] = sc.newblk[Nnew - 1] >> 5;  // every lower free block was taken

  // ---- phase 2b: the first needOpen[m] open slots of each model, lexicographic -------
  for (int m = 0; m < M; ++m) {
    const int need = needOpen[m];
    if (need == 0) continue;
    const int sub = pr.sub[m];
    const unsigned long long fm = full_mask(sub);
    const uint32_t* pb = st.partial_bits + (size_t)m * pr.W;
    int cum = 0;
    for (int w0 = hint[1 + m]; w0 < pr.W && cum < need; w0 += NT) {
      const int w = w0 + tid;
      uint32_t bits = w < pr.W ? pb[w] : 0u;
      int cnt = 0;
      for (uint32_t t = bits; t; t &= t - 1) {
        const int blk = w * 32 + __ffs(t) - 1;
        cnt += sub - __popcll(st.blk_occ[blk] & fm);
      }
      int tot;
      int r = cum + block_excl_scan(cnt, &tot, sm_warp);
      for (uint32_t t = bits; t && r < need; t &= t - 1) {
        const int blk = w * 32 + __ffs(t) - 1;
        unsigned long long freem = ~st.blk_occ[blk] & fm;
        while (freem && r < need) {
          const int s = __ffsll(freem) - 1;
          sc.openlist[offOpen[m] + r++] = make_int2(blk, s);
          freem &= freem - 1;
        }
      }
      cum += tot;
    }
    if (tid == 0 && cum < need) atomicExch(st.status, 2);
    __syncthreads();
    // blocks before the last one taken are now full (their partial bits clear in phase 5)
    if (tid == 0) hint[1 + m] = sc.openlist[offOpen[m] + need - 1].x >> 5;
  }

  // ---- phase 3: model-local fresh block -> global rank -----------------------------
  for (int i = tid; i < n; i += NT) {
    const int nn = sc.nnew[i];
    if (nn == 0) continue;
    const int m = ops[i].model;
    const int b0 = sc.base[i], f0 = sc.nbfirst[i];
    for (int t = 0; t < nn; ++t) sc.newrank[offNew[m] + f0 + t] = b0 + t;
  }
  __syncthreads();

  // ---- phase 4: materialise every claim --------------------------------------------
  for (int g = tid; g < Tcl; g += NT) {
    int lo = 0, hi = n - 1;  // last op with cbeg <= g
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (sc.cbeg[mid] <= g) lo = mid; else hi = mid - 1;
    }
    const GrowOp op = ops[lo];
    const int j = g - sc.cbeg[lo];
    const int m = op.model, sub = pr.sub[m];
    const int k = sc.S[lo] + j;
    const int Om = (int)O[m];
    int blk, s;
    if (k < Om) {
      const int2 e = sc.openlist[offOpen[m] + k];
      blk = e.x;
      s = e.y;
    } else {
      const int kp = k - Om;
      s = kp % sub;
      blk = sc.newblk[sc.newrank[offNew[m] + kp / sub]];
      if (s == 0) {  // claim_slot's free-list branch (kv_cache.hpp:207-217)
        st.blk_model[blk] = m;
        atomicAnd(&st.free_bits[blk >> 5], ~(1u << (blk & 31)));
      }
    }
    st.req_table[(size_t)op.handle * pr.cap + op.have + j] = make_int2(blk, s);
    st.slot_owner[(size_t)blk * pr.maxsub + s] = op.id;
    atomicOr(&st.blk_occ[blk], 1ull << s);
  }
  __syncthreads();

  // ---- phase 5: partial-set membership, request rows, counters ----------------------
  for (int g = tid; g < Tcl; g += NT) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (sc.cbeg[mid] <= g) lo = mid; else hi = mid - 1;
    }
    const int m = ops[lo].model, sub = pr.sub[m];
    if (sub <= 1) continue;
    const int2 e = st.req_table[(size_t)ops[lo].handle * pr.cap + ops[lo].have + (g - sc.cbeg[lo])];
    const uint32_t bit = 1u << (e.x & 31);
    uint32_t* word = &st.partial_bits[(size_t)m * pr.W + (e.x >> 5)];
    if (st.blk_occ[e.x] == full_mask(sub)) {
      atomicAnd(word, ~bit);  // :204
    } else {
      atomicOr(word, bit);  // :217
      atomicMin(&hint[1 + m], e.x >> 5);
    }
  }
  for (int i = tid; i < n; i += NT) {
    const GrowOp op = ops[i];
    atomicMax(&st.req_nslots[op.handle], op.have + op.claims);
    atomicMax(&st.req_tokens[op.handle], op.tokens_after);
    st.req_model[op.handle] = op.model;
    st.req_id[op.handle] = op.id;
  }
  if (tid < M) {
    st.open[tid] = O[tid] + (long long)newcnt[tid] * pr.sub[tid] - carryC[tid];
  }
  if (tid == 0) st.free_count[0] -= Nnew;
  __syncthreads();
  if (tid <= M) st.hints[tid] = hint[tid];
  (void)Tcl;
}

// Release every slot of the freed requests (kv_cache.hpp:224-240).  One warp per
// request; emptied-block counts are warp-aggregated (ballot + popc) before the atomic.
__global__ void free_release_kernel(DevAlloc st, AllocParams pr, const FreeOp* __restrict__ ops,
                                    int n) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < n; i += nwarps) {
    const FreeOp op = ops[i];
    const int2* row = st.req_table + (size_t)op.handle * pr.cap;
    int emptied = 0;
    for (int j0 = 0; j0 < op.nslots; j0 += 32) {
      const int j = j0 + lane;
      bool e = false;
      if (j < op.nslots) {
        const int2 bs = row[j];
        const unsigned long long bit = 1ull << bs.y;
        st.slot_owner[(size_t)bs.x * pr.maxsub + bs.y] = 0ull;
        const unsigned long long old = atomicAnd(&st.blk_occ[bs.x], ~bit);
        if (old == bit) {  // last occupant left: back to the free list (:228-234)
          e = true;
          st.blk_model[bs.x] = -1;
          atomicOr(&st.free_bits[bs.x >> 5], 1u << (bs.x & 31));
          atomicMin(&st.hints[0], bs.x >> 5);
        }
      }
      emptied += __popc(__ballot_sync(0xffffffffu, e));
    }
    if (lane == 0) {
      if (emptied) atomicAdd(&st.free_E[op.model], emptied);
      atomicAdd(&st.free_R[op.model], op.nslots);
    }
  }
}

// Idempotent fix-up of partial-set membership from the final occupancy, then the
// counters (block 0): open += R - E*sub, free += E.
__global__ void free_fixup_kernel(DevAlloc st, AllocParams pr, const FreeOp* __restrict__ ops,
                                  int n, int32_t* out_E) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int i = warp; i < n; i += nwarps) {
    const FreeOp op = ops[i];
    const int2* row = st.req_table + (size_t)op.handle * pr.cap;
    if (pr.sub[op.model] > 1) {
      for (int j = lane; j < op.nslots; j += 32) {
        const int2 bs = row[j];
        const uint32_t bit = 1u << (bs.x & 31);
        uint32_t* word = &st.partial_bits[(size_t)op.model * pr.W + (bs.x >> 5)];
        if (st.blk_occ[bs.x] == 0ull) {
          atomicAnd(word, ~bit);  // :229
        } else {
          atomicOr(word, bit);  // :236
          atomicMin(&st.hints[1 + op.model], bs.x >> 5);
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      st.req_nslots[op.handle] = 0;
      st.req_tokens[op.handle] = 0;
      st.req_model[op.handle] = -1;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < pr.M) {
    const int m = threadIdx.x;
    const int E = st.free_E[m], R = st.free_R[m];
    st.open[m] += (long long)R - (long long)E * pr.sub[m];
    atomicAdd((unsigned long long*)st.free_count, (unsigned long long)(long long)E);
    out_E[m] = E;
    st.free_E[m] = 0;
    st.free_R[m] = 0;
  }
}

}  // namespace

// Host (pinned, mapped) -> device copy done by SMs instead of a copy engine: the small
// per-step op uploads must not queue behind a caller's bulk H2D/D2H copies in the copy
// engines' FIFOs (measured: a 200 MB input copy on another stream delayed the step's
// allocator upload by its full duration).
__global__ void stage_copy_kernel(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// bytes: a multiple of 4 (ops and index arrays)
void launch_stage_copy(void* dst, const void* src_host_mapped, size_t bytes, cudaStream_t s) {
  const size_t n4 = bytes / 4;
  if (!n4) return;
  const int threads = 256;
  const int blocks = (int)std::min<size_t>((n4 + threads - 1) / threads, 64);
  stage_copy_kernel<<<blocks, threads, 0, s>>>(static_cast<uint32_t*>(dst), static_cast<const uint32_t*>(src_host_mapped),
                                               n4);
}

// Split scheme: claim c of op i (c in [0, nblk*L*H)) is native block blk0 + c/(L*H),
// layer (c/H)%L, head c%H; it takes stack[base + c] (the host moved the stack top).
__device__ __forceinline__ int split_op_of(const SplitOp* ops, int n, long long c) {
  int lo = 0, hi = n - 1;  // last op with cbeg <= c
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (ops[mid].cbeg <= c) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void split_claim_kernel(const SplitOp* __restrict__ ops, int n, long long total,
                                   const int32_t* __restrict__ stack, int2* __restrict__ table, int Lmax, int Hmax,
                                   int cap) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < total; c += (long long)gridDim.x * blockDim.x) {
    const SplitOp op = ops[split_op_of(ops, n, c)];
    const long long k = c - op.cbeg;
    const int lh = op.L * op.H;
    const int blk = op.blk0 + (int)(k / lh), l = (int)(k / op.H) % op.L, h = (int)(k % op.H);
    table[(((size_t)op.handle * Lmax + l) * Hmax + h) * cap + blk] = make_int2(stack[op.base + k], 0);
  }
}

__global__ void split_release_kernel(const SplitOp* __restrict__ ops, int n, long long total,
                                     int32_t* __restrict__ stack, const int2* __restrict__ table, int Lmax, int Hmax,
                                     int cap) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < total; c += (long long)gridDim.x * blockDim.x) {
    const SplitOp op = ops[split_op_of(ops, n, c)];
    const long long k = c - op.cbeg;
    const int lh = op.L * op.H;
    const int blk = op.blk0 + (int)(k / lh), l = (int)(k / op.H) % op.L, h = (int)(k % op.H);
    stack[op.base + k] = table[(((size_t)op.handle * Lmax + l) * Hmax + h) * cap + blk].x;
  }
}

void launch_split_claim(const SplitOp* ops, int n, long long total, const int32_t* stack, int2* table, int Lmax,
                        int Hmax, int cap, cudaStream_t s) {
  if (total <= 0) return;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 8);
  split_claim_kernel<<<blocks, 256, 0, s>>>(ops, n, total, stack, table, Lmax, Hmax, cap);
}

void launch_split_release(const SplitOp* ops, int n, long long total, int32_t* stack, const int2* table, int Lmax,
                          int Hmax, int cap, cudaStream_t s) {
  if (total <= 0) return;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 8);
  split_release_kernel<<<blocks, 256, 0, s>>>(ops, n, total, stack, table, Lmax, Hmax, cap);
}

template <bool STEP>
void launch_grow_t(const DevAlloc& st, const AllocParams& pr, const GrowOp* ops, int n, long long claims,
                   const GrowScratch& sc, StepArgs sa, cudaStream_t s) {
  if (n <= 0) return;
  if (n <= 256 && claims <= kSmallClaims) {  // small batches: 8 warps (cheaper block barriers)
    static std::atomic<uint64_t> attr{0};
    ensure_smem_attr(grow_kernel<STEP, true, 256>, kSmallSmem, attr);
    grow_kernel<STEP, true, 256><<<1, 256, kSmallSmem, s>>>(st, pr, ops, n, sc, sa);
  } else if (n <= kSmallOps && claims <= kSmallClaims) {
    static std::atomic<uint64_t> attr{0};
    ensure_smem_attr(grow_kernel<STEP, true, kGrowThreads>, kSmallSmem, attr);
    grow_kernel<STEP, true, kGrowThreads><<<1, kGrowThreads, kSmallSmem, s>>>(st, pr, ops, n, sc, sa);
  } else {
    grow_kernel<STEP, false, kGrowThreads><<<1, kGrowThreads, 0, s>>>(st, pr, ops, n, sc, sa);
  }
}

void launch_grow_step(const DevAlloc& st, const AllocParams& pr, int tpb, const int32_t* handles,
                      const int32_t* group, StepModels gm, int n, int delta, GrowOp* ops, const GrowScratch& sc,
                      cudaStream_t s) {
  StepArgs sa{handles, group, gm, delta, tpb};
  launch_grow_t<true>(st, pr, ops, n, (long long)n * ((delta + tpb - 1) / tpb + 1), sc, sa, s);
}

void launch_grow(const DevAlloc& st, const AllocParams& pr, const GrowOp* ops, int n, long long claims,
                 const GrowScratch& sc, cudaStream_t s) {
  launch_grow_t<false>(st, pr, ops, n, claims, sc, StepArgs{}, s);
}

void launch_free(const DevAlloc& st, const AllocParams& pr, const FreeOp* ops, int n,
                 int32_t* out_E, cudaStream_t s) {
  if (n <= 0) return;
  const int threads = 256;
  int blocks = (n * 32 + threads - 1) / threads;
  if (blocks > 4 * 148) blocks = 4 * 148;
  free_release_kernel<<<blocks, threads, 0, s>>>(st, pr, ops, n);
  free_fixup_kernel<<<blocks, threads, 0, s>>>(st, pr, ops, n, out_E);
}

}  // namespace skv

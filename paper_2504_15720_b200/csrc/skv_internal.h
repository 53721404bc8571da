// skv_internal.h — structures shared by the host runtime (skv_capi.cpp) and the
// sm_100a kernels (skv_alloc.cu, skv_attn.cu).  Not part of the public ABI.
#pragma once
#include <cuda.h>  // CUtensorMap (header only; the driver entry point is resolved at run time)
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace skv {

// Kernel function attributes are per device: the dynamic shared-memory opt-in of a kernel is
// applied once per (kernel, device) — `done` is the kernel's own device bitmask — so a pool on
// a second device (or another thread) never launches without it.
template <typename K>
inline cudaError_t ensure_smem_attr(K kernel, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

// SM count of the current device (cached per device ordinal, thread-safe).
int num_sms();

constexpr int kMaxModels = 16;   // services sharing one pool
constexpr int kMaxGroups = 16;   // groups in one data-path batch
constexpr int kMaxSub = 64;      // sub-slots per merged block (occupancy is a u64 mask)

// ------------------------------------------------------------------ allocator state --
// Device-resident canonical allocator state.  The reference keeps
// std::set free list / partial sets and per-block slot_owner vectors
// (kv_cache.hpp:173-177, 254-258); here they are bitmaps + flat arrays so a single
// CTA can evaluate a whole batch of claims with block-wide scans.
struct DevAlloc {
  uint32_t* free_bits;           // [W]     1 = merged block on the free list
  uint32_t* partial_bits;        // [M][W]  1 = claimed by model m and not full
  int32_t* blk_model;            // [P]     owner model, -1 = free
  unsigned long long* blk_occ;   // [P]     occupied sub-slot mask
  unsigned long long* slot_owner;// [P*maxsub] request id per sub-slot (0 = empty)
  long long* open;               // [M]     open_slots_ (kv_cache.hpp:254)
  long long* free_count;         // [1]
  int2* req_table;               // [R*cap] (merged block, sub index) per native block
  int32_t* req_nslots;           // [R]
  int32_t* req_tokens;           // [R]     tokens covered (decode context length)
  int32_t* req_model;            // [R]
  unsigned long long* req_id;    // [R]     request id of the handle (written by every grow)
  int32_t* hints;                // [1+M]   lowest bitmap word that may hold a free block / a
                                 //         partial block of model m (scan starts; lower bounds)
  int32_t* status;               // [1]     device invariant violations (0 = ok)
  int32_t* free_E;               // [M]     scratch: blocks emptied by the current free run
  int32_t* free_R;               // [M]     scratch: slots released by the current free run
};

struct AllocParams {
  int M, W, maxsub, cap;
  long long P;
  int sub[kMaxModels];
};

// One granted grow, decided on the host (mirror arithmetic, no device sync).
struct GrowOp {
  int32_t handle, model, have, claims;
  int32_t tokens_after, pad;
  unsigned long long id;
};

struct FreeOp {
  int32_t handle, model, nslots, pad;
};

// Scratch for the grow kernel, sized by the host for the batch.
struct GrowScratch {
  int32_t* S;        // [n] model-local claim index of the op's first claim
  int32_t* cbeg;     // [n] global claim prefix
  int32_t* nnew;     // [n] new merged blocks taken by the op
  int32_t* base;     // [n] global rank of the op's first new block
  int32_t* nbfirst;  // [n] model-local index of the op's first new block
  int32_t* newblk;   // [Nnew] the lowest free block ids, ascending
  int32_t* newrank;  // [Nnew] (per-model regions) model-local new block -> global rank
  int2* openlist;    // [Topen] (per-model regions) open (block, slot) pairs, lexicographic
  long long* out_E;  // [M] (free runs) host-visible copy of emptied-block counts
};

void launch_stage_copy(void* dst, const void* src_host_mapped, size_t bytes, cudaStream_t s);
// Decode-step growth generated on the device: op i = try_allocate(req_id[h], model, tokens + delta)
// of batch request i (h = handles[i], model = group_model[group[i]]), written to ops[i].
struct StepModels {
  int m[kMaxGroups];
};
// Decode-step growth in one launch: the grow kernel generates its ops (written to `ops`) first.
void launch_grow_step(const DevAlloc& st, const AllocParams& pr, int tpb, const int32_t* handles,
                      const int32_t* group, StepModels gm, int n, int delta, GrowOp* ops, const GrowScratch& sc,
                      cudaStream_t s);
void launch_grow(const DevAlloc& st, const AllocParams& pr, const GrowOp* ops, int n, long long claims,
                 const GrowScratch& sc, cudaStream_t s);
void launch_free(const DevAlloc& st, const AllocParams& pr, const FreeOp* ops, int n,
                 int32_t* out_E, cudaStream_t s);

// ------------------------------------------------------------------ data path ------
struct DataGroup {
  const void* q;            // [B_g][Hq][D]
  void* out;                // [B_g][Hq][D]
  const void* k;            // append: [B_g][n_new][Hkv][D]
  const void* v;
  long long native_stride;  // bytes between sub-slots of this model
  long long layer_off;      // bytes: (layer % phys_layers) * layer_stride
  long long head_stride;    // bytes between kv heads
  int Hq, Hkv, G, active;   // active = num_layers > layer
  int req_begin, nreq;      // slice of the batch
  int D;                    // head_dim (64, 128, 256)
  float scale_log2;         // softmax scale * log2(e) (default 1/sqrt(D))
  int pf_base, pf_npairs;   // prefill: first work item of the group, query-tile pairs per (request, head)
};

struct DataParams {
  // TMA descriptor of the whole pool viewed as a 2-D fp16 tensor [pool_bytes/256 rows][128]
  // (one row = one token's head_dim run), box {64, 16}, 128B swizzle: one box = one
  // 64-element half of a native block's K or V tile, landing in UMMA operand layout.
  alignas(64) CUtensorMap kv_tmap;
  alignas(64) CUtensorMap kv_tmap64;   // head_dim 64: rows of 128 B, box {64, 16}, SW128 (K tiles)
  alignas(64) CUtensorMap kv_tmap64v;  // head_dim 64: rows of 128 B, box {32, 16}, SW64 (V halves)
  alignas(64) CUtensorMap kv_tmap256;  // head_dim 256: rows of 512 B, box {64, 16}, SW128
  int has_tmap;                        // bit d/64: the pool has a descriptor for head_dim d
  const int32_t* q_lens;               // prefill: per-request chunk length [nreq] (NULL: n_new)
  const int32_t* q_offs;               // prefill: request's first row in its group's q/out [nreq]
  int max_q_len;
  DataGroup g[kMaxGroups];
  int ngroups;
  int nreq;                  // batch size
  const int32_t* handles;    // [nreq]
  const int32_t* req_group;  // [nreq]
  const int32_t* req_tokens; // [R]
  const int2* req_table;     // [R*cap]
  int cap;
  char* pool;
  long long merged_stride;
  int head_dim, tpb, dtype;
  float scale_log2;          // softmax scale * log2(e)
  int split_tokens;          // decode: max tokens of a phase-1 piece (multiple of tpb)
  int n_cut;                 // decode: (request, kv head)s given trailing pieces (the last ones)
  int n_new;                 // append / prefill tokens per request
  // decode plan
  int4* items;               // [max_items] {req, (group<<16)|kv_head, tok_begin, tok_end}, by phase
  int* n_items;
  int* counter;              // [2] dynamic work counter, finished-CTA count (both self-resetting)
  int prefetch;              // 1: K/V loads may be issued before the PDL wait (see skv_capi.cpp)
  int4* itemx;               // [max_items] {pieces of the (request, kv head), partial-slot base,
                             //  piece index, arrival counter index}
  int* rscr;                 // [5*nreq] plan scratch
  int items_cap, slots_cap;  // capacities of items/itemx/arrive and ws_o/ws_ml (plan guard)
  int32_t* status;           // device invariant flag (DevAlloc::status): plan overflow -> code 3
  int* arrive;               // [items] pieces finished per (request, kv head) (self-resetting)
  int dbg;                   // debug knobs (prefill v5: bit1 = polynomial exp2 for 1/4)
  // split scheme (skv_split.cpp): split_L > 0 -> req_table rows are per (request, layer,
  // kv head): row (handle*split_L + layer)*split_H + head, entry .x = split block id,
  // address = pool + id * merged_stride (8 KiB), every per-group offset/stride is 0
  int split_L, split_H, layer;
  unsigned long long* trace; // debug (SKV_TRACE=1): per warp {start, after wait, end, tiles<<32|items} ns
  float* ws_o;               // [slots][D] unnormalised partial outputs
  float2* ws_ml;             // [slots] (running max (log2 domain), sum)
};

// Split-scheme view installed on an allocator-only registry pool while a split pool
// runs its data path through the shared decode machinery (skv_split.cpp).
struct SplitView {
  int2* table;     // [R][L][H][cap] (split block id, 0)
  char* storage;   // [blocks][8 KiB]
  int L, H, cap;
};

// split-scheme block claims / releases (skv_alloc.cu): op i covers claims
// [cbeg[i], cbeg[i+1]) of the batch, native blocks [blk0, blk0 + nblk) of request
// `handle` for all (layer, head) of its model; ids come from / return to stack[base..]
struct SplitOp {
  int32_t handle, L, H, blk0, nblk, base, cbeg, pad;
};
void launch_split_claim(const SplitOp* ops, int n, long long total, const int32_t* stack, int2* table, int Lmax,
                        int Hmax, int cap, cudaStream_t s);
void launch_split_release(const SplitOp* ops, int n, long long total, int32_t* stack, const int2* table, int Lmax,
                          int Hmax, int cap, cudaStream_t s);

void launch_decode_plan(const DataParams& p, cudaStream_t s);

}  // namespace skv

struct skv_pool;
// hooks of the registry pool used by skv_split.cpp (skv_capi.cpp)
void skv_internal_set_split(skv_pool* p, const skv::SplitView* view);
int skv_internal_handle(const skv_pool* p, uint64_t id);  // -1 if unknown

namespace skv {
void launch_decode(const DataParams& p, int max_g, int grid, cudaStream_t s);
void launch_append(const DataParams& p, cudaStream_t s);
void launch_prefill(const DataParams& p, cudaStream_t s);
void launch_synth_fill(void* pool, size_t bytes, int dtype, unsigned long long seed, float amp,
                       cudaStream_t s);
int decode_ctas_per_sm();
int decode_warps_per_cta();

}  // namespace skv

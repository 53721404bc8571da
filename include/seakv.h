/*
 * seakv.h — C-ABI of libseakv.so, the B200-native unified KV-cache path.
 *
 * Drop-in boundary for seasim::UnifiedKvCache
 * (/root/reference/proj/include/seasim/kv_cache.hpp:46-267).  Every allocator
 * entry point below replaces exactly one reference member/free function and
 * cites it; the C++ drop-in header include/seakv/unified_kv_cache.hpp maps the
 * status codes back to the reference's exception types (ConfigError,
 * ValidationError, std::logic_error; CacheFull stays `false`).
 *
 * The data path (append / decode / prefill attention) has no reference
 * counterpart — the reference prices decode with a cost model at the spot
 * where it records context reads (kv_cache.hpp:138-142, simulation.hpp:281).
 *
 * Conventions: plain pointers and sizes only.  `stream` is a cudaStream_t
 * passed as void* (NULL = the pool's own stream).  Device pointers are marked
 * [dev], host pointers [host].  Every call is single-threaded per pool, as the
 * reference is (kv_cache.hpp:45); different pools may be used from different
 * threads (no global mutable state).
 */
#ifndef SEAKV_H_
#define SEAKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SKV_OK = 0,
  SKV_CACHE_FULL = 1,      /* try_allocate -> false (kv_cache.hpp:110-112) */
  SKV_ERR_CONFIG = -1,     /* seasim::ConfigError */
  SKV_ERR_VALIDATION = -2, /* seasim::ValidationError */
  SKV_ERR_LOGIC = -3,      /* std::logic_error */
  SKV_ERR_CUDA = -4,       /* CUDA runtime / device-side invariant failure */
  SKV_ERR_ARG = -5         /* bad argument or capacity exceeded */
} skv_status;

typedef enum { SKV_FP16 = 0, SKV_BF16 = 1 } skv_dtype;

/* seasim::ModelSpec (cost_model.hpp:19-40) restricted to the fields the KV
 * path reads, plus num_q_heads (GQA; the reference has none). */
typedef struct {
  const char* model_id;
  int32_t num_layers;
  int32_t num_heads;   /* KV heads: ModelSpec::num_heads, sizes the native block */
  int32_t num_q_heads; /* query heads; 0 means num_heads (MHA) */
  int32_t head_dim;
  int32_t dtype_bytes;
} skv_model_desc;

typedef struct {
  int32_t device;                 /* CUDA device ordinal */
  int32_t dtype;                  /* skv_dtype of the stored K/V */
  int32_t phys_layers;            /* 0: every layer stored (faithful merged-block layout).
                                     k>0: layer-sliced pool, k physical layers per native
                                     block, logical layer l -> l % k */
  int32_t max_requests;           /* initial capacity of the device request table (grows on
                                     demand: the reference has no limit, kv_cache.hpp:104-106) */
  int32_t max_blocks_per_request; /* initial block-table row capacity in native blocks (0: min(
                                     pool_blocks * max sub-slots, 4096)); grows on demand.  A
                                     growth re-allocates the device table: CUDA graphs captured
                                     before it must be re-captured.  Fixed for the split scheme. */
  int32_t allocate_storage;       /* 1: allocate the KV bytes in HBM; 0: allocator only */
} skv_pool_opts;

typedef struct skv_pool skv_pool;
typedef struct skv_batch skv_batch;

void skv_default_opts(skv_pool_opts* opts);
const char* skv_version(void);

/* kv_cache.hpp:17-22 */
skv_status skv_native_block_bytes(const skv_model_desc* model, int32_t tokens_per_block,
                                  int32_t tp_size, double* out);
/* kv_cache.hpp:26-33 (n == 0 -> SKV_ERR_CONFIG) */
skv_status skv_plan_merged_shape(const skv_model_desc* models, int32_t n,
                                 int32_t tokens_per_block, int32_t tp_size, double* out);

/* UnifiedKvCache(models, tokens_per_block, tp_size, pool_blocks), kv_cache.hpp:50-66 */
skv_status skv_pool_create(const skv_model_desc* models, int32_t n, int32_t tokens_per_block,
                           int32_t tp_size, size_t pool_blocks, const skv_pool_opts* opts,
                           skv_pool** out);
void skv_pool_destroy(skv_pool* pool);
/* Message of the last failed call on this pool (pool == NULL: this thread's last
 * pool-less failure). */
const char* skv_last_error(const skv_pool* pool);

/* ---- allocator: one entry per reference member ------------------------------------ */
skv_status skv_model_index(const skv_pool* p, const char* model_id, int32_t* out); /* :68-72 */
int32_t skv_sub_slots_per_merged(const skv_pool* p, int32_t model_idx);            /* :74 */
double skv_merged_block_bytes(const skv_pool* p);                                  /* :75 */
size_t skv_pool_size(const skv_pool* p);                                           /* :76 */
size_t skv_free_blocks(skv_pool* p);                                               /* :77 */
size_t skv_allocated_blocks(skv_pool* p);                                          /* :78 */
int32_t skv_tokens_per_block(const skv_pool* p);                                   /* :79 */
size_t skv_native_blocks_for(const skv_pool* p, int64_t tokens);                   /* :81-83 */
int32_t skv_registered(const skv_pool* p, uint64_t request_id);                    /* :85 */
/* Entry::tokens of a registered request (kv_cache.hpp:180); -1 if unknown. */
int64_t skv_request_tokens(const skv_pool* p, uint64_t request_id);
size_t skv_available_slots(skv_pool* p, int32_t model_idx);                        /* :88-90 */
skv_status skv_can_grow_to(skv_pool* p, uint64_t request_id, int32_t model_idx,    /* :92-99 */
                           int64_t tokens_needed, int32_t* out);
/* :104-123 — SKV_OK = granted (true), SKV_CACHE_FULL = false.  Returns without a
 * device sync; the block assignment itself runs on the GPU (lazily, on the pool stream). */
skv_status skv_try_allocate(skv_pool* p, uint64_t request_id, int32_t model_idx,
                            int64_t tokens_needed);
skv_status skv_free_request(skv_pool* p, uint64_t request_id);        /* :126-134 */
skv_status skv_record_context_read(skv_pool* p, uint64_t request_id); /* :138-142 */
/* :144-148 — copies the (merged block, sub index) pairs (int32 x2, token order) of
 * the request into pairs[0..2*cap); *n = table length.  Synchronises the pool. */
skv_status skv_block_table(skv_pool* p, uint64_t request_id, int32_t* pairs, size_t cap,
                           size_t* n);
skv_status skv_owner_of(skv_pool* p, int32_t block, int32_t slot, uint64_t* owner); /* :150-154 */
size_t skv_table_entries(const skv_pool* p);                                        /* :156 */
double skv_fragmentation_bytes(skv_pool* p);                                        /* :161 */

typedef struct { /* CacheStats, kv_cache.hpp:35-40 */
  uint64_t block_table_entries;
  uint64_t native_reads_writes;
  double internal_fragmentation_bytes;
  double peak_utilization;
} skv_cache_stats;
skv_status skv_stats(skv_pool* p, skv_cache_stats* out); /* :163-170 */

/* ---- batched / replay API (no reference counterpart beyond compare_schemes' loop) ---- */
typedef struct { /* KvOp, kv_cache.hpp:270-275: kind 0 = kGrow, 1 = kFree */
  int32_t kind;
  int32_t model_idx;
  uint64_t request_id;
  int64_t tokens;
} skv_kv_op;
/* Applies ops in order with try_allocate/free_request semantics; granted[i] = 1/0
 * for grows (may be NULL).  Stops at the first protocol error. */
skv_status skv_replay(skv_pool* p, const skv_kv_op* ops, size_t n, int32_t* granted);
/* Pushes queued allocator work to the GPU on `stream` (NULL = pool stream). */
skv_status skv_flush(skv_pool* p, void* stream);
skv_status skv_synchronize(skv_pool* p);
skv_status skv_set_stream(skv_pool* p, void* stream);
void* skv_get_stream(const skv_pool* p);

/* ---- request batches for the data path -------------------------------------------- */
/* A batch lists the requests a decode/append/prefill launch covers, grouped by
 * service (model index).  request_ids are concatenated group by group. */
skv_status skv_batch_create(skv_pool* p, const int32_t* group_models, const int32_t* group_sizes,
                            int32_t n_groups, const uint64_t* request_ids, skv_batch** out);
void skv_batch_destroy(skv_batch* b);
/* Re-points an existing batch at a new request list (same semantics as create); device
 * buffers are reused when large enough, so a serving loop can rebatch every iteration. */
skv_status skv_batch_reset(skv_pool* p, skv_batch* b, const int32_t* group_models,
                           const int32_t* group_sizes, int32_t n_groups, const uint64_t* request_ids);
/* Decode-step growth: try_allocate(id, model, tokens + delta) for every request of
 * the batch, in batch order.  *n_granted = number granted (may be NULL). */
skv_status skv_batch_grow(skv_pool* p, skv_batch* b, int64_t delta_tokens, int32_t* n_granted);
/* Decode-step growth with the placement generated on the device (no op upload; the device
 * half can be captured in a CUDA graph together with the step's attention launches):
 *  - skv_batch_grow_mirror: the host mirror of try_allocate(id, model, tokens + delta) for
 *    every request of the batch, applied only when ALL of them are granted and every request
 *    already owns slots (*all_granted = 1); otherwise nothing changes (*all_granted = 0: use
 *    skv_batch_grow, which handles CacheFull per request);
 *  - skv_batch_grow_launch: the device half (op generation from the device's request state
 *    + the placement kernel) on `stream`.  Call (or replay a graph of) it exactly once after
 *    each successful mirror call with the same delta; its buffers are the batch's own and are
 *    sized by the first eager call (capture before that is refused). */
skv_status skv_batch_grow_mirror(skv_pool* p, skv_batch* b, int64_t delta, int32_t* all_granted);
skv_status skv_batch_grow_launch(skv_pool* p, skv_batch* b, int64_t delta, void* stream);
/* Sum over the batch of the attended context tokens x kv-heads x 2 x head_dim x dtype
 * bytes for one layer index (the algorithmic K/V bytes a decode launch must read). */
skv_status skv_batch_decode_bytes(skv_pool* p, skv_batch* b, int32_t layer, double* kv_bytes,
                                  double* total_bytes);

typedef struct {
  const void* const* q; /* [host array of n_groups dev ptrs] each [B_g][Hq/tp][d] */
  void* const* out;     /* [host array of n_groups dev ptrs] each [B_g][Hq/tp][d] */
  float softmax_scale;  /* 0 -> 1/sqrt(head_dim) */
  int32_t layer;        /* logical layer index; groups with num_layers <= layer are skipped */
  int32_t split_tokens; /* split-KV: max tokens of a (request, kv head)'s first piece (the
                           work list also cuts ~1/4 of every context into two trailing
                           pieces, see plan_kernel); 0 = automatic */
  /* Optional fused KV append (NULL = none): the step's new token of every request,
   * [host array of n_groups dev ptrs] each [B_g][1][Hkv/tp][d], is written at position
   * tokens-1 of `layer` and attended in the same launch (== skv_append_kv with n_new 1
   * followed by the decode, one kernel instead of two). */
  const void* const* k;
  const void* const* v;
} skv_decode_args;
/* Paged decode attention over the unified pool: one launch covers every group of
 * the batch (mixed head counts / GQA ratios).  Context of request r = its current
 * token count.  Runs on `stream` after the queued allocator work. */
skv_status skv_decode_attention(skv_pool* p, skv_batch* b, const skv_decode_args* args,
                                void* stream);

/* Work-list schedule chosen by the batch's last decode launch: split_tokens (max tokens of a
 * (request, kv head)'s leading piece; >= 2^30 = no chunking), n_cut (the last n_cut
 * (request, kv head)s of the batch get two trailing pieces, merged in-kernel) and sum_hkv
 * (the (request, kv head)s of the launch).  For tests and the bench's parity sample. */
skv_status skv_batch_plan_info(skv_pool* p, skv_batch* b, int32_t* split_tokens, int64_t* n_cut,
                               int64_t* sum_hkv);

typedef struct {
  const void* const* k; /* [host array of n_groups dev ptrs] each [B_g][n_new][Hkv/tp][d] */
  const void* const* v;
  int32_t layer;
  int32_t n_new; /* new tokens per request, written at positions [tokens-n_new, tokens) */
  const int32_t* n_news; /* optional per-request counts (host, [nreq], batch order); then each
                            group's k / v are packed by request: [sum of its n_news][Hkv/tp][d] */
} skv_append_args;
skv_status skv_append_kv(skv_pool* p, skv_batch* b, const skv_append_args* args, void* stream);

/* Causal chunked-prefill attention: each request's last q_len tokens (positions
 * [tokens-q_len, tokens)) attend to keys [0, pos] already in the pool.  Per-request chunk
 * lengths: q_lens[nreq] (host array, batch order; NULL = q_len for every request), and then
 * each group's q / out are packed by request: [sum of its q_lens][Hq/tp][d].  Head dims 64,
 * 128 and 256 (one tcgen05 launch per head dim present in the batch). */
typedef struct {
  const void* const* q; /* [host array of n_groups dev ptrs] each [B_g][q_len][Hq/tp][d] */
  void* const* out;     /* same shape */
  float softmax_scale;  /* 0 -> 1/sqrt(head_dim) of each group */
  int32_t layer;
  int32_t q_len;
  const int32_t* q_lens; /* optional per-request chunk lengths (host, [nreq]) */
} skv_prefill_args;
skv_status skv_prefill_attention(skv_pool* p, skv_batch* b, const skv_prefill_args* args,
                                 void* stream);

/* ---- pool storage ------------------------------------------------------------------ */
typedef struct { /* byte layout of one model's native blocks */
  int64_t merged_stride, native_stride, layer_stride, head_stride, kv_stride;
  int32_t tpb, head_dim, kv_heads, q_heads, phys_layers, dtype;
} skv_layout;
skv_status skv_model_layout(const skv_pool* p, int32_t model_idx, skv_layout* out);
void* skv_storage(const skv_pool* p, size_t* bytes); /* [dev] base of the KV pool */
/* Fills the pool with SplitMix64 U(-amp, amp) values (element i of the pool viewed as
 * dtype: mix(seed + (i+1)*0x9e3779b97f4a7c15), common.hpp:46-51 constants). */
skv_status skv_synth_fill(skv_pool* p, uint64_t seed, float amp, void* stream);
/* Copies merged blocks ids[0..n) to host dst (n * merged_stride bytes). Syncs. */
skv_status skv_read_blocks(skv_pool* p, const int32_t* ids, size_t n, void* dst);
/* Number of GPU kernels this pool has launched (instrumentation for bench.py). */
/* ---- split scheme (reference: SplitCacheCounter, kv_cache.hpp:277-348) ----
 * The alternative the paper compares against: every native
 * block of a request is split into per-(layer, kv head) blocks of 8 KiB, each with its
 * own table entry (L*H entries per native block instead of one).  The GPU pool below
 * stores those blocks and runs the SAME decode kernel through per-(request, layer,
 * head) tables, so merged and split are measured on one data path.  Accounting
 * (skv_split_stats) is SplitCacheCounter's.  Batches for the split data path are
 * created on the registry pool (skv_split_registry) from registered request ids; grow
 * and free go through skv_split_grow / skv_split_free only. */
typedef struct skv_split skv_split;
skv_status skv_split_create(const skv_model_desc* models, int32_t n, int32_t tokens_per_block,
                            int32_t tp_size, size_t split_blocks, const skv_pool_opts* opts,
                            skv_split** out);
void skv_split_destroy(skv_split* s);
const char* skv_split_last_error(const skv_split* s);
skv_pool* skv_split_registry(skv_split* s);
size_t skv_split_free_blocks(const skv_split* s);
size_t skv_split_pool_size(const skv_split* s);
uint64_t skv_split_kernel_launches(const skv_split* s);
/* SplitCacheCounter::grow for each (id, model, total tokens) (:286-302), all-or-nothing per
 * op against the split-block pool (granted[i] = 0: pool exhausted, nothing changed), plus
 * one GPU launch assigning the new split blocks and writing their table entries. */
skv_status skv_split_grow(skv_split* s, const uint64_t* ids, const int32_t* models,
                          const int64_t* tokens, int32_t n, int32_t* granted);
skv_status skv_split_free(skv_split* s, const uint64_t* ids, int32_t n); /* :304-309 */
skv_status skv_split_stats(const skv_split* s, skv_cache_stats* out);    /* :311-318 */
uint64_t skv_split_table_entries(const skv_split* s); /* live entries (current_entries_) */
skv_status skv_split_synth_fill(skv_split* s, uint64_t seed, float amp, void* stream);
skv_status skv_split_decode(skv_split* s, skv_batch* b, const skv_decode_args* args, void* stream);
skv_status skv_split_append(skv_split* s, skv_batch* b, const skv_append_args* args, void* stream);
/* split block ids of one (request, layer, kv head) row, in token order (tests) */
skv_status skv_split_block_ids(skv_split* s, uint64_t id, int32_t layer, int32_t head, int32_t* out,
                               size_t cap, size_t* n);
/* copies 8 KiB blocks (K then V, [16 tokens][128]) to host memory (tests) */
skv_status skv_split_read_blocks(skv_split* s, const int32_t* ids, size_t n, void* dst);

/* Debug: with SKV_TRACE=1 in the environment every decode launch of `b` records, per
 * warp, {start, after the dependent-launch wait, end} (globaltimer ns) and
 * tiles<<32 | items; this copies the last launch's records (4 u64 each) to `host`
 * (*n = records).  *n = 0 when tracing is off. */
skv_status skv_debug_decode_trace(skv_pool* p, skv_batch* b, uint64_t* host, size_t cap, size_t* n);
uint64_t skv_kernel_launches(const skv_pool* p);

#ifdef __cplusplus
}
#endif
#endif /* SEAKV_H_ */

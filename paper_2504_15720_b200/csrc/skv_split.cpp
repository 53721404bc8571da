// skv_split.cpp — the split scheme on the GPU: the reference's
// alternative to merged blocks, where every native block of a request is split into
// per-(layer, kv head) blocks, each with its own block-table entry
// (SplitCacheCounter, kv_cache.hpp:277-348).
//
// Storage is an array of 8 KiB split blocks (K and V of 16 tokens of one (layer, kv
// head)), handed out from a free-id stack; a request's tables are
// [layer][kv head][native block] rows.  The accounting (entries, reads/writes,
// fragmentation) follows SplitCacheCounter exactly.  The data path reuses the unified
// decode machinery through an allocator-only registry pool (request ids, device token
// counts, batches) whose kernels address the split tables while a SplitView is
// installed — so merged and split run the same decode kernel and differ only in
// table layout, table size, block placement and allocation work.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/seakv.h"
#include "skv_internal.h"

namespace {

struct SplitReq {
  int model = 0;
  long long blocks = 0;  // native blocks covered
  long long tokens = 0;
};

struct SplitModel {
  int L, H;             // layers, kv heads per rank (physical blocks and table rows)
  int H_full;           // ModelSpec::num_heads: SplitCacheCounter's split factor ignores tp (:320-323)
  double kv_per_token;  // ModelSpec::kv_bytes_per_token (cost_model.hpp:37-39)
};

constexpr long long kSplitBytes = 2LL * 16 * 128 * 2;  // K + V of 16 tokens x 128 dims

}  // namespace

struct skv_split {
  skv_pool* reg = nullptr;  // request registry + batches (allocator only, no KV storage)
  int device = 0, dtype = 0, M = 0, Lmax = 0, Hmax = 0, cap = 0, R = 0;
  std::vector<SplitModel> models;
  size_t nblocks = 0;
  long long top = 0;  // free-stack depth
  int32_t* d_stack = nullptr;
  int2* d_table = nullptr;
  char* storage = nullptr;
  skv::SplitView view{};
  std::vector<skv::SplitOp> ops;
  skv::SplitOp* d_ops = nullptr;
  skv::SplitOp* h_ops = nullptr;  // pinned, mapped staging (read by an SM copy, see flush())
  cudaEvent_t stage_ev = nullptr;
  size_t d_ops_cap = 0;
  // SplitCacheCounter state (kv_cache.hpp:281-348)
  std::unordered_map<uint64_t, SplitReq> live;
  uint64_t entries = 0, peak = 0, rw = 0;
  double frag = 0.0;
  uint64_t launches = 0;
  std::string err;
};

namespace {

skv_status sfail(skv_split* s, skv_status st, const std::string& m) {
  if (s) s->err = m;
  return st;
}

#define SPLIT_CUDA(s, call)                                                              \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) return sfail(s, SKV_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// the ops queued in s->ops as one claim (kind 0) or release (kind 1) launch
skv_status launch_ops(skv_split* s, int kind) {
  if (s->ops.empty()) return SKV_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != s->device) cudaSetDevice(s->device);
  cudaStream_t st = static_cast<cudaStream_t>(skv_get_stream(s->reg));
  long long total = 0;
  for (auto& o : s->ops) {
    o.cbeg = (int)total;
    total += (long long)o.nblk * o.L * o.H;
  }
  if (total > 0x7fffffffLL) return sfail(s, SKV_ERR_ARG, "split: too many claims in one call");
  if (s->stage_ev) SPLIT_CUDA(s, cudaEventSynchronize(s->stage_ev));  // staging buffer reuse
  if (s->ops.size() > s->d_ops_cap) {
    SPLIT_CUDA(s, cudaStreamSynchronize(st));
    if (s->d_ops) cudaFree(s->d_ops);
    if (s->h_ops) cudaFreeHost(s->h_ops);
    s->d_ops_cap = std::max<size_t>(s->ops.size() * 2, 256);
    SPLIT_CUDA(s, cudaMalloc(&s->d_ops, s->d_ops_cap * sizeof(skv::SplitOp)));
    SPLIT_CUDA(s, cudaHostAlloc(&s->h_ops, s->d_ops_cap * sizeof(skv::SplitOp), cudaHostAllocMapped));
  }
  // the registry's allocator work (ids, token counts) goes first on the same stream
  skv_status rs = skv_flush(s->reg, nullptr);
  if (rs) return sfail(s, rs, std::string("split: registry flush: ") + skv_last_error(s->reg));
  std::memcpy(s->h_ops, s->ops.data(), s->ops.size() * sizeof(skv::SplitOp));
  skv::launch_stage_copy(s->d_ops, s->h_ops, s->ops.size() * sizeof(skv::SplitOp), st);
  if (kind == 0)
    skv::launch_split_claim(s->d_ops, (int)s->ops.size(), total, s->d_stack, s->d_table, s->Lmax, s->Hmax, s->cap, st);
  else
    skv::launch_split_release(s->d_ops, (int)s->ops.size(), total, s->d_stack, s->d_table, s->Lmax, s->Hmax, s->cap,
                              st);
  s->launches++;
  SPLIT_CUDA(s, cudaGetLastError());
  if (!s->stage_ev) SPLIT_CUDA(s, cudaEventCreateWithFlags(&s->stage_ev, cudaEventDisableTiming));
  SPLIT_CUDA(s, cudaEventRecord(s->stage_ev, st));
  s->ops.clear();
  if (dev != s->device) cudaSetDevice(dev);
  return SKV_OK;
}

double token_waste(const skv_split* s) {  // SplitCacheCounter::total_token_waste (:337-344)
  double w = 0.0;
  for (const auto& kv : s->live)
    w += (double)(kv.second.blocks * 16 - kv.second.tokens) * s->models[kv.second.model].kv_per_token;
  return w;
}

}  // namespace

extern "C" {

skv_status skv_split_create(const skv_model_desc* models, int32_t n, int32_t tpb, int32_t tp, size_t blocks,
                            const skv_pool_opts* opts, skv_split** out) {
  *out = nullptr;
  if (tpb != 16) return SKV_ERR_ARG;
  if (blocks == 0 || blocks > 0x7fffffffULL) return SKV_ERR_ARG;
  skv_pool_opts o;
  skv_default_opts(&o);
  if (opts) o = *opts;
  auto s = new skv_split();
  s->device = o.device;
  s->dtype = o.dtype;
  s->M = n;
  for (int i = 0; i < n; ++i) {
    const skv_model_desc& m = models[i];
    if (m.head_dim != 128 || m.dtype_bytes != 2 || tp < 1 || m.num_heads % tp) {
      delete s;
      return SKV_ERR_CONFIG;
    }
    s->models.push_back({m.num_layers, m.num_heads / tp, m.num_heads,
                         2.0 * m.num_layers * m.num_heads * m.head_dim * m.dtype_bytes});
    s->Lmax = std::max(s->Lmax, m.num_layers);
    s->Hmax = std::max(s->Hmax, m.num_heads / tp);
  }
  // registry: same models, allocator only; its merged capacity never binds before ours
  skv_pool_opts ro = o;
  ro.allocate_storage = 0;
  ro.phys_layers = 0;
  skv_status st = skv_pool_create(models, n, tpb, tp, blocks, &ro, &s->reg);
  if (st) {
    delete s;
    return st;
  }
  s->cap = o.max_blocks_per_request > 0 ? o.max_blocks_per_request : 4096;
  s->R = o.max_requests > 0 ? o.max_requests : 4096;
  s->nblocks = blocks;
  s->top = (long long)blocks;
  cudaSetDevice(s->device);
  std::vector<int32_t> stack(blocks);
  for (size_t i = 0; i < blocks; ++i) stack[i] = (int32_t)(blocks - 1 - i);  // pops hand out 0, 1, 2, ...
  const size_t tbytes = (size_t)s->R * s->Lmax * s->Hmax * s->cap * sizeof(int2);
  if (cudaMalloc(&s->d_stack, blocks * sizeof(int32_t)) != cudaSuccess ||
      cudaMalloc(&s->d_table, tbytes) != cudaSuccess ||
      cudaMalloc(&s->storage, blocks * (size_t)kSplitBytes) != cudaSuccess ||
      cudaMemcpy(s->d_stack, stack.data(), blocks * sizeof(int32_t), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(s->d_table, 0, tbytes) != cudaSuccess) {
    skv_split_destroy(s);
    return SKV_ERR_CUDA;
  }
  s->view = {s->d_table, s->storage, s->Lmax, s->Hmax, s->cap};
  *out = s;
  return SKV_OK;
}

void skv_split_destroy(skv_split* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  cudaDeviceSynchronize();
  for (void* q : {(void*)s->d_stack, (void*)s->d_table, (void*)s->storage, (void*)s->d_ops})
    if (q) cudaFree(q);
  if (s->h_ops) cudaFreeHost(s->h_ops);
  if (s->stage_ev) cudaEventDestroy(s->stage_ev);
  if (s->reg) skv_pool_destroy(s->reg);
  delete s;
}

const char* skv_split_last_error(const skv_split* s) { return s ? s->err.c_str() : ""; }
skv_pool* skv_split_registry(skv_split* s) { return s->reg; }
size_t skv_split_free_blocks(const skv_split* s) { return (size_t)s->top; }
size_t skv_split_pool_size(const skv_split* s) { return s->nblocks; }
uint64_t skv_split_kernel_launches(const skv_split* s) { return s->launches; }

skv_status skv_split_grow(skv_split* s, const uint64_t* ids, const int32_t* models, const int64_t* tokens, int32_t n,
                          int32_t* granted) {
  // Validate every op before any state changes: an early error return must not leave
  // queued claims behind (they would be replayed by the next launch_ops as releases).
  {
    std::unordered_map<uint64_t, int> seen;  // model of ids first seen in this call
    for (int i = 0; i < n; ++i) {
      const int m = models[i];
      if (m < 0 || m >= s->M) return sfail(s, SKV_ERR_ARG, "split grow: model index out of range");
      if (tokens[i] < 0) return sfail(s, SKV_ERR_VALIDATION, "split grow: negative tokens");
      auto it = s->live.find(ids[i]);
      const int prev = it != s->live.end() ? it->second.model : (seen.count(ids[i]) ? seen[ids[i]] : m);
      if (prev != m) return sfail(s, SKV_ERR_LOGIC, "split grow: model changed");
      seen[ids[i]] = m;
      if (it == s->live.end() && s->live.size() + seen.size() > (size_t)s->R)
        return sfail(s, SKV_ERR_ARG, "split grow: more live requests than max_requests");
      if ((tokens[i] + 15) / 16 > s->cap)
        return sfail(s, SKV_ERR_ARG, "split grow: request exceeds max_blocks_per_request");
    }
  }
  for (int i = 0; i < n; ++i) {
    const int m = models[i];
    auto it = s->live.find(ids[i]);
    const long long have = it == s->live.end() ? 0 : it->second.blocks;
    const long long need = (tokens[i] + 15) / 16;
    const SplitModel& sm = s->models[m];
    const long long claims = need > have ? (need - have) * sm.L * sm.H : 0;
    if (claims > s->top) {  // all-or-nothing, no change (as kv_cache.hpp:110-112)
      if (granted) granted[i] = 0;
      continue;
    }
    skv_status st = skv_try_allocate(s->reg, ids[i], m, tokens[i]);
    if (st != SKV_OK) {  // registry capacity: keep what was already granted consistent on the GPU
      const std::string msg = std::string("split grow: registry: ") + skv_last_error(s->reg);
      launch_ops(s, 0);
      return sfail(s, st == SKV_CACHE_FULL ? SKV_ERR_LOGIC : st, msg);
    }
    if (granted) granted[i] = 1;
    if (claims > 0) {
      skv::SplitOp op{};
      op.handle = skv_internal_handle(s->reg, ids[i]);
      op.L = sm.L;
      op.H = sm.H;
      op.blk0 = (int)have;
      op.nblk = (int)(need - have);
      op.base = (int)(s->top - claims);
      s->top -= claims;
      s->ops.push_back(op);
    }
    // SplitCacheCounter::grow (kv_cache.hpp:286-302)
    SplitReq& r = s->live[ids[i]];
    r.model = m;
    const uint64_t factor = (uint64_t)sm.L * sm.H_full;
    if (need > r.blocks) {
      s->entries += (uint64_t)(need - r.blocks) * factor;
      r.blocks = need;
    }
    if (tokens[i] > r.tokens) {
      s->rw += (uint64_t)(tokens[i] - r.tokens) * factor;
      r.tokens = tokens[i];
    }
    s->peak = std::max(s->peak, s->entries);
    s->frag = std::max(s->frag, token_waste(s));
  }
  return launch_ops(s, 0);
}

skv_status skv_split_free(skv_split* s, const uint64_t* ids, int32_t n) {
  {  // validate first (unknown or repeated id -> error, nothing changed)
    std::unordered_map<uint64_t, int> seen;
    for (int i = 0; i < n; ++i)
      if (!s->live.count(ids[i]) || seen[ids[i]]++)
        return sfail(s, SKV_ERR_LOGIC, "split free: unknown request");
  }
  for (int i = 0; i < n; ++i) {  // SplitCacheCounter::free (kv_cache.hpp:304-309)
    auto it = s->live.find(ids[i]);
    if (it == s->live.end()) return sfail(s, SKV_ERR_LOGIC, "split free: unknown request");
    const SplitModel& sm = s->models[it->second.model];
    const long long cnt = it->second.blocks * sm.L * sm.H;
    if (cnt > 0) {
      skv::SplitOp op{};
      op.handle = skv_internal_handle(s->reg, ids[i]);
      op.L = sm.L;
      op.H = sm.H;
      op.blk0 = 0;
      op.nblk = (int)it->second.blocks;
      op.base = (int)s->top;
      s->top += cnt;
      s->ops.push_back(op);
    }
    s->entries -= (uint64_t)it->second.blocks * sm.L * sm.H_full;
    s->live.erase(it);
  }
  // ids go back to the stack before the registry recycles the request handles
  skv_status st = launch_ops(s, 1);
  if (st) return st;
  for (int i = 0; i < n; ++i) {
    st = skv_free_request(s->reg, ids[i]);
    if (st) return sfail(s, st, std::string("split free: registry: ") + skv_last_error(s->reg));
  }
  return SKV_OK;
}

skv_status skv_split_stats(const skv_split* s, skv_cache_stats* out) {  // SplitCacheCounter::stats (:311-318)
  out->block_table_entries = s->peak;
  out->native_reads_writes = s->rw;
  out->internal_fragmentation_bytes = s->frag;
  out->peak_utilization = 0.0;
  return SKV_OK;
}

uint64_t skv_split_table_entries(const skv_split* s) { return s->entries; }

skv_status skv_split_synth_fill(skv_split* s, uint64_t seed, float amp, void* stream) {
  cudaSetDevice(s->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : static_cast<cudaStream_t>(skv_get_stream(s->reg));
  skv::launch_synth_fill(s->storage, s->nblocks * (size_t)kSplitBytes, s->dtype, seed, amp, st);
  s->launches++;
  SPLIT_CUDA(s, cudaGetLastError());
  return SKV_OK;
}

skv_status skv_split_decode(skv_split* s, skv_batch* b, const skv_decode_args* a, void* stream) {
  skv_internal_set_split(s->reg, &s->view);
  const skv_status st = skv_decode_attention(s->reg, b, a, stream);
  skv_internal_set_split(s->reg, nullptr);
  if (st) return sfail(s, st, std::string("split decode: ") + skv_last_error(s->reg));
  return SKV_OK;
}

skv_status skv_split_append(skv_split* s, skv_batch* b, const skv_append_args* a, void* stream) {
  skv_internal_set_split(s->reg, &s->view);
  const skv_status st = skv_append_kv(s->reg, b, a, stream);
  skv_internal_set_split(s->reg, nullptr);
  if (st) return sfail(s, st, std::string("split append: ") + skv_last_error(s->reg));
  return SKV_OK;
}

skv_status skv_split_block_ids(skv_split* s, uint64_t id, int32_t layer, int32_t head, int32_t* out, size_t cap,
                               size_t* n) {
  *n = 0;
  auto it = s->live.find(id);
  if (it == s->live.end()) return sfail(s, SKV_ERR_LOGIC, "split block_ids: unknown request");
  const SplitModel& sm = s->models[it->second.model];
  if (layer < 0 || layer >= sm.L || head < 0 || head >= sm.H) return sfail(s, SKV_ERR_ARG, "split block_ids: range");
  const size_t nb = (size_t)it->second.blocks;
  if (nb > cap) return sfail(s, SKV_ERR_ARG, "split block_ids: buffer too small");
  cudaSetDevice(s->device);
  SPLIT_CUDA(s, cudaStreamSynchronize(static_cast<cudaStream_t>(skv_get_stream(s->reg))));
  std::vector<int2> row(nb);
  const int h = skv_internal_handle(s->reg, id);
  SPLIT_CUDA(s, cudaMemcpy(row.data(), s->d_table + (((size_t)h * s->Lmax + layer) * s->Hmax + head) * s->cap,
                           nb * sizeof(int2), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < nb; ++i) out[i] = row[i].x;
  *n = nb;
  return SKV_OK;
}

skv_status skv_split_read_blocks(skv_split* s, const int32_t* ids, size_t n, void* dst) {
  cudaSetDevice(s->device);
  SPLIT_CUDA(s, cudaDeviceSynchronize());
  for (size_t i = 0; i < n; ++i) {
    if (ids[i] < 0 || (size_t)ids[i] >= s->nblocks) return sfail(s, SKV_ERR_ARG, "split read_blocks: id");
    SPLIT_CUDA(s, cudaMemcpy(static_cast<char*>(dst) + i * kSplitBytes, s->storage + (size_t)ids[i] * kSplitBytes,
                             kSplitBytes, cudaMemcpyDeviceToHost));
  }
  return SKV_OK;
}

}  // extern "C"

// unified_kv_cache.hpp — C++ drop-in for seasim::UnifiedKvCache backed by the GPU.
//
// Same namespace, class name, member signatures, exception types and return
// semantics as /root/reference/proj/include/seasim/kv_cache.hpp:16-369, so code
// written against the reference (its simulator, its kv_cache_test.cpp) compiles
// unchanged; every call forwards through the C-ABI in include/seakv.h to
// libseakv.so, where the block assignment runs on the B200.
//
//   reference                          here
//   ---------------------------------  -------------------------------------------
//   native_block_bytes   :17-22        skv_native_block_bytes
//   plan_merged_shape    :26-33        skv_plan_merged_shape
//   UnifiedKvCache(...)  :50-66        skv_pool_create (move-only owner of the pool)
//   try_allocate         :104-123      skv_try_allocate (CacheFull -> false)
//   free_request         :126-134      skv_free_request
//   block_table          :144-148      skv_block_table (const& valid until next call
//                                      that mutates the cache, as in the reference)
//   compare_schemes      :352-369      GPU merged scheme + host SplitCacheCounter
//
// Request ids cross the C-ABI as id+1, so id 0 — which the reference uses as its
// empty-slot sentinel and which its simulator hands out (simulation.hpp:169-172) —
// is a normal request here (the reference's Q2 aliasing for id 0 is not reproduced;
// UINT64_MAX is the one id that cannot be represented).  The object is move-only (it
// owns device memory), as the simulator's Engine already requires (simulation.hpp:219).
//
// Define SEAKV_USE_REFERENCE_TYPES before including this header to take ModelSpec,
// kGiB, the exception types and detail::Rng from the reference's own common.hpp /
// cost_model.hpp (e.g. when building the reference simulator against the GPU cache,
// tests/shim_sim/seasim/kv_cache.hpp).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <utility>
#include <vector>

#include "seakv.h"

namespace seasim {

#ifndef SEAKV_USE_REFERENCE_TYPES
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ParseError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ValidationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InfeasibleError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline constexpr double kGiB = 1073741824.0;

// The fields of the reference ModelSpec (cost_model.hpp:19-40) plus num_q_heads.
struct ModelSpec {
  std::string model_id;
  int num_layers = 0;
  int num_heads = 0;  // KV heads; sizes the native block
  int head_dim = 0;
  int dtype_bytes = 0;
  double weight_bytes = 0.0;
  int min_tp = 1;
  int num_q_heads = 0;  // GQA extension (0 = num_heads)

  double kv_bytes_per_token() const { return 2.0 * num_layers * num_heads * head_dim * dtype_bytes; }
};
#endif  // SEAKV_USE_REFERENCE_TYPES

struct CacheStats {
  std::uint64_t block_table_entries = 0;
  std::uint64_t native_reads_writes = 0;
  double internal_fragmentation_bytes = 0.0;
  double peak_utilization = 0.0;
};

namespace seakv_detail {

template <typename M, typename = void>
struct q_heads_of {
  static int get(const M&) { return 0; }  // reference ModelSpec: no GQA field -> MHA
};
template <typename M>
struct q_heads_of<M, std::void_t<decltype(std::declval<const M&>().num_q_heads)>> {
  static int get(const M& m) { return m.num_q_heads; }
};

inline skv_model_desc to_desc(const ModelSpec& m) {
  skv_model_desc d;
  d.model_id = m.model_id.c_str();
  d.num_layers = m.num_layers;
  d.num_heads = m.num_heads;
  d.num_q_heads = q_heads_of<ModelSpec>::get(m);
  d.head_dim = m.head_dim;
  d.dtype_bytes = m.dtype_bytes;
  return d;
}

// ids cross the ABI shifted by one (0 is the ABI's reserved sentinel)
inline std::uint64_t abi_id(std::uint64_t id) { return id + 1; }

[[noreturn]] inline void raise(skv_status st, const char* msg) {
  const std::string what = msg ? msg : "seakv error";
  switch (st) {
    case SKV_ERR_CONFIG: throw ConfigError(what);
    case SKV_ERR_VALIDATION: throw ValidationError(what);
    case SKV_ERR_LOGIC: throw std::logic_error(what);
    default: throw std::runtime_error("seakv: " + what);
  }
}

inline int check(skv_status st, const skv_pool* p) {
  if (st < 0) raise(st, skv_last_error(p));
  return st;
}

inline int default_device() {
  const char* e = std::getenv("SEAKV_DEVICE");
  return e ? std::atoi(e) : 0;
}

}  // namespace seakv_detail

inline double native_block_bytes(const ModelSpec& model, int tokens_per_block, int tp_size) {
  const skv_model_desc d = seakv_detail::to_desc(model);
  double out = 0.0;
  seakv_detail::check(skv_native_block_bytes(&d, tokens_per_block, tp_size, &out), nullptr);
  return out;
}

inline double plan_merged_shape(const std::vector<ModelSpec>& models, int tokens_per_block, int tp_size) {
  std::vector<skv_model_desc> d;
  for (const auto& m : models) d.push_back(seakv_detail::to_desc(m));
  double out = 0.0;
  seakv_detail::check(skv_plan_merged_shape(d.data(), static_cast<int32_t>(d.size()), tokens_per_block,
                                            tp_size, &out),
                      nullptr);
  return out;
}

class UnifiedKvCache {
 public:
  UnifiedKvCache() = default;

  UnifiedKvCache(std::vector<ModelSpec> models, int tokens_per_block, int tp_size, std::size_t pool_blocks)
      : models_(std::move(models)) {
    std::vector<skv_model_desc> d;
    for (const auto& m : models_) d.push_back(seakv_detail::to_desc(m));
    skv_pool_opts opts;
    skv_default_opts(&opts);
    // max_requests / max_blocks_per_request are only initial capacities: the device request
    // table grows on demand, so like the reference there is no limit on live requests or on a
    // request's length other than the pool itself (kv_cache.hpp:104-123).
    opts.device = seakv_detail::default_device();
    skv_pool* p = nullptr;
    seakv_detail::check(skv_pool_create(d.data(), static_cast<int32_t>(d.size()), tokens_per_block, tp_size,
                                        pool_blocks, &opts, &p),
                        nullptr);
    pool_ = p;
  }

  UnifiedKvCache(const UnifiedKvCache&) = delete;
  UnifiedKvCache& operator=(const UnifiedKvCache&) = delete;
  UnifiedKvCache(UnifiedKvCache&& o) noexcept { *this = std::move(o); }
  UnifiedKvCache& operator=(UnifiedKvCache&& o) noexcept {
    if (this != &o) {
      reset();
      pool_ = o.pool_;
      o.pool_ = nullptr;
      models_ = std::move(o.models_);
      tables_ = std::move(o.tables_);
    }
    return *this;
  }
  ~UnifiedKvCache() { reset(); }

  int model_index(const std::string& model_id) const {
    int32_t m = -1;
    seakv_detail::check(skv_model_index(pool_, model_id.c_str(), &m), pool_);
    return m;
  }
  int sub_slots_per_merged(int model_idx) const { return skv_sub_slots_per_merged(pool_, model_idx); }
  double merged_block_bytes() const { return skv_merged_block_bytes(pool_); }
  std::size_t pool_size() const { return skv_pool_size(pool_); }
  std::size_t free_blocks() const { return skv_free_blocks(pool_); }
  std::size_t allocated_blocks() const { return skv_allocated_blocks(pool_); }
  int tokens_per_block() const { return skv_tokens_per_block(pool_); }
  std::size_t native_blocks_for(long tokens) const { return skv_native_blocks_for(pool_, tokens); }
  bool registered(std::uint64_t request_id) const { return skv_registered(pool_, seakv_detail::abi_id(request_id)) != 0; }
  std::size_t available_slots(int model_idx) const { return skv_available_slots(pool_, model_idx); }

  bool can_grow_to(std::uint64_t request_id, int model_idx, long tokens_needed) const {
    int32_t out = 0;
    seakv_detail::check(skv_can_grow_to(pool_, seakv_detail::abi_id(request_id), model_idx, tokens_needed, &out), pool_);
    return out != 0;
  }

  bool try_allocate(std::uint64_t request_id, int model_idx, long tokens_needed) {
    return seakv_detail::check(skv_try_allocate(pool_, seakv_detail::abi_id(request_id), model_idx, tokens_needed), pool_) == SKV_OK;
  }

  void free_request(std::uint64_t request_id) {
    seakv_detail::check(skv_free_request(pool_, seakv_detail::abi_id(request_id)), pool_);
    tables_.erase(request_id);
  }

  void record_context_read(std::uint64_t request_id) {
    seakv_detail::check(skv_record_context_read(pool_, seakv_detail::abi_id(request_id)), pool_);
  }

  const std::vector<std::pair<int, int>>& block_table(std::uint64_t request_id) const {
    size_t n = 0;
    seakv_detail::check(skv_block_table(pool_, seakv_detail::abi_id(request_id), nullptr, 0, &n), pool_);
    std::vector<int32_t> raw(2 * n);
    if (n) seakv_detail::check(skv_block_table(pool_, seakv_detail::abi_id(request_id), raw.data(), n, &n), pool_);
    auto& t = tables_[request_id];
    t.resize(n);
    for (size_t i = 0; i < n; ++i) t[i] = {raw[2 * i], raw[2 * i + 1]};
    return t;
  }

  std::uint64_t owner_of(int block, int slot) const {
    uint64_t o = 0;
    seakv_detail::check(skv_owner_of(pool_, block, slot, &o), pool_);
    return o ? o - 1 : 0;  // 0 = empty, as the reference reports it
  }

  std::size_t table_entries() const { return skv_table_entries(pool_); }
  double fragmentation_bytes() const { return skv_fragmentation_bytes(pool_); }

  CacheStats stats() const {
    skv_cache_stats s{};
    seakv_detail::check(skv_stats(pool_, &s), pool_);
    CacheStats c;
    c.block_table_entries = s.block_table_entries;
    c.native_reads_writes = s.native_reads_writes;
    c.internal_fragmentation_bytes = s.internal_fragmentation_bytes;
    c.peak_utilization = s.peak_utilization;
    return c;
  }

  // Access to the GPU pool for the data path (append / decode / prefill).
  skv_pool* pool() const { return pool_; }

 private:
  void reset() {
    if (pool_) skv_pool_destroy(pool_);
    pool_ = nullptr;
  }

  skv_pool* pool_ = nullptr;
  std::vector<ModelSpec> models_;
  mutable std::unordered_map<std::uint64_t, std::vector<std::pair<int, int>>> tables_;
};

// One step of a cache workload replay (kv_cache.hpp:270-275).
struct KvOp {
  enum class Kind { kGrow, kFree } kind = Kind::kGrow;
  std::uint64_t request_id = 0;
  int model_idx = 0;
  long tokens = 0;
};

// Split-scheme accounting (kv_cache.hpp:277-348): per-layer-per-head blocks, so a
// native block of model m costs L*H table entries and each token touches L*H blocks.
class SplitCacheCounter {
 public:
  explicit SplitCacheCounter(std::vector<ModelSpec> models, int tokens_per_block)
      : models_(std::move(models)), tpb_(tokens_per_block) {}

  void grow(std::uint64_t id, int model_idx, long tokens) {
    Req& r = live_[id];
    r.model = model_idx;
    const std::uint64_t per_block = cost(model_idx);
    const long blocks = (tokens + tpb_ - 1) / tpb_;
    if (blocks > r.blocks) {
      entries_ += static_cast<std::uint64_t>(blocks - r.blocks) * per_block;
      r.blocks = blocks;
    }
    if (tokens > r.tokens) {
      touches_ += static_cast<std::uint64_t>(tokens - r.tokens) * per_block;
      r.tokens = tokens;
    }
    if (entries_ > peak_) peak_ = entries_;
    double waste = 0.0;  // integer-valued: summation order is irrelevant
    for (const auto& kv : live_)
      waste += (static_cast<double>(kv.second.blocks) * tpb_ - kv.second.tokens) *
               models_[kv.second.model].kv_bytes_per_token();
    if (waste > frag_) frag_ = waste;
  }

  void free(std::uint64_t id) {
    auto it = live_.find(id);
    if (it == live_.end()) return;
    entries_ -= static_cast<std::uint64_t>(it->second.blocks) * cost(it->second.model);
    live_.erase(it);
  }

  CacheStats stats() const {
    CacheStats s;
    s.block_table_entries = peak_;
    s.native_reads_writes = touches_;
    s.internal_fragmentation_bytes = frag_;
    s.peak_utilization = 0.0;
    return s;
  }

 private:
  struct Req {
    int model = 0;
    long blocks = 0, tokens = 0;
  };
  std::uint64_t cost(int m) const {
    return static_cast<std::uint64_t>(models_[m].num_layers) * static_cast<std::uint64_t>(models_[m].num_heads);
  }
  std::vector<ModelSpec> models_;
  int tpb_;
  std::map<std::uint64_t, Req> live_;
  std::uint64_t entries_ = 0, peak_ = 0, touches_ = 0;
  double frag_ = 0.0;
};

inline std::pair<CacheStats, CacheStats> compare_schemes(const std::vector<ModelSpec>& models,
                                                         int tokens_per_block, int tp_size,
                                                         const std::vector<KvOp>& ops, std::size_t pool_blocks) {
  UnifiedKvCache merged(models, tokens_per_block, tp_size, pool_blocks);
  SplitCacheCounter split(models, tokens_per_block);
  for (const KvOp& op : ops) {
    if (op.kind == KvOp::Kind::kFree) {
      merged.free_request(op.request_id);
      split.free(op.request_id);
      continue;
    }
    if (!merged.try_allocate(op.request_id, op.model_idx, op.tokens))
      throw ValidationError("compare_schemes: pool too small for workload sample");
    split.grow(op.request_id, op.model_idx, op.tokens);
  }
  return {merged.stats(), split.stats()};
}

#ifndef SEAKV_USE_REFERENCE_TYPES
namespace detail {

// Counter-based SplitMix64 stream with the reference's draw functions
// (common.hpp:41-74), so seeded drivers replay identically on either backend.
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : s_(seed) {}
  std::uint64_t next_u64() {
    s_ += 0x9e3779b97f4a7c15ULL;
    std::uint64_t x = s_;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
  }
  double next_double() { return static_cast<double>(next_u64() >> 11) * (1.0 / 9007199254740992.0); }
  double next_open_double() { return 1.0 - next_double(); }
  std::uint64_t next_below(std::uint64_t bound) { return next_u64() % bound; }
  std::uint64_t fork_seed() { return next_u64(); }

 private:
  std::uint64_t s_;
};

}  // namespace detail
#endif  // SEAKV_USE_REFERENCE_TYPES

}  // namespace seasim

// ref_kv.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference allocator, compiled from the
// read-only tree: g++ -I/root/reference/proj/include (see oracle/Makefile).
// No reference source is copied; this file only includes the header and
// forwards calls, so the differ (tests/test_oracle_alloc.py) and bench.py's
// cpu_baseline can run the reference's own code path.  The build output goes
// to oracle/_ref/libref_kv.so (git-ignored, shipped to the GPU box as a
// prebuilt file because /root/reference does not exist there).
#include <cstdint>
#include <cstring>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "seasim/kv_cache.hpp"  // /root/reference/proj/include/seasim/kv_cache.hpp

namespace {
thread_local std::string g_err;

seasim::ModelSpec spec(int i, int layers, int heads, int head_dim, int dtype_bytes) {
  seasim::ModelSpec m;
  m.model_id = "m" + std::to_string(i);
  m.num_layers = layers;
  m.num_heads = heads;
  m.head_dim = head_dim;
  m.dtype_bytes = dtype_bytes;
  m.weight_bytes = 1.0 * seasim::kGiB;
  m.min_tp = 1;
  return m;
}
}  // namespace

extern "C" {

// status: 0 ok, 1 cache full, -1 ConfigError, -2 ValidationError, -3 logic_error
const char* ref_kv_last_error() { return g_err.c_str(); }

int ref_kv_native_block_bytes(int layers, int heads, int head_dim, int dtype_bytes, int tpb, int tp,
                              double* out) {
  try {
    *out = seasim::native_block_bytes(spec(0, layers, heads, head_dim, dtype_bytes), tpb, tp);
    return 0;
  } catch (const seasim::ConfigError& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_kv_plan_merged_shape(int n, const int* layers, const int* heads, const int* head_dim,
                             const int* dtype_bytes, int tpb, int tp, double* out) {
  std::vector<seasim::ModelSpec> ms;
  for (int i = 0; i < n; ++i) ms.push_back(spec(i, layers[i], heads[i], head_dim[i], dtype_bytes[i]));
  try {
    *out = seasim::plan_merged_shape(ms, tpb, tp);
    return 0;
  } catch (const seasim::ConfigError& e) {
    g_err = e.what();
    return -1;
  }
}

void* ref_kv_create(int n, const int* layers, const int* heads, const int* head_dim,
                    const int* dtype_bytes, int tpb, int tp, size_t pool, int* status) {
  std::vector<seasim::ModelSpec> ms;
  for (int i = 0; i < n; ++i) ms.push_back(spec(i, layers[i], heads[i], head_dim[i], dtype_bytes[i]));
  try {
    *status = 0;
    return new seasim::UnifiedKvCache(ms, tpb, tp, pool);
  } catch (const seasim::ConfigError& e) {
    g_err = e.what();
    *status = -1;
    return nullptr;
  }
}

void ref_kv_destroy(void* c) { delete static_cast<seasim::UnifiedKvCache*>(c); }

#define C static_cast<seasim::UnifiedKvCache*>(c)
#define CC static_cast<const seasim::UnifiedKvCache*>(c)

int ref_kv_sub_slots(void* c, int m) { return CC->sub_slots_per_merged(m); }
double ref_kv_merged_block_bytes(void* c) { return CC->merged_block_bytes(); }
size_t ref_kv_free_blocks(void* c) { return CC->free_blocks(); }
size_t ref_kv_allocated_blocks(void* c) { return CC->allocated_blocks(); }
size_t ref_kv_table_entries(void* c) { return CC->table_entries(); }
size_t ref_kv_available_slots(void* c, int m) { return CC->available_slots(m); }
int ref_kv_registered(void* c, uint64_t id) { return CC->registered(id) ? 1 : 0; }
int ref_kv_can_grow_to(void* c, uint64_t id, int m, long tokens) {
  return CC->can_grow_to(id, m, tokens) ? 1 : 0;
}
double ref_kv_fragmentation_bytes(void* c) { return CC->fragmentation_bytes(); }
uint64_t ref_kv_owner_of(void* c, int b, int s) { return CC->owner_of(b, s); }
void ref_kv_record_context_read(void* c, uint64_t id) { C->record_context_read(id); }

int ref_kv_try_allocate(void* c, uint64_t id, int m, long tokens) {
  try {
    return C->try_allocate(id, m, tokens) ? 0 : 1;
  } catch (const seasim::ValidationError& e) {
    g_err = e.what();
    return -2;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return -3;
  }
}

int ref_kv_free_request(void* c, uint64_t id) {
  try {
    C->free_request(id);
    return 0;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return -3;
  }
}

long ref_kv_block_table(void* c, uint64_t id, int32_t* pairs, size_t cap) {
  try {
    const auto& t = CC->block_table(id);
    for (size_t i = 0; i < t.size() && i < cap; ++i) {
      pairs[2 * i] = t[i].first;
      pairs[2 * i + 1] = t[i].second;
    }
    return static_cast<long>(t.size());
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return -3;
  }
}

void ref_kv_stats(void* c, uint64_t* entries, uint64_t* rw, double* frag, double* util) {
  const seasim::CacheStats s = CC->stats();
  *entries = s.block_table_entries;
  *rw = s.native_reads_writes;
  *frag = s.internal_fragmentation_bytes;
  *util = s.peak_utilization;
}

// Same op record as oracle/kv_alloc_oracle.c:skvo_op.
struct ref_op {
  int32_t kind, model;
  uint64_t id;
  int64_t tokens;
};

long ref_kv_replay(void* c, const ref_op* ops, size_t n) {
  long granted = 0;
  try {
    for (size_t i = 0; i < n; ++i) {
      if (ops[i].kind == 0) {
        if (C->try_allocate(ops[i].id, ops[i].model, static_cast<long>(ops[i].tokens))) ++granted;
      } else {
        C->free_request(ops[i].id);
      }
    }
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
  return granted;
}

// compare_schemes (kv_cache.hpp:352-369): out[0..3] merged stats, out[4..7] split stats
int ref_kv_compare_schemes(int n, const int* layers, const int* heads, const int* head_dim,
                           const int* dtype_bytes, int tpb, int tp, const ref_op* ops, size_t nops,
                           size_t pool, double* out) {
  std::vector<seasim::ModelSpec> ms;
  for (int i = 0; i < n; ++i) ms.push_back(spec(i, layers[i], heads[i], head_dim[i], dtype_bytes[i]));
  std::vector<seasim::KvOp> kops;
  for (size_t i = 0; i < nops; ++i) {
    seasim::KvOp k;
    k.kind = ops[i].kind == 0 ? seasim::KvOp::Kind::kGrow : seasim::KvOp::Kind::kFree;
    k.request_id = ops[i].id;
    k.model_idx = ops[i].model;
    k.tokens = static_cast<long>(ops[i].tokens);
    kops.push_back(k);
  }
  try {
    auto [a, b] = seasim::compare_schemes(ms, tpb, tp, kops, pool);
    out[0] = static_cast<double>(a.block_table_entries);
    out[1] = static_cast<double>(a.native_reads_writes);
    out[2] = a.internal_fragmentation_bytes;
    out[3] = a.peak_utilization;
    out[4] = static_cast<double>(b.block_table_entries);
    out[5] = static_cast<double>(b.native_reads_writes);
    out[6] = b.internal_fragmentation_bytes;
    out[7] = b.peak_utilization;
    return 0;
  } catch (const seasim::ValidationError& e) {
    g_err = e.what();
    return -2;
  } catch (const seasim::ConfigError& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"

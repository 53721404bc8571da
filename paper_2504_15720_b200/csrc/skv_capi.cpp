// skv_capi.cpp — host runtime behind include/seakv.h.
//
// Split of responsibilities:
//  * The HOST keeps an exact integer mirror of everything try_allocate's return
//    value and CacheStats depend on — per-request (model, tokens, table length),
//    per-model open-slot counts, the free-block count and the fragmentation
//    terms — so `try_allocate` answers synchronously, without a device round trip,
//    with the reference's semantics (kv_cache.hpp:104-123).  All reference doubles
//    are integer-valued (< 2^53) and are carried as int64, so they are bit-exact.
//  * The GPU owns the canonical block state and decides WHICH merged block and
//    sub-slot every claim gets (skv_alloc.cu), writes the device block tables the
//    attention kernels read, and executes frees.  After a free run the host only
//    needs the number of merged blocks each model emptied (E_m), read back once
//    before the next admission decision.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/seakv.h"
#include "skv_internal.h"

namespace {

thread_local std::string g_tls_err;

struct ModelInfo {
  std::string id;
  int L, Hkv, Hq, d, e;       // per-rank head counts
  long long native;           // native block bytes (kv_cache.hpp:17-22), exact
  int sub;                    // sub_slots_ (kv_cache.hpp:62)
  int phys_L;                 // physical layers stored per native block
  long long layer_stride, head_stride, kv_stride, native_stride;
};

struct ReqHost {
  uint64_t id = 0;
  int model = -1;
  long long tokens = 0;
  int nslots = 0;
  bool live = false;
};

struct Run {
  int kind;  // 0 grow, 1 free
  size_t begin, end;
};

struct FreeResult {
  int slot;
  std::vector<long long> R;
  cudaEvent_t ev;
};

constexpr int kResultSlots = 64;

inline long long ceil_div_ll(long long a, long long b) { return (a + b - 1) / b; }
inline long long round_up(long long a, long long b) { return ceil_div_ll(a, b) * b; }

}  // namespace

struct skv_pool {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::vector<ModelInfo> models;
  int M = 0, tpb = 16, tp = 1, dtype = 0, phys_layers = 0;
  size_t P = 0;
  double merged = 0.0;
  long long merged_i = 0, merged_stride = 0;
  int maxsub = 1, cap = 0, R = 0;
  bool allocate_storage = false;

  // host mirror (exact)
  std::unordered_map<uint64_t, int> id2h;
  std::vector<ReqHost> req;
  std::vector<int> free_handles;
  std::vector<long long> open;
  long long free_count = 0;
  size_t cur_entries = 0;
  uint64_t peak_entries = 0, rw = 0;
  long long slot_frag = 0, token_waste = 0, peak_frag = 0, peak_used = 0;
  uint64_t token_epoch = 0;
  uint64_t free_epoch = 1;  // bumped by every free_request (batches re-check their ids after one)

  // queued device work
  std::vector<skv::GrowOp> grow_ops;
  std::vector<skv::FreeOp> free_ops;
  std::vector<Run> runs;
  std::vector<long long> run_claims;  // per grow run: total claims
  std::vector<FreeResult> pending;
  std::vector<long long> pending_R;   // R_m of the free run being queued
  int next_slot = 0;

  // device state
  skv::DevAlloc dev{};
  skv::AllocParams prm{};
  void* d_ops = nullptr;
  size_t d_ops_cap = 0;
  void* h_stage = nullptr;
  size_t h_stage_cap = 0;
  cudaEvent_t stage_ev = nullptr;
  skv::GrowScratch scr{};
  size_t scr_n = 0, scr_t = 0;
  int32_t* d_outE = nullptr;  // [kResultSlots][M]
  int32_t* h_outE = nullptr;  // pinned
  cudaEvent_t sync_ev = nullptr;

  void* storage = nullptr;
  size_t storage_bytes = 0;
  alignas(64) CUtensorMap kv_tmap;     // head_dim 128
  alignas(64) CUtensorMap kv_tmap64;   // head_dim 64 (K boxes)
  alignas(64) CUtensorMap kv_tmap64v;  // head_dim 64 (V boxes, SW64)
  alignas(64) CUtensorMap kv_tmap256;  // head_dim 256
  int has_tmap = 0;                    // bit d/64 set: descriptor for head_dim d encoded
  uint64_t launches = 0;
  const skv::SplitView* split = nullptr;  // data path addresses a split-scheme pool (skv_split.cpp)
  std::string err;
};

struct skv_batch {
  skv_pool* pool = nullptr;
  int ngroups = 0;
  std::vector<int> gmodel, gsize, gbegin;
  std::vector<uint64_t> ids;
  std::vector<int> handles;
  std::vector<int32_t> h_group;
  int32_t* d_handles = nullptr;
  int32_t* d_group = nullptr;
  size_t req_cap = 0;
  void* h_stage = nullptr;  // pinned upload staging
  cudaEvent_t stage_ev = nullptr;
  int nreq = 0;
  // decode plan workspace
  int4* d_items = nullptr;
  int4* d_itemx = nullptr;
  int* d_arrive = nullptr;      // [2][items_cap] arrival counters, two alternating sets
  size_t items_cap = 0;
  int* d_nitems = nullptr;
  int* d_counter = nullptr;     // [2][2] work counter + finished CTAs, two alternating sets
  int* d_rscr = nullptr;        // [5 * req_cap] plan scratch
  float* d_ws_o = nullptr;
  float2* d_ws_ml = nullptr;
  size_t slots_cap = 0;
  uint64_t plan_epoch = ~0ull;
  uint64_t launch_seq = 0;
  int plan_split = 0;
  long long last_sum_hkv = 0, last_ncut = 0;  // schedule of the last decode launch (skv_batch_plan_info)
  unsigned long long* d_trace = nullptr;  // SKV_TRACE=1: per-warp timing of the last decode
  size_t trace_n = 0;
  int32_t* d_qlen = nullptr;  // ragged append/prefill: per-request lengths [req_cap] and row offsets [req_cap]
  int32_t* h_qlen = nullptr;  // pinned staging of the same
  size_t qlen_cap = 0;
  cudaEvent_t qlen_ev = nullptr;
  std::vector<int32_t> qlen_last;  // lengths currently on the device (skip identical re-uploads)
  skv::GrowOp* d_gops = nullptr;   // device-generated decode-step grow ops [gops_cap]
  skv::GrowScratch gscr{};         // their placement scratch (per batch: stable for CUDA graphs)
  size_t gops_cap = 0, gscr_t = 0;
  uint64_t qlen_epoch = 0, launch_epoch = 1;  // launch_epoch bumps when the batch is re-pointed
  uint64_t checked_epoch = 0;  // pool free_epoch at the last full id check (check_batch)
};

namespace {

skv_status fail(skv_pool* p, skv_status st, const std::string& msg) {
  if (p) p->err = msg;
  else g_tls_err = msg;
  return st;
}

skv_status cuda_fail(skv_pool* p, cudaError_t e, const char* where) {
  return fail(p, SKV_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define SKV_CUDA(p, call)                                   \
  do {                                                      \
    cudaError_t e_ = (call);                                \
    if (e_ != cudaSuccess) return cuda_fail(p, e_, #call); \
  } while (0)

class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev_);
    if (prev_ != dev) cudaSetDevice(dev);
    dev_ = dev;
  }
  ~DeviceGuard() {
    if (prev_ != dev_) cudaSetDevice(prev_);
  }

 private:
  int prev_ = 0, dev_ = 0;
};

skv_status validate_model(const skv_model_desc& m, int tpb, int tp, long long* native) {
  std::string id = m.model_id ? m.model_id : "";
  if (m.num_layers < 1 || m.num_heads < 1 || m.head_dim < 1 || m.dtype_bytes < 1)
    return fail(nullptr, SKV_ERR_CONFIG, "model " + id + ": all counts must be >= 1");
  if (tp < 1 || m.num_heads % tp != 0)  // kv_cache.hpp:18-19
    return fail(nullptr, SKV_ERR_CONFIG, "model " + id + ": tp does not divide num_heads");
  const int hq = m.num_q_heads > 0 ? m.num_q_heads : m.num_heads;
  if (hq % m.num_heads != 0 || hq % tp != 0)
    return fail(nullptr, SKV_ERR_CONFIG, "model " + id + ": num_q_heads must be a multiple of num_heads");
  *native = (long long)tpb * m.num_layers * 2LL * (m.num_heads / tp) * m.head_dim * m.dtype_bytes;
  return SKV_OK;
}

long long entry_waste(const skv_pool* p, const ReqHost& r) {  // kv_cache.hpp:184-189
  if (r.model < 0) return 0;
  const long long per_token = p->models[r.model].native / p->tpb;
  return ((long long)r.nslots * p->tpb - r.tokens) * per_token;
}

void note_watermarks(skv_pool* p) {  // kv_cache.hpp:242-246
  p->peak_entries = std::max<uint64_t>(p->peak_entries, p->cur_entries);
  p->peak_used = std::max<long long>(p->peak_used, (long long)p->P - p->free_count);
  p->peak_frag = std::max<long long>(p->peak_frag, p->slot_frag + p->token_waste);
}

template <typename T>
skv_status dev_alloc(skv_pool* p, T** ptr, size_t count, bool zero = true) {
  if (count == 0) count = 1;
  SKV_CUDA(p, cudaMalloc(reinterpret_cast<void**>(ptr), count * sizeof(T)));
  if (zero) SKV_CUDA(p, cudaMemsetAsync(*ptr, 0, count * sizeof(T), p->stream));
  return SKV_OK;
}

skv_status ensure_scratch(skv_pool* p, size_t n, size_t t) {
  if (n <= p->scr_n && t <= p->scr_t) return SKV_OK;
  n = std::max<size_t>({n, p->scr_n * 2, 1024});
  t = std::max<size_t>({t, p->scr_t * 2, 4096});
  SKV_CUDA(p, cudaStreamSynchronize(p->stream));
  skv::GrowScratch& s = p->scr;
  for (void* q : {(void*)s.S, (void*)s.cbeg, (void*)s.nnew, (void*)s.base, (void*)s.nbfirst,
                  (void*)s.newblk, (void*)s.newrank, (void*)s.openlist})
    if (q) cudaFree(q);
  skv_status st;
  if ((st = dev_alloc(p, &s.S, n, false)) || (st = dev_alloc(p, &s.cbeg, n, false)) ||
      (st = dev_alloc(p, &s.nnew, n, false)) || (st = dev_alloc(p, &s.base, n, false)) ||
      (st = dev_alloc(p, &s.nbfirst, n, false)) || (st = dev_alloc(p, &s.newblk, t, false)) ||
      (st = dev_alloc(p, &s.newrank, t, false)) || (st = dev_alloc(p, &s.openlist, t, false)))
    return st;
  p->scr_n = n;
  p->scr_t = t;
  return SKV_OK;
}

// Pushes the queued allocator runs to the GPU on the pool stream.
skv_status flush(skv_pool* p) {
  if (p->runs.empty()) return SKV_OK;
  DeviceGuard g(p->device);
  const size_t gbytes = p->grow_ops.size() * sizeof(skv::GrowOp);
  const size_t fbytes = p->free_ops.size() * sizeof(skv::FreeOp);
  const size_t bytes = gbytes + fbytes;
  if (p->stage_ev) SKV_CUDA(p, cudaEventSynchronize(p->stage_ev));  // staging buffer reuse
  if (bytes > p->h_stage_cap) {
    if (p->h_stage) cudaFreeHost(p->h_stage);
    p->h_stage_cap = std::max(bytes * 2, (size_t)1 << 16);
    SKV_CUDA(p, cudaHostAlloc(&p->h_stage, p->h_stage_cap, cudaHostAllocMapped));
  }
  if (bytes > p->d_ops_cap) {
    SKV_CUDA(p, cudaStreamSynchronize(p->stream));
    if (p->d_ops) cudaFree(p->d_ops);
    p->d_ops_cap = std::max(bytes * 2, (size_t)1 << 16);
    SKV_CUDA(p, cudaMalloc(&p->d_ops, p->d_ops_cap));
  }
  size_t max_n = 0;
  long long max_t = 0;
  size_t gi = 0;
  for (const Run& r : p->runs)
    if (r.kind == 0) {
      max_n = std::max(max_n, r.end - r.begin);
      max_t = std::max(max_t, p->run_claims[gi++]);
    }
  gi = 0;
  if (max_n) {
    skv_status st = ensure_scratch(p, max_n, (size_t)max_t);
    if (st) return st;
  }
  std::memcpy(p->h_stage, p->grow_ops.data(), gbytes);
  std::memcpy(static_cast<char*>(p->h_stage) + gbytes, p->free_ops.data(), fbytes);
  skv::launch_stage_copy(p->d_ops, p->h_stage, bytes, p->stream);  // SM copy, not a copy engine
  p->launches++;
  const skv::GrowOp* dg = static_cast<const skv::GrowOp*>(p->d_ops);
  const skv::FreeOp* df = reinterpret_cast<const skv::FreeOp*>(static_cast<char*>(p->d_ops) + gbytes);
  size_t kf = 0;
  for (const Run& r : p->runs) kf += r.kind == 1;
  size_t fr = p->pending.size() - kf;  // results of the free runs queued since the last flush
  for (const Run& r : p->runs) {
    const int n = (int)(r.end - r.begin);
    if (r.kind == 0) {
      skv::launch_grow(p->dev, p->prm, dg + r.begin, n, p->run_claims[gi++], p->scr, p->stream);
      p->launches += 1;
    } else {
      FreeResult& fresult = p->pending[fr++];
      // emptied-block counts are written by the kernel straight into pinned host memory
      // (no copy-engine D2H that could queue behind a caller's bulk copies)
      skv::launch_free(p->dev, p->prm, df + r.begin, n, p->h_outE + fresult.slot * p->M, p->stream);
      p->launches += 2;
      if (!fresult.ev) SKV_CUDA(p, cudaEventCreateWithFlags(&fresult.ev, cudaEventDisableTiming));
      SKV_CUDA(p, cudaEventRecord(fresult.ev, p->stream));
    }
  }
  (void)fr;
  SKV_CUDA(p, cudaGetLastError());
  if (!p->stage_ev) SKV_CUDA(p, cudaEventCreateWithFlags(&p->stage_ev, cudaEventDisableTiming));
  SKV_CUDA(p, cudaEventRecord(p->stage_ev, p->stream));
  p->runs.clear();
  p->run_claims.clear();
  p->grow_ops.clear();
  p->free_ops.clear();
  return SKV_OK;
}

// Applies the emptied-block counts of completed free runs to the host mirror.
skv_status ensure_counters(skv_pool* p) {
  if (p->pending.empty()) return SKV_OK;
  skv_status st = flush(p);
  if (st) return st;
  DeviceGuard g(p->device);
  for (FreeResult& r : p->pending) {
    if (!r.ev) return fail(p, SKV_ERR_CUDA, "free result without event");
    SKV_CUDA(p, cudaEventSynchronize(r.ev));
    for (int m = 0; m < p->M; ++m) {
      const long long E = p->h_outE[r.slot * p->M + m];
      const long long Rm = r.R[m];
      const ModelInfo& mi = p->models[m];
      p->free_count += E;
      p->open[m] += Rm - E * mi.sub;  // release_slot, kv_cache.hpp:228-239
      p->slot_frag += (Rm - E) * mi.native - E * (p->merged_i - mi.native);
    }
    cudaEventDestroy(r.ev);
  }
  p->pending.clear();
  return SKV_OK;
}

void queue_grow(skv_pool* p, const skv::GrowOp& op) {
  if (p->runs.empty() || p->runs.back().kind != 0) {
    p->runs.push_back({0, p->grow_ops.size(), p->grow_ops.size()});
    p->run_claims.push_back(0);
  }
  p->grow_ops.push_back(op);
  p->runs.back().end = p->grow_ops.size();
  p->run_claims.back() += op.claims;
}

skv_status queue_free(skv_pool* p, const skv::FreeOp& op) {
  if (p->runs.empty() || p->runs.back().kind != 1) {
    if ((int)p->pending.size() >= kResultSlots - 1) {
      skv_status st = ensure_counters(p);
      if (st) return st;
    }
    FreeResult fr;
    fr.slot = p->next_slot;
    p->next_slot = (p->next_slot + 1) % kResultSlots;
    fr.R.assign(p->M, 0);
    fr.ev = nullptr;
    p->pending.push_back(fr);
    p->runs.push_back({1, p->free_ops.size(), p->free_ops.size()});
  }
  p->free_ops.push_back(op);
  p->runs.back().end = p->free_ops.size();
  p->pending.back().R[op.model] += op.nslots;
  return SKV_OK;
}

// Grows the device request table on demand.  The reference has no limit on live requests
// or on a request's length beyond the pool itself (kv_cache.hpp:104-123, simulation.hpp:248),
// so opts.max_requests / max_blocks_per_request are initial capacities: the handle count and
// the per-request row capacity double until `rows` handles / `cap` native blocks fit.  The
// copy is stream-ordered after all work already on the pool stream (queued claims are
// launched later against the new layout); CUDA graphs captured before a growth still point at
// the old table and must be re-captured.
skv_status grow_tables(skv_pool* p, long long rows, long long cap) {
  if (rows <= p->R && cap <= p->cap) return SKV_OK;
  if (cap > 0x7fffffffLL) return fail(p, SKV_ERR_ARG, "allocate: request longer than 2^31 native blocks");
  DeviceGuard g(p->device);
  int nR = p->R, ncap = p->cap;
  while (nR < rows) nR *= 2;
  while (ncap < cap) ncap = (int)std::min<long long>(2LL * ncap, 0x7fffffffLL);
  skv::DevAlloc& d = p->dev;
  int2* tab = nullptr;
  int32_t *ns = nullptr, *tk = nullptr, *md = nullptr;
  unsigned long long* ids = nullptr;
  SKV_CUDA(p, cudaMalloc(&ids, (size_t)nR * sizeof(unsigned long long)));
  SKV_CUDA(p, cudaMemsetAsync(ids, 0, (size_t)nR * sizeof(unsigned long long), p->stream));
  SKV_CUDA(p, cudaMemcpyAsync(ids, d.req_id, (size_t)p->R * sizeof(unsigned long long), cudaMemcpyDeviceToDevice,
                              p->stream));
  SKV_CUDA(p, cudaMalloc(&tab, (size_t)nR * ncap * sizeof(int2)));
  SKV_CUDA(p, cudaMalloc(&ns, (size_t)nR * sizeof(int32_t)));
  SKV_CUDA(p, cudaMalloc(&tk, (size_t)nR * sizeof(int32_t)));
  SKV_CUDA(p, cudaMalloc(&md, (size_t)nR * sizeof(int32_t)));
  SKV_CUDA(p, cudaMemcpy2DAsync(tab, (size_t)ncap * sizeof(int2), d.req_table, (size_t)p->cap * sizeof(int2),
                                (size_t)p->cap * sizeof(int2), (size_t)p->R, cudaMemcpyDeviceToDevice, p->stream));
  SKV_CUDA(p, cudaMemsetAsync(ns + p->R, 0, (size_t)(nR - p->R) * sizeof(int32_t), p->stream));
  SKV_CUDA(p, cudaMemsetAsync(tk + p->R, 0, (size_t)(nR - p->R) * sizeof(int32_t), p->stream));
  SKV_CUDA(p, cudaMemsetAsync(md + p->R, 0xff, (size_t)(nR - p->R) * sizeof(int32_t), p->stream));
  SKV_CUDA(p, cudaMemcpyAsync(ns, d.req_nslots, (size_t)p->R * sizeof(int32_t), cudaMemcpyDeviceToDevice, p->stream));
  SKV_CUDA(p, cudaMemcpyAsync(tk, d.req_tokens, (size_t)p->R * sizeof(int32_t), cudaMemcpyDeviceToDevice, p->stream));
  SKV_CUDA(p, cudaMemcpyAsync(md, d.req_model, (size_t)p->R * sizeof(int32_t), cudaMemcpyDeviceToDevice, p->stream));
  SKV_CUDA(p, cudaStreamSynchronize(p->stream));  // other streams may still read the old table
  SKV_CUDA(p, cudaDeviceSynchronize());
  cudaFree(d.req_table);
  cudaFree(d.req_nslots);
  cudaFree(d.req_tokens);
  cudaFree(d.req_model);
  cudaFree(d.req_id);
  d.req_id = ids;
  d.req_table = tab;
  d.req_nslots = ns;
  d.req_tokens = tk;
  d.req_model = md;
  p->req.resize(nR);
  for (int h = nR - 1; h >= p->R; --h) p->free_handles.push_back(h);  // lowest new handle on top
  p->R = nR;
  p->cap = ncap;
  p->prm.cap = ncap;
  return SKV_OK;
}

// try_allocate (kv_cache.hpp:104-123) on the host mirror; queues the claims (queue = false: the
// device generates the same op itself, skv_batch_grow_launch).
skv_status grow_handle_impl(skv_pool* p, int h, uint64_t id, int m, long long tokens, bool queue = true);

skv_status try_allocate_impl(skv_pool* p, uint64_t id, int m, long long tokens) {
  if (tokens < 0) return fail(p, SKV_ERR_VALIDATION, "allocate: negative tokens_needed");
  if (m < 0 || m >= p->M) return fail(p, SKV_ERR_ARG, "allocate: model index out of range");
  if (id == 0)  // id 0 is the reference's empty-slot sentinel
    return fail(p, SKV_ERR_VALIDATION, "allocate: request id 0 is reserved (empty-slot sentinel)");
  int h;
  auto it = p->id2h.find(id);
  if (it == p->id2h.end()) {  // registers on first touch (:106), even if it then fails (Q3)
    if (p->free_handles.empty()) {
      skv_status st = grow_tables(p, (long long)p->R + 1, p->cap);
      if (st) return st;
    }
    h = p->free_handles.back();
    p->free_handles.pop_back();
    p->id2h.emplace(id, h);
    ReqHost& r = p->req[h];
    r = ReqHost();
    r.id = id;
    r.live = true;
  } else {
    h = it->second;
  }
  return grow_handle_impl(p, h, id, m, tokens);
}

// try_allocate for a registered request whose handle is known (the batch path skips the
// id -> handle lookup)
skv_status grow_handle_impl(skv_pool* p, int h, uint64_t id, int m, long long tokens, bool queue) {
  ReqHost& r = p->req[h];
  if (r.nslots == 0) r.model = m;
  if (r.model != m) return fail(p, SKV_ERR_LOGIC, "allocate: request changed model");
  const long long need = ceil_div_ll(tokens, p->tpb);
  skv_status st = ensure_counters(p);
  if (st) return st;
  const ModelInfo& mi = p->models[m];
  long long c = 0;
  if (need > r.nslots) {
    c = need - r.nslots;
    const long long avail = p->open[m] + p->free_count * mi.sub;  // :88-90
    if (avail < c) return SKV_CACHE_FULL;                           // :110-112
    if (need > p->cap) {
      skv_status st = grow_tables(p, p->R, need);
      if (st) return st;
    }
  }
  const long long w0 = entry_waste(p, r);
  const int have = r.nslots;
  if (c > 0) {
    // claim_slot x c (:191-222): open slots first, then fresh blocks
    const long long from_open = std::min<long long>(c, p->open[m]);
    const long long rest = c - from_open;
    const long long nb = ceil_div_ll(rest, mi.sub);
    p->open[m] += -from_open + nb * mi.sub - rest;
    p->free_count -= nb;
    p->slot_frag += -from_open * mi.native + nb * (p->merged_i - mi.native) - (rest - nb) * mi.native;
    r.nslots += (int)c;
    p->cur_entries += (size_t)c;
  }
  const bool grew_tokens = tokens > r.tokens;
  if (grew_tokens) {
    p->rw += (uint64_t)(tokens - r.tokens);
    r.tokens = tokens;
  }
  // Net waste change incl. quirk Q1: every claim leaks native bytes into the waste term.
  p->token_waste += entry_waste(p, r) - w0 + c * mi.native;
  note_watermarks(p);
  if (c > 0 || grew_tokens) p->token_epoch++;
  if (queue && (c > 0 || grew_tokens)) {
    skv::GrowOp op{};
    op.handle = h;
    op.model = m;
    op.have = have;
    op.claims = (int)c;
    op.tokens_after = (int)r.tokens;
    op.id = id;
    queue_grow(p, op);
  }
  return SKV_OK;
}

skv_status free_impl(skv_pool* p, uint64_t id) {  // kv_cache.hpp:126-134
  auto it = p->id2h.find(id);
  if (it == p->id2h.end()) return fail(p, SKV_ERR_LOGIC, "free_request: unknown request");
  const int h = it->second;
  ReqHost& r = p->req[h];
  p->cur_entries -= (size_t)r.nslots;
  p->token_waste -= entry_waste(p, r);
  if (r.nslots > 0 || r.tokens > 0) {
    skv::FreeOp op{};
    op.handle = h;
    op.model = r.model < 0 ? 0 : r.model;
    op.nslots = r.nslots;
    skv_status st = queue_free(p, op);
    if (st) return st;
  }
  p->id2h.erase(it);
  r = ReqHost();
  p->free_handles.push_back(h);
  p->token_epoch++;
  p->free_epoch++;
  return SKV_OK;
}

// TMA descriptors of the pool for the chunked-prefill kernel: the pool viewed as a 2-D
// tensor of 16-bit elements with one row per token row of a head dim d present in the pool
// ([pool_bytes / 2d rows][d]), box {64, 16} with 128-B swizzle (d = 64: also a {32, 16}
// SW64 box for the V halves).  Returns a mask of bits d/64.
int encode_pool_tmaps(skv_pool* p) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode || p->tpb != 16) return 0;
  int mask = 0;
  auto enc = [&](CUtensorMap* m, int d, int box_x, CUtensorMapSwizzle sw) {
    const cuuint64_t rows = p->storage_bytes / (2 * d);
    if (rows == 0 || rows > 0x7fffffffull) return false;  // TMA coordinates are signed 32-bit
    const cuuint64_t dims[2] = {(cuuint64_t)d, rows};
    const cuuint64_t strides[1] = {(cuuint64_t)(2 * d)};
    const cuuint32_t box[2] = {(cuuint32_t)box_x, 16};
    const cuuint32_t estr[2] = {1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, p->storage, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  for (const ModelInfo& mi : p->models) {
    if (mi.e != 2) continue;
    if (mi.d == 128 && !(mask & 2) && enc(&p->kv_tmap, 128, 64, CU_TENSOR_MAP_SWIZZLE_128B)) mask |= 2;
    if (mi.d == 64 && !(mask & 1) && enc(&p->kv_tmap64, 64, 64, CU_TENSOR_MAP_SWIZZLE_128B) &&
        enc(&p->kv_tmap64v, 64, 32, CU_TENSOR_MAP_SWIZZLE_64B))
      mask |= 1;
    if (mi.d == 256 && !(mask & 4) && enc(&p->kv_tmap256, 256, 64, CU_TENSOR_MAP_SWIZZLE_128B)) mask |= 4;
  }
  return mask;
}

skv_status ensure_storage(skv_pool* p) {
  if (p->storage) return SKV_OK;
  DeviceGuard g(p->device);
  const size_t bytes = (size_t)p->merged_stride * p->P;
  if (bytes == 0) return fail(p, SKV_ERR_ARG, "empty pool");
  SKV_CUDA(p, cudaMalloc(&p->storage, bytes));
  p->storage_bytes = bytes;
  p->has_tmap = encode_pool_tmaps(p);
  return SKV_OK;
}

}  // namespace

extern "C" {

const char* skv_version(void) { return "seakv 0.1 (sm_100a)"; }

void skv_default_opts(skv_pool_opts* o) {
  o->device = 0;
  o->dtype = SKV_FP16;
  o->phys_layers = 0;
  o->max_requests = 4096;
  o->max_blocks_per_request = 0;  // 0 -> min(pool_blocks * max_sub, 4096)
  o->allocate_storage = 0;        // storage is allocated on first data-path use
}

skv_status skv_native_block_bytes(const skv_model_desc* model, int32_t tpb, int32_t tp, double* out) {
  long long nb;
  skv_status st = validate_model(*model, tpb, tp, &nb);
  if (st) return st;
  *out = (double)nb;
  return SKV_OK;
}

skv_status skv_plan_merged_shape(const skv_model_desc* models, int32_t n, int32_t tpb, int32_t tp,
                                 double* out) {
  if (n <= 0) return fail(nullptr, SKV_ERR_CONFIG, "plan_merged_shape: empty model list");
  long long merged = 0;
  for (int i = 0; i < n; ++i) {
    long long nb;
    skv_status st = validate_model(models[i], tpb, tp, &nb);
    if (st) return st;
    merged = std::max(merged, nb);
  }
  *out = (double)merged;
  return SKV_OK;
}

skv_status skv_pool_create(const skv_model_desc* models, int32_t n, int32_t tpb, int32_t tp,
                           size_t pool_blocks, const skv_pool_opts* opts_in, skv_pool** out) {
  *out = nullptr;
  skv_pool_opts opts;
  skv_default_opts(&opts);
  if (opts_in) opts = *opts_in;
  if (n <= 0) return fail(nullptr, SKV_ERR_CONFIG, "plan_merged_shape: empty model list");
  if (n > skv::kMaxModels) return fail(nullptr, SKV_ERR_ARG, "too many models for one pool (max 16)");
  if (tpb < 1) return fail(nullptr, SKV_ERR_CONFIG, "tokens_per_block must be >= 1");
  if (pool_blocks > (size_t)0x7fffffff) return fail(nullptr, SKV_ERR_ARG, "pool_blocks too large");
  auto p = new skv_pool();
  p->device = opts.device;
  p->M = n;
  p->tpb = tpb;
  p->tp = tp;
  p->dtype = opts.dtype;
  p->phys_layers = opts.phys_layers;
  p->P = pool_blocks;
  p->allocate_storage = opts.allocate_storage != 0;
  long long merged = 0;
  for (int i = 0; i < n; ++i) {
    long long nb;
    skv_status st = validate_model(models[i], tpb, tp, &nb);
    if (st) {
      delete p;
      return st;
    }
    ModelInfo mi;
    mi.id = models[i].model_id ? models[i].model_id : ("m" + std::to_string(i));
    mi.L = models[i].num_layers;
    mi.Hkv = models[i].num_heads / tp;
    mi.Hq = (models[i].num_q_heads > 0 ? models[i].num_q_heads : models[i].num_heads) / tp;
    mi.d = models[i].head_dim;
    mi.e = models[i].dtype_bytes;
    mi.native = nb;
    p->models.push_back(mi);
    merged = std::max(merged, nb);
  }
  p->merged_i = merged;
  p->merged = (double)merged;
  long long phys_merged = 0;
  for (ModelInfo& mi : p->models) {
    mi.sub = (int)(p->merged / (double)mi.native);  // kv_cache.hpp:62
    p->maxsub = std::max(p->maxsub, mi.sub);
    mi.phys_L = p->phys_layers > 0 ? std::min(p->phys_layers, mi.L) : mi.L;
    mi.kv_stride = (long long)tpb * mi.d * mi.e;
    mi.head_stride = 2 * mi.kv_stride;
    mi.layer_stride = (long long)mi.Hkv * mi.head_stride;
    mi.native_stride = (long long)mi.phys_L * mi.layer_stride;
    phys_merged = std::max(phys_merged, (long long)mi.sub * mi.native_stride);
  }
  if (p->maxsub > skv::kMaxSub) {
    delete p;
    return fail(nullptr, SKV_ERR_ARG, "more than 64 sub-slots per merged block");
  }
  // 1 KiB aligned: every model's K/V rows (2*head_dim B) start on a TMA row boundary
  p->merged_stride = round_up(p->phys_layers > 0 ? phys_merged : merged, 1024);
  p->R = opts.max_requests > 0 ? opts.max_requests : 4096;
  long long cap = opts.max_blocks_per_request > 0 ? opts.max_blocks_per_request
                                                  : std::min<long long>((long long)pool_blocks * p->maxsub, 4096);
  p->cap = (int)std::max<long long>(cap, 1);
  p->open.assign(n, 0);
  p->free_count = (long long)pool_blocks;
  p->req.assign(p->R, ReqHost());
  p->free_handles.reserve(p->R);
  for (int h = p->R - 1; h >= 0; --h) p->free_handles.push_back(h);

  {
    cudaError_t e = cudaSetDevice(p->device);
    if (e != cudaSuccess) {
      skv_status st = cuda_fail(nullptr, e, "cudaSetDevice");
      delete p;
      return st;
    }
  }
  DeviceGuard guard(p->device);
  auto bail = [&](skv_status st) {
    g_tls_err = p->err;
    skv_pool_destroy(p);
    return st;
  };
  if (cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(p, SKV_ERR_CUDA, "cudaStreamCreate failed"));
  p->own_stream = true;
  const int W = (int)((pool_blocks + 31) / 32);
  p->prm.M = n;
  p->prm.W = W;
  p->prm.maxsub = p->maxsub;
  p->prm.cap = p->cap;
  p->prm.P = (long long)pool_blocks;
  for (int m = 0; m < n; ++m) p->prm.sub[m] = p->models[m].sub;
  skv::DevAlloc& d = p->dev;
  skv_status st;
  if ((st = dev_alloc(p, &d.free_bits, W)) || (st = dev_alloc(p, &d.partial_bits, (size_t)W * n)) ||
      (st = dev_alloc(p, &d.blk_model, pool_blocks, false)) || (st = dev_alloc(p, &d.blk_occ, pool_blocks)) ||
      (st = dev_alloc(p, &d.slot_owner, pool_blocks * p->maxsub)) || (st = dev_alloc(p, &d.open, n)) ||
      (st = dev_alloc(p, &d.free_count, 1)) || (st = dev_alloc(p, &d.req_table, (size_t)p->R * p->cap, false)) ||
      (st = dev_alloc(p, &d.req_nslots, p->R)) || (st = dev_alloc(p, &d.req_tokens, p->R)) ||
      (st = dev_alloc(p, &d.req_model, p->R, false)) || (st = dev_alloc(p, &d.req_id, p->R)) ||
      (st = dev_alloc(p, &d.hints, 1 + n)) ||
      (st = dev_alloc(p, &d.status, 1)) ||
      (st = dev_alloc(p, &d.free_E, n)) || (st = dev_alloc(p, &d.free_R, n)) ||
      (st = dev_alloc(p, &p->d_outE, (size_t)kResultSlots * n)))
    return bail(st);
  {
    cudaError_t e1 = cudaMemsetAsync(d.blk_model, 0xff, std::max<size_t>(pool_blocks, 1) * sizeof(int32_t), p->stream);
    cudaError_t e2 = cudaMemsetAsync(d.req_model, 0xff, (size_t)p->R * sizeof(int32_t), p->stream);
    if (e1 != cudaSuccess || e2 != cudaSuccess)
      return bail(cuda_fail(p, e1 != cudaSuccess ? e1 : e2, "memset"));
  }
  {  // free bitmap: blocks [0, P) set
    std::vector<uint32_t> fb(W, 0u);
    for (size_t b = 0; b < pool_blocks; ++b) fb[b >> 5] |= 1u << (b & 31);
    long long fc = (long long)pool_blocks;
    // same stream as the zeroing memsets above (the pool stream does not sync with stream 0)
    if (cudaMemcpyAsync(d.free_bits, fb.data(), W * sizeof(uint32_t), cudaMemcpyHostToDevice, p->stream) !=
            cudaSuccess ||
        cudaMemcpyAsync(d.free_count, &fc, sizeof(fc), cudaMemcpyHostToDevice, p->stream) != cudaSuccess ||
        cudaStreamSynchronize(p->stream) != cudaSuccess)
      return bail(fail(p, SKV_ERR_CUDA, "init copy failed"));
  }
  if (cudaHostAlloc(reinterpret_cast<void**>(&p->h_outE), sizeof(int32_t) * kResultSlots * n, cudaHostAllocMapped) != cudaSuccess)
    return bail(fail(p, SKV_ERR_CUDA, "cudaMallocHost failed"));
  if (p->allocate_storage && (st = ensure_storage(p))) return bail(st);
  if (cudaStreamSynchronize(p->stream) != cudaSuccess) return bail(fail(p, SKV_ERR_CUDA, "init sync failed"));
  *out = p;
  return SKV_OK;
}

void skv_pool_destroy(skv_pool* p) {
  if (!p) return;
  DeviceGuard g(p->device);
  if (p->stream) cudaStreamSynchronize(p->stream);
  skv::DevAlloc& d = p->dev;
  for (void* q : {(void*)d.free_bits, (void*)d.partial_bits, (void*)d.blk_model, (void*)d.blk_occ,
                  (void*)d.slot_owner, (void*)d.open, (void*)d.free_count, (void*)d.req_table,
                  (void*)d.req_nslots, (void*)d.req_tokens, (void*)d.req_model, (void*)d.req_id, (void*)d.hints,
                  (void*)d.status,
                  (void*)d.free_E, (void*)d.free_R, (void*)p->d_outE, p->d_ops, p->storage,
                  (void*)p->scr.S, (void*)p->scr.cbeg, (void*)p->scr.nnew, (void*)p->scr.base,
                  (void*)p->scr.nbfirst, (void*)p->scr.newblk, (void*)p->scr.newrank, (void*)p->scr.openlist})
    if (q) cudaFree(q);
  if (p->h_stage) cudaFreeHost(p->h_stage);
  if (p->h_outE) cudaFreeHost(p->h_outE);
  for (FreeResult& r : p->pending)
    if (r.ev) cudaEventDestroy(r.ev);
  if (p->stage_ev) cudaEventDestroy(p->stage_ev);
  if (p->sync_ev) cudaEventDestroy(p->sync_ev);
  if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
  delete p;
}

const char* skv_last_error(const skv_pool* p) { return p ? p->err.c_str() : g_tls_err.c_str(); }

skv_status skv_model_index(const skv_pool* p, const char* model_id, int32_t* out) {
  for (int m = 0; m < p->M; ++m)
    if (p->models[m].id == model_id) {
      *out = m;
      return SKV_OK;
    }
  return fail(const_cast<skv_pool*>(p), SKV_ERR_CONFIG,
              std::string("kv cache: model not shared on this engine: ") + model_id);
}

int32_t skv_sub_slots_per_merged(const skv_pool* p, int32_t m) {
  return (m >= 0 && m < p->M) ? p->models[m].sub : 0;
}
double skv_merged_block_bytes(const skv_pool* p) { return p->merged; }
size_t skv_pool_size(const skv_pool* p) { return p->P; }
size_t skv_free_blocks(skv_pool* p) {
  ensure_counters(p);
  return (size_t)p->free_count;
}
size_t skv_allocated_blocks(skv_pool* p) {
  ensure_counters(p);
  return p->P - (size_t)p->free_count;
}
int32_t skv_tokens_per_block(const skv_pool* p) { return p->tpb; }
size_t skv_native_blocks_for(const skv_pool* p, int64_t tokens) {
  return (size_t)((tokens + p->tpb - 1) / p->tpb);
}
int32_t skv_registered(const skv_pool* p, uint64_t id) { return p->id2h.count(id) ? 1 : 0; }
int64_t skv_request_tokens(const skv_pool* p, uint64_t id) {
  auto it = p->id2h.find(id);
  return it == p->id2h.end() ? -1 : p->req[it->second].tokens;
}
size_t skv_available_slots(skv_pool* p, int32_t m) {
  if (m < 0 || m >= p->M) return 0;
  ensure_counters(p);
  return (size_t)(p->open[m] + p->free_count * p->models[m].sub);
}

skv_status skv_can_grow_to(skv_pool* p, uint64_t id, int32_t m, int64_t tokens, int32_t* out) {
  if (m < 0 || m >= p->M) return fail(p, SKV_ERR_ARG, "model index out of range");
  const long long need = ceil_div_ll(tokens, p->tpb);
  if (need < 0) {  // the reference's size_t need wraps to a huge count: never satisfiable (:93-98)
    *out = 0;
    return SKV_OK;
  }
  long long have = 0;
  auto it = p->id2h.find(id);
  if (it != p->id2h.end()) have = p->req[it->second].nslots;
  if (need <= have) {
    *out = 1;
    return SKV_OK;
  }
  skv_status st = ensure_counters(p);
  if (st) return st;
  *out = (p->open[m] + p->free_count * p->models[m].sub) >= need - have ? 1 : 0;
  return SKV_OK;
}

skv_status skv_try_allocate(skv_pool* p, uint64_t id, int32_t m, int64_t tokens) {
  return try_allocate_impl(p, id, m, tokens);
}

skv_status skv_free_request(skv_pool* p, uint64_t id) { return free_impl(p, id); }

skv_status skv_record_context_read(skv_pool* p, uint64_t id) {  // :138-142
  auto it = p->id2h.find(id);
  if (it != p->id2h.end()) p->rw += (uint64_t)p->req[it->second].nslots;
  return SKV_OK;
}

skv_status skv_synchronize(skv_pool* p) {
  skv_status st = flush(p);
  if (st) return st;
  st = ensure_counters(p);
  if (st) return st;
  DeviceGuard g(p->device);
  SKV_CUDA(p, cudaStreamSynchronize(p->stream));
  int32_t status = 0;
  SKV_CUDA(p, cudaMemcpy(&status, p->dev.status, sizeof(status), cudaMemcpyDeviceToHost));
  if (status == 3)
    return fail(p, SKV_ERR_CUDA, "decode plan exceeded the work-list capacity sized at capture time "
                                 "(a CUDA graph replayed at longer contexts): re-capture the graph");
  if (status) return fail(p, SKV_ERR_CUDA, "device allocator invariant violated (code " + std::to_string(status) + ")");
  return SKV_OK;
}

skv_status skv_block_table(skv_pool* p, uint64_t id, int32_t* pairs, size_t cap, size_t* n) {
  auto it = p->id2h.find(id);
  if (it == p->id2h.end()) return fail(p, SKV_ERR_LOGIC, "block_table: unknown request");
  const int h = it->second;
  const int ns = p->req[h].nslots;
  *n = (size_t)ns;
  if (!pairs || cap == 0 || ns == 0) return SKV_OK;
  skv_status st = skv_synchronize(p);
  if (st) return st;
  const size_t cnt = std::min<size_t>(cap, (size_t)ns);
  SKV_CUDA(p, cudaMemcpy(pairs, p->dev.req_table + (size_t)h * p->cap, cnt * sizeof(int2),
                         cudaMemcpyDeviceToHost));
  return SKV_OK;
}

skv_status skv_owner_of(skv_pool* p, int32_t block, int32_t slot, uint64_t* owner) {
  if (block < 0 || (size_t)block >= p->P) return fail(p, SKV_ERR_ARG, "owner_of: block out of range");
  *owner = 0;
  if (slot < 0 || slot >= p->maxsub) return SKV_OK;
  skv_status st = skv_synchronize(p);
  if (st) return st;
  int32_t bm = -1;
  SKV_CUDA(p, cudaMemcpy(&bm, p->dev.blk_model + block, sizeof(bm), cudaMemcpyDeviceToHost));
  if (bm < 0 || slot >= p->models[bm].sub) return SKV_OK;  // slot_owner.size() check (:152)
  unsigned long long o = 0;
  SKV_CUDA(p, cudaMemcpy(&o, p->dev.slot_owner + (size_t)block * p->maxsub + slot, sizeof(o),
                         cudaMemcpyDeviceToHost));
  *owner = o;
  return SKV_OK;
}

size_t skv_table_entries(const skv_pool* p) { return p->cur_entries; }

double skv_fragmentation_bytes(skv_pool* p) {
  ensure_counters(p);
  return (double)(p->slot_frag + p->token_waste);
}

skv_status skv_stats(skv_pool* p, skv_cache_stats* out) {
  out->block_table_entries = p->peak_entries;
  out->native_reads_writes = p->rw;
  out->internal_fragmentation_bytes = (double)p->peak_frag;
  out->peak_utilization = p->P == 0 ? 0.0 : (double)p->peak_used / (double)p->P;
  return SKV_OK;
}

skv_status skv_replay(skv_pool* p, const skv_kv_op* ops, size_t n, int32_t* granted) {
  for (size_t i = 0; i < n; ++i) {
    skv_status st;
    if (ops[i].kind == 0) {
      st = try_allocate_impl(p, ops[i].request_id, ops[i].model_idx, ops[i].tokens);
      if (granted) granted[i] = st == SKV_OK ? 1 : 0;
      if (st == SKV_CACHE_FULL) continue;
    } else {
      st = free_impl(p, ops[i].request_id);
      if (granted) granted[i] = 0;
    }
    if (st) return st;
  }
  return SKV_OK;
}

skv_status skv_flush(skv_pool* p, void* stream) {
  skv_status st = flush(p);
  if (st) return st;
  if (stream && stream != p->stream) {
    DeviceGuard g(p->device);
    if (!p->sync_ev) SKV_CUDA(p, cudaEventCreateWithFlags(&p->sync_ev, cudaEventDisableTiming));
    SKV_CUDA(p, cudaEventRecord(p->sync_ev, p->stream));
    SKV_CUDA(p, cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), p->sync_ev, 0));
  }
  return SKV_OK;
}

skv_status skv_set_stream(skv_pool* p, void* stream) {
  skv_status st = flush(p);
  if (st) return st;
  DeviceGuard g(p->device);
  cudaStream_t ns = static_cast<cudaStream_t>(stream);
  if (ns == p->stream) return SKV_OK;
  if (!p->sync_ev) SKV_CUDA(p, cudaEventCreateWithFlags(&p->sync_ev, cudaEventDisableTiming));
  SKV_CUDA(p, cudaEventRecord(p->sync_ev, p->stream));
  if (ns) SKV_CUDA(p, cudaStreamWaitEvent(ns, p->sync_ev, 0));
  else SKV_CUDA(p, cudaStreamSynchronize(p->stream));
  if (p->own_stream) {
    SKV_CUDA(p, cudaStreamSynchronize(p->stream));
    cudaStreamDestroy(p->stream);
    p->own_stream = false;
  }
  p->stream = ns;
  return SKV_OK;
}

void* skv_get_stream(const skv_pool* p) { return p->stream; }

// ------------------------------------------------------------------ batches --------
static skv_status batch_fill(skv_pool* p, skv_batch* b, const int32_t* group_models, const int32_t* group_sizes,
                             int32_t n_groups, const uint64_t* request_ids) {
  if (n_groups <= 0 || n_groups > skv::kMaxGroups) return fail(p, SKV_ERR_ARG, "batch: 1..16 groups");
  b->ngroups = n_groups;
  b->gmodel.clear();
  b->gsize.clear();
  b->gbegin.clear();
  b->ids.clear();
  b->handles.clear();
  b->h_group.clear();
  int total = 0;
  for (int g = 0; g < n_groups; ++g) {
    if (group_models[g] < 0 || group_models[g] >= p->M || group_sizes[g] < 0)
      return fail(p, SKV_ERR_ARG, "batch: bad group");
    b->gmodel.push_back(group_models[g]);
    b->gsize.push_back(group_sizes[g]);
    b->gbegin.push_back(total);
    for (int i = 0; i < group_sizes[g]; ++i) {
      const uint64_t id = request_ids[total + i];
      auto it = p->id2h.find(id);
      if (it == p->id2h.end()) return fail(p, SKV_ERR_LOGIC, "batch: unknown request " + std::to_string(id));
      if (p->req[it->second].nslots > 0 && p->req[it->second].model != group_models[g])
        return fail(p, SKV_ERR_LOGIC, "batch: request belongs to another model");
      b->ids.push_back(id);
      b->handles.push_back(it->second);
      b->h_group.push_back(g);
    }
    total += group_sizes[g];
  }
  b->nreq = total;
  DeviceGuard guard(p->device);
  if ((size_t)total > b->req_cap) {
    SKV_CUDA(p, cudaStreamSynchronize(p->stream));
    for (void* q : {(void*)b->d_handles, (void*)b->d_group, (void*)b->d_rscr})
      if (q) cudaFree(q);
    b->req_cap = std::max<size_t>((size_t)total * 2, 64);
    skv_status st;
    if ((st = dev_alloc(p, &b->d_handles, b->req_cap, false)) || (st = dev_alloc(p, &b->d_group, b->req_cap, false)) ||
        (st = dev_alloc(p, &b->d_rscr, 5 * b->req_cap)))
      return st;
    if (b->h_stage) cudaFreeHost(b->h_stage);
    SKV_CUDA(p, cudaHostAlloc(&b->h_stage, b->req_cap * 2 * sizeof(int32_t), cudaHostAllocMapped));
  }
  if (!b->d_nitems) {
    skv_status st;
    if ((st = dev_alloc(p, &b->d_nitems, 1)) || (st = dev_alloc(p, &b->d_counter, 6))) return st;  // [0..3] decode sets, [4] prefill items
  }
  if (total) {
    // stage through pinned memory on the pool stream (wait for the previous upload first)
    if (b->stage_ev) SKV_CUDA(p, cudaEventSynchronize(b->stage_ev));
    int32_t* hs = static_cast<int32_t*>(b->h_stage);
    std::memcpy(hs, b->handles.data(), total * 4);
    std::memcpy(hs + b->req_cap, b->h_group.data(), total * 4);
    skv::launch_stage_copy(b->d_handles, hs, total * 4, p->stream);  // SM copies (see flush)
    skv::launch_stage_copy(b->d_group, hs + b->req_cap, total * 4, p->stream);
    if (!b->stage_ev) SKV_CUDA(p, cudaEventCreateWithFlags(&b->stage_ev, cudaEventDisableTiming));
    SKV_CUDA(p, cudaEventRecord(b->stage_ev, p->stream));
  }
  b->plan_epoch = ~0ull;
  b->launch_epoch++;
  b->checked_epoch = p->free_epoch;  // ids were just resolved against the registry
  return SKV_OK;
}

skv_status skv_batch_create(skv_pool* p, const int32_t* group_models, const int32_t* group_sizes,
                            int32_t n_groups, const uint64_t* request_ids, skv_batch** out) {
  *out = nullptr;
  auto b = new skv_batch();
  b->pool = p;
  skv_status st = batch_fill(p, b, group_models, group_sizes, n_groups, request_ids);
  if (st) {
    skv_batch_destroy(b);
    return st;
  }
  *out = b;
  return SKV_OK;
}

skv_status skv_batch_reset(skv_pool* p, skv_batch* b, const int32_t* group_models, const int32_t* group_sizes,
                           int32_t n_groups, const uint64_t* request_ids) {
  if (!b || b->pool != p) return fail(p, SKV_ERR_ARG, "batch belongs to another pool");
  return batch_fill(p, b, group_models, group_sizes, n_groups, request_ids);
}

void skv_batch_destroy(skv_batch* b) {
  if (!b) return;
  DeviceGuard g(b->pool->device);
  cudaStreamSynchronize(b->pool->stream);
  for (void* q : {(void*)b->d_handles, (void*)b->d_group, (void*)b->d_items, (void*)b->d_itemx,
                  (void*)b->d_nitems, (void*)b->d_counter, (void*)b->d_rscr, (void*)b->d_arrive,
                  (void*)b->d_ws_o, (void*)b->d_ws_ml, (void*)b->d_trace})
    if (q) cudaFree(q);
  if (b->h_stage) cudaFreeHost(b->h_stage);
  if (b->stage_ev) cudaEventDestroy(b->stage_ev);
  if (b->d_qlen) cudaFree(b->d_qlen);
  if (b->h_qlen) cudaFreeHost(b->h_qlen);
  if (b->qlen_ev) cudaEventDestroy(b->qlen_ev);
  for (void* q : {(void*)b->d_gops, (void*)b->gscr.S, (void*)b->gscr.cbeg, (void*)b->gscr.nnew, (void*)b->gscr.base,
                  (void*)b->gscr.nbfirst, (void*)b->gscr.newblk, (void*)b->gscr.newrank, (void*)b->gscr.openlist})
    if (q) cudaFree(q);
  delete b;
}

static skv_status check_batch(skv_pool* p, skv_batch* b) {
  if (!b || b->pool != p) return fail(p, SKV_ERR_ARG, "batch belongs to another pool");
  if (b->checked_epoch == p->free_epoch) return SKV_OK;  // no free since the last full check
  for (int i = 0; i < b->nreq; ++i) {
    auto it = p->id2h.find(b->ids[i]);
    if (it == p->id2h.end() || it->second != b->handles[i])
      return fail(p, SKV_ERR_LOGIC, "batch: request " + std::to_string(b->ids[i]) + " was freed");
  }
  b->checked_epoch = p->free_epoch;
  return SKV_OK;
}

skv_status skv_batch_grow(skv_pool* p, skv_batch* b, int64_t delta, int32_t* n_granted) {
  skv_status st = check_batch(p, b);
  if (st) return st;
  int granted = 0;
  for (int g = 0; g < b->ngroups; ++g) {
    for (int i = 0; i < b->gsize[g]; ++i) {
      const int r = b->gbegin[g] + i;
      const int h = b->handles[r];
      const ReqHost& rh = p->req[h];
      if (!rh.live || rh.id != b->ids[r]) return fail(p, SKV_ERR_LOGIC, "batch grow: request no longer registered");
      if (delta < 0) return fail(p, SKV_ERR_VALIDATION, "allocate: negative tokens_needed");
      st = grow_handle_impl(p, h, b->ids[r], b->gmodel[g], rh.tokens + delta);
      if (st == SKV_OK) granted++;
      else if (st != SKV_CACHE_FULL) return st;
    }
  }
  if (n_granted) *n_granted = granted;
  return SKV_OK;
}

static skv_status order_streams(skv_pool* p, cudaStream_t s);
static skv_status after_data(skv_pool* p, cudaStream_t s);

// Decode-step growth with device-generated ops.  Host side: the exact mirror of
// try_allocate(id, model, tokens + delta) for every request in batch order, applied only if
// ALL are granted (the sequential claims of model m need ceil(max(0, C_m - open_m) / sub_m)
// fresh blocks in total, so all-granted <=> their sum <= free blocks) and every request
// already owns slots (its id is on the device).  Otherwise nothing changes.
skv_status skv_batch_grow_mirror(skv_pool* p, skv_batch* b, int64_t delta, int32_t* all_granted) {
  *all_granted = 0;
  skv_status st = check_batch(p, b);
  if (st) return st;
  if (delta < 0) return fail(p, SKV_ERR_VALIDATION, "allocate: negative tokens_needed");
  if ((st = ensure_counters(p))) return st;
  long long C[skv::kMaxModels] = {0};
  long long max_need = 0;
  for (int g = 0; g < b->ngroups; ++g) {
    const int m = b->gmodel[g];
    for (int i = 0; i < b->gsize[g]; ++i) {
      const ReqHost& r = p->req[b->handles[b->gbegin[g] + i]];
      if (!r.live || r.nslots == 0 || r.model != m) return SKV_OK;  // host path handles these
      const long long need = ceil_div_ll(r.tokens + delta, p->tpb);
      C[m] += std::max(0LL, need - r.nslots);
      max_need = std::max(max_need, need);
    }
  }
  long long blocks = 0;
  for (int m = 0; m < p->M; ++m)
    blocks += C[m] > p->open[m] ? ceil_div_ll(C[m] - p->open[m], p->models[m].sub) : 0;
  if (blocks > p->free_count || max_need > p->cap) return SKV_OK;
  // grow_handle_impl's arithmetic for the granted case, inlined with per-model constants (the
  // watermarks are still taken after every op, as note_watermarks is, kv_cache.hpp:242-246)
  const long long tpb = p->tpb;
  for (int g = 0; g < b->ngroups; ++g) {
    const int m = b->gmodel[g];
    const ModelInfo& mi = p->models[m];
    const long long native = mi.native, per_token = mi.native / tpb, sub = mi.sub;
    for (int i = 0; i < b->gsize[g]; ++i) {
      ReqHost& r = p->req[b->handles[b->gbegin[g] + i]];
      const long long tokens = r.tokens + delta;
      const long long c = std::max(0LL, (tokens + tpb - 1) / tpb - r.nslots);
      if (c > 0) {  // claim_slot x c (:191-222): open slots first, then fresh blocks
        const long long from_open = std::min<long long>(c, p->open[m]);
        const long long rest = c - from_open;
        const long long nb = (rest + sub - 1) / sub;
        p->open[m] += -from_open + nb * sub - rest;
        p->free_count -= nb;
        p->slot_frag += -from_open * native + nb * (p->merged_i - native) - (rest - nb) * native;
        r.nslots += (int)c;
        p->cur_entries += (size_t)c;
      }
      const long long grew = delta > 0 ? delta : 0;  // tokens only grow (:115-119)
      p->rw += (uint64_t)grew;
      r.tokens = tokens;
      p->token_waste += (c * tpb - grew) * per_token + c * native;  // incl. quirk Q1
      p->peak_entries = std::max<uint64_t>(p->peak_entries, p->cur_entries);
      p->peak_used = std::max<long long>(p->peak_used, (long long)p->P - p->free_count);
      p->peak_frag = std::max<long long>(p->peak_frag, p->slot_frag + p->token_waste);
    }
  }
  p->token_epoch++;
  *all_granted = 1;
  return SKV_OK;
}

// The device half: op generation from the device's request state + the placement kernel, on
// `stream` (capturable in a CUDA graph: every buffer is the batch's own).
skv_status skv_batch_grow_launch(skv_pool* p, skv_batch* b, int64_t delta, void* stream) {
  skv_status st = check_batch(p, b);
  if (st) return st;
  if (delta < 0 || delta > (1 << 20)) return fail(p, SKV_ERR_ARG, "grow_launch: delta out of range");
  DeviceGuard guard(p->device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : p->stream;
  const size_t n = (size_t)b->nreq;
  if (!n) return SKV_OK;
  const size_t t = n * (size_t)(ceil_div_ll(delta, p->tpb) + 1);  // claims bound
  if (n > b->gops_cap || t > b->gscr_t) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cs);
    if (cs != cudaStreamCaptureStatusNone)
      return fail(p, SKV_ERR_ARG, "grow_launch: buffers must be sized by an eager call before graph capture");
    SKV_CUDA(p, cudaStreamSynchronize(s));
    skv::GrowScratch& g = b->gscr;
    for (void* q : {(void*)b->d_gops, (void*)g.S, (void*)g.cbeg, (void*)g.nnew, (void*)g.base, (void*)g.nbfirst,
                    (void*)g.newblk, (void*)g.newrank, (void*)g.openlist})
      if (q) cudaFree(q);
    b->gops_cap = n;
    b->gscr_t = t;
    if ((st = dev_alloc(p, &b->d_gops, n, false)) || (st = dev_alloc(p, &g.S, n, false)) ||
        (st = dev_alloc(p, &g.cbeg, n, false)) || (st = dev_alloc(p, &g.nnew, n, false)) ||
        (st = dev_alloc(p, &g.base, n, false)) || (st = dev_alloc(p, &g.nbfirst, n, false)) ||
        (st = dev_alloc(p, &g.newblk, t, false)) || (st = dev_alloc(p, &g.newrank, t, false)) ||
        (st = dev_alloc(p, &g.openlist, t, false)))
      return st;
  }
  if ((st = order_streams(p, s))) return st;  // queued host-side allocator work first
  skv::StepModels gm{};
  for (int g = 0; g < b->ngroups; ++g) gm.m[g] = b->gmodel[g];
  skv::launch_grow_step(p->dev, p->prm, p->tpb, b->d_handles, b->d_group, gm, (int)n, (int)delta, b->d_gops, b->gscr,
                        s);
  p->launches += 1;
  return after_data(p, s);
}

skv_status skv_batch_decode_bytes(skv_pool* p, skv_batch* b, int32_t layer, double* kv_bytes,
                                  double* total_bytes) {
  double kv = 0.0, tot = 0.0;
  for (int g = 0; g < b->ngroups; ++g) {
    const ModelInfo& mi = p->models[b->gmodel[g]];
    if (layer >= mi.L) continue;
    for (int i = 0; i < b->gsize[g]; ++i) {
      const long long ctx = p->req[b->handles[b->gbegin[g] + i]].tokens;
      const double k = (double)ctx * mi.Hkv * mi.d * 2.0 * mi.e;
      kv += k;
      tot += k + 2.0 * mi.Hq * mi.d * mi.e + (double)ceil_div_ll(ctx, p->tpb) * 8.0;
    }
  }
  if (kv_bytes) *kv_bytes = kv;
  if (total_bytes) *total_bytes = tot;
  return SKV_OK;
}

// Common DataParams for one batch / layer.
static skv_status make_params(skv_pool* p, skv_batch* b, int layer, skv::DataParams* dp) {
  std::memset(static_cast<void*>(dp), 0, sizeof(*dp));
  dp->ngroups = b->ngroups;
  dp->nreq = b->nreq;
  dp->handles = b->d_handles;
  dp->req_group = b->d_group;
  dp->req_tokens = p->dev.req_tokens;
  dp->req_table = p->dev.req_table;
  dp->cap = p->cap;
  dp->pool = static_cast<char*>(p->storage);
  dp->has_tmap = p->has_tmap;
  if (p->has_tmap & 2) dp->kv_tmap = p->kv_tmap;
  if (p->has_tmap & 1) {
    dp->kv_tmap64 = p->kv_tmap64;
    dp->kv_tmap64v = p->kv_tmap64v;
  }
  if (p->has_tmap & 4) dp->kv_tmap256 = p->kv_tmap256;
  dp->merged_stride = p->merged_stride;
  dp->tpb = p->tpb;
  dp->dtype = p->dtype;
  dp->head_dim = 0;  // per group (DataGroup::D); this is the largest in the batch
  for (int g = 0; g < b->ngroups; ++g) dp->head_dim = std::max(dp->head_dim, p->models[b->gmodel[g]].d);
  dp->layer = layer;
  if (p->split) {  // split scheme: per (request, layer, head) rows of 8 KiB block ids
    dp->req_table = p->split->table;
    dp->cap = p->split->cap;
    dp->pool = p->split->storage;
    dp->merged_stride = 2 * 16 * 128 * 2;
    dp->split_L = p->split->L;
    dp->split_H = p->split->H;
    dp->has_tmap = 0;
  }
  for (int g = 0; g < b->ngroups; ++g) {
    const ModelInfo& mi = p->models[b->gmodel[g]];
    if ((mi.d != 64 && mi.d != 128 && mi.d != 256) || mi.e != 2 || p->tpb != 16)
      return fail(p, SKV_ERR_ARG, "data path kernels need head_dim 64, 128 or 256, 2-byte dtype, tokens_per_block 16");
    if (p->split && mi.d != 128) return fail(p, SKV_ERR_ARG, "split scheme: head_dim 128 only (8 KiB split blocks)");
    skv::DataGroup& dg = dp->g[g];
    dg.D = mi.d;
    dg.scale_log2 = 1.4426950408889634f / std::sqrt((float)mi.d);
    dg.native_stride = p->split ? 0 : mi.native_stride;
    dg.layer_off = p->split ? 0 : (long long)(layer % mi.phys_L) * mi.layer_stride;
    dg.head_stride = p->split ? 0 : mi.head_stride;
    dg.Hq = mi.Hq;
    dg.Hkv = mi.Hkv;
    dg.G = mi.Hq / mi.Hkv;
    dg.active = layer < mi.L ? 1 : 0;
    dg.req_begin = b->gbegin[g];
    dg.nreq = b->gsize[g];
    if (dg.G != 1 && dg.G != 2 && dg.G != 4 && dg.G != 8)
      return fail(p, SKV_ERR_ARG, "GQA ratio must be 1, 2, 4 or 8");
  }
  return SKV_OK;
}

static skv_status order_streams(skv_pool* p, cudaStream_t s) {
  skv_status st = flush(p);
  if (st) return st;
  if (s != p->stream) {
    if (!p->sync_ev) SKV_CUDA(p, cudaEventCreateWithFlags(&p->sync_ev, cudaEventDisableTiming));
    SKV_CUDA(p, cudaEventRecord(p->sync_ev, p->stream));
    SKV_CUDA(p, cudaStreamWaitEvent(s, p->sync_ev, 0));
  }
  return SKV_OK;
}

static skv_status after_data(skv_pool* p, cudaStream_t s) {
  SKV_CUDA(p, cudaGetLastError());
  if (s != p->stream) {
    SKV_CUDA(p, cudaEventRecord(p->sync_ev, s));
    SKV_CUDA(p, cudaStreamWaitEvent(p->stream, p->sync_ev, 0));
  }
  return SKV_OK;
}

skv_status skv_decode_attention(skv_pool* p, skv_batch* b, const skv_decode_args* a, void* stream) {
  skv_status st = check_batch(p, b);
  if (st) return st;
  if (!p->split && (st = ensure_storage(p))) return st;
  DeviceGuard guard(p->device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : p->stream;
  skv::DataParams dp;
  if ((st = make_params(p, b, a->layer, &dp))) return st;
  int maxg = 1;
  long long sum_hkv = 0, work = 0, max_ctx = 0;
  if ((a->k == nullptr) != (a->v == nullptr))
    return fail(p, SKV_ERR_ARG, "decode: fused append needs both k and v");
  dp.n_new = a->k ? 1 : 0;  // 1 = fused append of the step's token
  for (int g = 0; g < b->ngroups; ++g) {
    dp.g[g].q = a->q[g];
    dp.g[g].out = a->out[g];
    if (a->k) {
      dp.g[g].k = a->k[g];
      dp.g[g].v = a->v[g];
    }
    maxg = std::max(maxg, dp.g[g].G);
    for (int i = 0; i < b->gsize[g]; ++i) {
      const long long ctx = p->req[b->handles[b->gbegin[g] + i]].tokens;
      sum_hkv += dp.g[g].Hkv;
      work += ctx * dp.g[g].Hkv * dp.g[g].D / 128;  // in d=128 token-head units (bytes / 512)
      max_ctx = std::max(max_ctx, ctx);
    }
  }
  if (a->softmax_scale > 0.f)  // else 1/sqrt(head_dim) of each group (make_params)
    for (int g = 0; g < b->ngroups; ++g) dp.g[g].scale_log2 = a->softmax_scale * 1.4426950408889634f;
  dp.scale_log2 = dp.g[0].scale_log2;
  // Work list (plan_kernel): the last n_cut (request, kv head)s get two small trailing
  // pieces (4 per warp slot: enough small work to even out the launch's tail); leading
  // parts are cut to <= split tokens only when there are too few (request, kv head)s to
  // keep every warp slot busy (~4 pieces per slot).
  const int nsm = skv::num_sms();  // current device = the pool's (DeviceGuard)
  const long long slots8 = (long long)nsm * skv::decode_warps_per_cta() * skv::decode_ctas_per_sm();
  int split = a->split_tokens;
  if (split < 0) return fail(p, SKV_ERR_ARG, "decode: split_tokens must be >= 0");
  // Measured on B200 (scripts/sweep_sched.sh, profiles/r01_sweep_sched.txt): chunk when
  // there are fewer than 1.5 (request, kv head)s per warp slot; give trailing pieces to
  // W/2 (request, kv head)s when pieces are short (< 64 tiles: per-piece overhead
  // dominates), else to 2W.  SKV_CHUNK_X4 / SKV_NCUT_X4 override both (in quarters of W).
  static const long long chunk_x4 = [] {
    const char* e = getenv("SKV_CHUNK_X4");
    return e ? atoll(e) : 6LL;
  }();
  static const long long ncut_x4 = [] {
    const char* e = getenv("SKV_NCUT_X4");
    return e ? atoll(e) : -1LL;
  }();
  if (split == 0) {
    if (4 * sum_hkv >= chunk_x4 * slots8 || max_ctx <= 256) split = 1 << 30;
    else split = (int)std::max<long long>(256, round_up(ceil_div_ll(work, 4 * slots8), 16));
  }
  split = (int)std::min<long long>(round_up(split, 16), 1 << 30);
  dp.split_tokens = split;
  const long long piece_tiles = std::min<long long>(ceil_div_ll(work, std::max(1LL, sum_hkv) * 16), split / 16);
  const long long ncut = ncut_x4 >= 0 ? ncut_x4 * slots8 / 4 : (piece_tiles < 64 ? slots8 / 2 : 2 * slots8);
  dp.n_cut = (int)std::min<long long>(ncut, sum_hkv);
  b->last_sum_hkv = sum_hkv;
  b->last_ncut = dp.n_cut;
  // capacities: an upper bound on pieces and partial slots (every head cut)
  long long items = 0, slots = 0;
  const long long maxt = std::max(1, split / 16);
  for (int g = 0; g < b->ngroups; ++g)
    for (int i = 0; i < b->gsize[g]; ++i) {
      const long long nt = ceil_div_ll(std::max<long long>(p->req[b->handles[b->gbegin[g] + i]].tokens, 0), 16);
      const long long k1 = nt > 0 ? ceil_div_ll(nt, maxt) : 1;
      const long long ns = k1 + 2;
      items += ns * dp.g[g].Hkv;
      slots += ns * dp.g[g].G * dp.g[g].Hkv;
    }
  if ((size_t)items > b->items_cap) {
    SKV_CUDA(p, cudaStreamSynchronize(s));
    for (void* q : {(void*)b->d_items, (void*)b->d_itemx, (void*)b->d_arrive})
      if (q) cudaFree(q);
    b->items_cap = (size_t)items * 2;
    SKV_CUDA(p, cudaMalloc(&b->d_items, b->items_cap * sizeof(int4)));
    SKV_CUDA(p, cudaMalloc(&b->d_itemx, b->items_cap * sizeof(int4)));
    if ((st = dev_alloc(p, &b->d_arrive, 2 * b->items_cap))) return st;
    b->plan_epoch = ~0ull;
  }
  if ((size_t)slots > b->slots_cap) {
    SKV_CUDA(p, cudaStreamSynchronize(s));
    if (b->d_ws_o) cudaFree(b->d_ws_o);
    if (b->d_ws_ml) cudaFree(b->d_ws_ml);
    b->slots_cap = (size_t)slots * 2;
    SKV_CUDA(p, cudaMalloc(&b->d_ws_o, b->slots_cap * 256 * sizeof(float)));  // up to head_dim 256 per slot
    SKV_CUDA(p, cudaMalloc(&b->d_ws_ml, b->slots_cap * sizeof(float2)));
  }
  dp.items = b->d_items;
  dp.n_items = b->d_nitems;
  // Consecutive decode launches alternate between two (work counter, arrival counter)
  // sets: under programmatic dependent launch the next launch starts fetching work
  // while this one drains, and each launch's last CTA / last split resets its own set.
  const int parity = (int)(b->launch_seq++ & 1);
  dp.counter = b->d_counter + 2 * parity;
  dp.itemx = b->d_itemx;
  dp.rscr = b->d_rscr;
  dp.items_cap = (int)std::min<size_t>(b->items_cap, 0x7fffffff);
  dp.slots_cap = (int)std::min<size_t>(b->slots_cap, 0x7fffffff);
  dp.status = p->dev.status;
  dp.arrive = b->d_arrive + parity * b->items_cap;
  dp.ws_o = b->d_ws_o;
  dp.ws_ml = b->d_ws_ml;
  if ((st = order_streams(p, s))) return st;
  bool planned = false;
  if (b->plan_epoch != p->token_epoch || b->plan_split != split) {
    skv::launch_decode_plan(dp, s);
    p->launches++;
    b->plan_epoch = p->token_epoch;
    b->plan_split = split;
    planned = true;
  }
  // K/V tiles may be prefetched before the previous launch completes only when nothing
  // that launch may still write is read early: the work list comes from an earlier
  // plan, and the new token (the only pool bytes written by a fused decode) is patched
  // in after the wait by this launch's own fused append.
  static const bool no_prefetch = [] {
    const char* e = getenv("SKV_NO_PREFETCH");
    return e && e[0] == '1';
  }();
  dp.prefetch = (!planned && dp.n_new == 1 && !no_prefetch) ? 1 : 0;
  static const bool trace_on = [] {
    const char* e = getenv("SKV_TRACE");
    return e && e[0] == '1';
  }();
  if (trace_on) {
    const size_t n = (size_t)slots8;
    if (!b->d_trace) {
      SKV_CUDA(p, cudaMalloc(&b->d_trace, n * 4 * sizeof(unsigned long long)));
      b->trace_n = n;
    }
    dp.trace = b->d_trace;
  }
  // split partials are merged inside the decode kernel; its work counter self-resets
  skv::launch_decode(dp, maxg, 0, s);
  p->launches++;
  return after_data(p, s);
}

// Per-request token counts of a ragged append / prefill: lens[r] (batch order) and each
// request's first row in its group's packed tensors go to the device ([lens | offsets]).
// Consecutive calls with the same lengths (append then prefill of a layer, every layer of a
// step) reuse the uploaded arrays; a new upload waits only for the previous one's copy.
static skv_status stage_lengths(skv_pool* p, skv_batch* b, const int32_t* lens, cudaStream_t s,
                                const int32_t** d_lens, const int32_t** d_offs) {
  const size_t n = (size_t)b->nreq;
  if (n > b->qlen_cap) {
    SKV_CUDA(p, cudaStreamSynchronize(s));
    if (b->d_qlen) cudaFree(b->d_qlen);
    if (b->h_qlen) cudaFreeHost(b->h_qlen);
    b->qlen_cap = std::max(b->req_cap, n);
    SKV_CUDA(p, cudaMalloc(&b->d_qlen, 2 * b->qlen_cap * sizeof(int32_t)));
    SKV_CUDA(p, cudaHostAlloc(&b->h_qlen, 2 * b->qlen_cap * sizeof(int32_t), cudaHostAllocMapped));
    b->qlen_last.clear();
  }
  *d_lens = b->d_qlen;
  *d_offs = b->d_qlen + b->qlen_cap;
  if (b->qlen_last.size() == n && std::equal(lens, lens + n, b->qlen_last.begin()) && b->qlen_epoch == b->launch_epoch)
    return SKV_OK;
  if (b->qlen_ev) SKV_CUDA(p, cudaEventSynchronize(b->qlen_ev));  // staging buffer reuse
  for (int g = 0; g < b->ngroups; ++g) {
    int off = 0;
    for (int i = 0; i < b->gsize[g]; ++i) {
      const int r = b->gbegin[g] + i;
      b->h_qlen[r] = lens[r];
      b->h_qlen[b->qlen_cap + r] = off;
      off += lens[r];
    }
  }
  skv::launch_stage_copy(b->d_qlen, b->h_qlen, n * sizeof(int32_t), s);
  skv::launch_stage_copy(b->d_qlen + b->qlen_cap, b->h_qlen + b->qlen_cap, n * sizeof(int32_t), s);
  if (!b->qlen_ev) SKV_CUDA(p, cudaEventCreateWithFlags(&b->qlen_ev, cudaEventDisableTiming));
  SKV_CUDA(p, cudaEventRecord(b->qlen_ev, s));
  b->qlen_last.assign(lens, lens + n);
  b->qlen_epoch = b->launch_epoch;
  p->launches += 2;
  return SKV_OK;
}

skv_status skv_batch_plan_info(skv_pool* p, skv_batch* b, int32_t* split_tokens, int64_t* n_cut,
                               int64_t* sum_hkv) {
  if (!b || b->pool != p) return fail(p, SKV_ERR_ARG, "batch belongs to another pool");
  if (split_tokens) *split_tokens = b->plan_split;
  if (n_cut) *n_cut = b->last_ncut;
  if (sum_hkv) *sum_hkv = b->last_sum_hkv;
  return SKV_OK;
}

skv_status skv_append_kv(skv_pool* p, skv_batch* b, const skv_append_args* a, void* stream) {
  skv_status st = check_batch(p, b);
  if (st) return st;
  if (!p->split && (st = ensure_storage(p))) return st;
  int max_new = a->n_new;
  if (a->n_news) {
    max_new = 0;
    for (int i = 0; i < b->nreq; ++i) {
      if (a->n_news[i] < 1) return fail(p, SKV_ERR_ARG, "append: every n_news[i] must be >= 1");
      if (p->req[b->handles[i]].tokens < a->n_news[i])
        return fail(p, SKV_ERR_ARG, "append: request " + std::to_string(b->ids[i]) + " holds fewer than n_new tokens");
      max_new = std::max(max_new, a->n_news[i]);
    }
  } else if (a->n_new < 1) {
    return fail(p, SKV_ERR_ARG, "append: n_new must be >= 1");
  }
  DeviceGuard guard(p->device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : p->stream;
  skv::DataParams dp;
  if ((st = make_params(p, b, a->layer, &dp))) return st;
  for (int g = 0; g < b->ngroups; ++g) {
    dp.g[g].k = a->k[g];
    dp.g[g].v = a->v[g];
  }
  dp.n_new = a->n_new;
  dp.max_q_len = max_new;
  if ((st = order_streams(p, s))) return st;
  if (a->n_news && b->nreq && (st = stage_lengths(p, b, a->n_news, s, &dp.q_lens, &dp.q_offs))) return st;
  if (b->nreq) {
    skv::launch_append(dp, s);
    p->launches++;
  }
  return after_data(p, s);
}

skv_status skv_prefill_attention(skv_pool* p, skv_batch* b, const skv_prefill_args* a, void* stream) {
  skv_status st = check_batch(p, b);
  if (st) return st;
  if ((st = ensure_storage(p))) return st;
  if (!a->q_lens && a->q_len < 1) return fail(p, SKV_ERR_ARG, "prefill: q_len must be >= 1");
  int max_q = a->q_len;
  if (a->q_lens) {
    max_q = 0;
    for (int i = 0; i < b->nreq; ++i) {
      if (a->q_lens[i] < 1) return fail(p, SKV_ERR_ARG, "prefill: every q_lens[i] must be >= 1");
      max_q = std::max(max_q, a->q_lens[i]);
    }
  }
  for (int i = 0; i < b->nreq; ++i)
    if (p->req[b->handles[i]].tokens < (a->q_lens ? a->q_lens[i] : a->q_len))
      return fail(p, SKV_ERR_ARG, "prefill: request " + std::to_string(b->ids[i]) + " holds fewer than q_len tokens");
  DeviceGuard guard(p->device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : p->stream;
  skv::DataParams dp;
  if ((st = make_params(p, b, a->layer, &dp))) return st;
  for (int g = 0; g < b->ngroups; ++g) {
    dp.g[g].q = a->q[g];
    dp.g[g].out = a->out[g];
    const int d = p->models[b->gmodel[g]].d;
    if (!(p->has_tmap & (d / 64)))
      return fail(p, SKV_ERR_ARG, "prefill: no TMA descriptor for head_dim " + std::to_string(d));
    if (a->softmax_scale > 0.f) dp.g[g].scale_log2 = a->softmax_scale * 1.4426950408889634f;
  }
  dp.scale_log2 = dp.g[0].scale_log2;
  dp.n_new = a->q_len;
  dp.max_q_len = max_q;
  if (a->q_lens && b->nreq) {  // per-request lengths + row offsets within each group's q/out
    if ((st = order_streams(p, s))) return st;
    if ((st = stage_lengths(p, b, a->q_lens, s, &dp.q_lens, &dp.q_offs))) return st;
  }
  static const int dbg = [] {
    const char* e = getenv("SKV_PREFILL_DBG");
    return e ? atoi(e) : 0;
  }();
  dp.dbg = dbg;
  dp.counter = b->d_counter + 4;  // persistent prefill work counter (reset per launch)
  static const bool trace_on = [] {
    const char* e = getenv("SKV_TRACE");
    return e && e[0] == '1';
  }();
  if (trace_on) {  // prefill kernels built with -DSKV_PF_TRACE: 16 u64 per CTA (4 records)
    int tiles = 1, heads = 1;
    for (int g = 0; g < b->ngroups; ++g) {
      tiles = std::max(tiles, (max_q * dp.g[g].G + 127) / 128);
      heads = std::max(heads, dp.g[g].Hkv);
    }
    const size_t n = (size_t)((tiles + 1) / 2) * heads * b->nreq * 4;
    if (b->trace_n < n) {
      if (b->d_trace) cudaFree(b->d_trace);
      SKV_CUDA(p, cudaMalloc(&b->d_trace, n * 4 * sizeof(unsigned long long)));
      b->trace_n = n;
    }
    SKV_CUDA(p, cudaMemsetAsync(b->d_trace, 0, n * 4 * sizeof(unsigned long long), s));
    dp.trace = b->d_trace;
  }
  if ((st = order_streams(p, s))) return st;
  skv::launch_prefill(dp, s);
  int dmask = 0;  // one launch per head dim present
  for (int g = 0; g < b->ngroups; ++g) dmask |= p->models[b->gmodel[g]].d / 64;
  p->launches += __builtin_popcount(dmask & 7);
  return after_data(p, s);
}

skv_status skv_model_layout(const skv_pool* p, int32_t m, skv_layout* out) {
  if (m < 0 || m >= p->M) return fail(const_cast<skv_pool*>(p), SKV_ERR_ARG, "model index out of range");
  const ModelInfo& mi = p->models[m];
  out->merged_stride = p->merged_stride;
  out->native_stride = mi.native_stride;
  out->layer_stride = mi.layer_stride;
  out->head_stride = mi.head_stride;
  out->kv_stride = mi.kv_stride;
  out->tpb = p->tpb;
  out->head_dim = mi.d;
  out->kv_heads = mi.Hkv;
  out->q_heads = mi.Hq;
  out->phys_layers = mi.phys_L;
  out->dtype = p->dtype;
  return SKV_OK;
}

void* skv_storage(const skv_pool* p, size_t* bytes) {
  if (bytes) *bytes = (size_t)p->merged_stride * p->P;
  return p->storage;
}

skv_status skv_synth_fill(skv_pool* p, uint64_t seed, float amp, void* stream) {
  skv_status st = ensure_storage(p);
  if (st) return st;
  DeviceGuard guard(p->device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : p->stream;
  if ((st = order_streams(p, s))) return st;
  skv::launch_synth_fill(p->storage, p->storage_bytes, p->dtype, seed, amp, s);
  p->launches++;
  return after_data(p, s);
}

skv_status skv_read_blocks(skv_pool* p, const int32_t* ids, size_t n, void* dst) {
  skv_status st = ensure_storage(p);
  if (st) return st;
  if ((st = skv_synchronize(p))) return st;
  DeviceGuard guard(p->device);
  SKV_CUDA(p, cudaDeviceSynchronize());
  for (size_t i = 0; i < n; ++i) {
    if (ids[i] < 0 || (size_t)ids[i] >= p->P) return fail(p, SKV_ERR_ARG, "read_blocks: id out of range");
    SKV_CUDA(p, cudaMemcpy(static_cast<char*>(dst) + i * p->merged_stride,
                           static_cast<char*>(p->storage) + (size_t)ids[i] * p->merged_stride,
                           p->merged_stride, cudaMemcpyDeviceToHost));
  }
  return SKV_OK;
}

uint64_t skv_kernel_launches(const skv_pool* p) { return p->launches; }

}  // extern "C"

skv_status skv_debug_decode_trace(skv_pool* p, skv_batch* b, uint64_t* host, size_t cap, size_t* n) {
  *n = 0;
  if (!b || b->pool != p) return fail(p, SKV_ERR_ARG, "batch belongs to another pool");
  if (!b->d_trace) return SKV_OK;
  DeviceGuard guard(p->device);
  SKV_CUDA(p, cudaDeviceSynchronize());
  const size_t m = std::min(cap / 4, b->trace_n);
  SKV_CUDA(p, cudaMemcpy(host, b->d_trace, m * 4 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  *n = m;
  return SKV_OK;
}

void skv_internal_set_split(skv_pool* p, const skv::SplitView* view) { p->split = view; }
int skv_internal_handle(const skv_pool* p, uint64_t id) {
  auto it = p->id2h.find(id);
  return it == p->id2h.end() ? -1 : it->second;
}

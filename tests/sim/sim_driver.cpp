// sim_driver.cpp — runs the reference discrete-event simulator (run_simulation,
// simulation.hpp:452-459) on a small deterministic two-engine scenario and prints
// every number that depends on the KV cache: per-engine CacheStats, aggregate
// serving metrics, and a hash of every request's outcome.  Built twice by
// oracle/Makefile: against the reference kv_cache.hpp (sim_ref) and against the
// GPU drop-in (sim_dropin); the two outputs must be identical.
//
// Optional 4th argument: an INI file of [cost <model> tp=<n>] sections (the reference's
// own format, config.hpp:311-328) that replaces default_cost_model entries -- e.g. the
// B200-measured decode attention cost written by scripts/calibrate_cost.py, so the
// reference simulator prices decode with this repository's measured kernel time.
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <vector>

#include "seasim/config.hpp"
#include "seasim/simulation.hpp"

using namespace seasim;

static ServiceProfile service(const CostModel& cost, const char* name, const char* model, double in_mean,
                              double in_sd, double out_mean, double out_sd) {
  ServiceProfile p;
  p.name = name;
  p.model_id = model;
  p.input_len_dist.mean = in_mean;
  p.input_len_dist.stddev = in_sd;
  p.output_len_dist.mean = out_mean;
  p.output_len_dist.stddev = out_sd;
  const int tp = cost.model(model).min_tp;
  p.mean_exec_time = cost.isolated_exec_time(model, tp, (long)in_mean, (long)out_mean) * tp;
  p.exec_time_stddev = 0.3 * p.mean_exec_time;
  p.slo = 5.0 * p.mean_exec_time;
  p.starvation_threshold = 10.0 * p.mean_exec_time;
  return p;
}

static std::uint64_t fnv(std::uint64_t h, std::uint64_t v) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xff;
    h *= 1099511628211ull;
  }
  return h;
}

int main(int argc, char** argv) {
  const double rate = argc > 1 ? std::atof(argv[1]) : 6.0;
  const double duration = argc > 2 ? std::atof(argv[2]) : 30.0;
  const double pool_gb = argc > 3 ? std::atof(argv[3]) : 2.0;
  CostModel cost = default_cost_model();
  if (argc > 4) {  // measured cost overrides, parsed with the reference's INI reader
    std::ifstream in(argv[4]);
    if (!in) {
      std::fprintf(stderr, "cannot open %s\n", argv[4]);
      return 2;
    }
    const detail::IniFile ini = detail::parse_ini(in, argv[4]);
    for (const auto* sec : ini.all("cost")) {
      std::istringstream hs(sec->header);
      std::string word, model_id, tp_word;
      hs >> word >> model_id >> tp_word;
      detail::SectionView view(sec, sec->header);
      CostCoeffs c;
      c.prefill_fixed = view.num("prefill_fixed", 0.0);
      c.prefill_per_token = view.num("prefill_per_token", 0.0);
      c.decode_fixed = view.num("decode_fixed", 0.0);
      c.decode_per_seq = view.num("decode_per_seq", 0.0);
      c.decode_per_context_token = view.num("decode_per_context_token", 0.0);
      c.activation_base = view.num("activation_base_gb", 0.5) * kGiB;
      c.activation_per_seq = view.num("activation_per_seq_gb", 0.02) * kGiB;
      cost.add_entry(model_id, std::stoi(tp_word.substr(3)), c);
    }
  }
  std::vector<ServiceProfile> profiles = {
      service(cost, "chat-7b", "llama2-7b", 73.0, 40.0, 427.0, 200.0),
      service(cost, "summ-13b", "llama2-13b", 2000.0, 600.0, 21.0, 8.0),
      service(cost, "chat-13b", "llama2-13b", 73.0, 40.0, 300.0, 100.0),
      service(cost, "code-opt", "opt-6.7b", 156.0, 60.0, 67.0, 30.0),
  };
  PlacementPlan plan;
  SharingGroup g0, g1;
  g0.services = {0, 1};
  g0.gpu_ids = {0};
  g1.services = {2, 3};
  g1.gpu_ids = {1};
  plan.groups = {g0, g1};
  GpuSpec cluster;
  SimOptions opts;
  opts.kv_pool_cap_bytes = pool_gb * 1e9;  // small pools: admission waits and evictions happen
  opts.seed = 7;
  const Trace trace = generate_trace(profiles, rate, duration, 4, 2025);
  const RunResult r = run_simulation(trace, plan, profiles, cost, cluster, opts);
  std::printf("requests %zu end_time %.17g\n", r.requests.size(), r.end_time);
  for (std::size_t e = 0; e < r.kv_stats.size(); ++e) {
    const CacheStats& s = r.kv_stats[e];
    std::printf("engine %zu kv entries %" PRIu64 " rw %" PRIu64 " frag %.17g util %.17g\n", e,
                s.block_table_entries, s.native_reads_writes, s.internal_fragmentation_bytes, s.peak_utilization);
  }
  const ServiceMetrics& a = r.metrics.aggregate;
  std::printf("finished %zu unservable %zu slo_met %zu l_n_mean %.17g p99 %.17g ttft %.17g tpot %.17g\n", a.finished,
              a.unservable, a.slo_met, a.l_n_mean, a.p99_latency, a.avg_ttft, a.avg_tpot);
  std::uint64_t h = 1469598103934665603ull;
  for (const Request& q : r.requests) {
    double ft = q.finish_time ? *q.finish_time : -1.0;
    std::uint64_t bits;
    std::memcpy(&bits, &ft, 8);
    h = fnv(fnv(fnv(h, q.id), bits), (std::uint64_t)q.tokens_generated);
  }
  std::printf("request_hash %016" PRIx64 "\n", h);
  return 0;
}

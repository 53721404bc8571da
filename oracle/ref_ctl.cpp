// ref_ctl.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference control-plane code the unified-KV path is fed
// by, compiled from the read-only tree (g++ -I/root/reference/proj/include, oracle/Makefile):
//   * seasim::generate_trace (workload.hpp:181-212): the config-3 arrival trace;
//   * seasim::dedicated_plan (placement.hpp:284-319, with required_tp :37-46 and can_allocate
//     :129-156): the config-5 placement.
// No reference source is copied.  tests/test_ref_control.py diffs the Python restatements
// (paper_2504_15720_b200/churn.py generate_trace, placement.py dedicated_plan) against these.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "seasim/placement.hpp"  // /root/reference/proj/include/seasim/placement.hpp
#include "seasim/workload.hpp"

extern "C" {

// Profiles with Gaussian length distributions (LengthDist mean/stddev); shape_kind 0 constant,
// 1 step.  Writes up to cap records; returns the trace length (or -1 on a ConfigError).
long ref_generate_trace(int n_prof, const double* in_mean, const double* in_sd, const double* out_mean,
                        const double* out_sd, double rate, double duration, int skewness, uint64_t seed,
                        int shape_kind, double step_time, double step_factor, long cap, double* t, int* svc,
                        int* in_len, int* out_len) {
  std::vector<seasim::ServiceProfile> profiles(n_prof);
  for (int i = 0; i < n_prof; ++i) {
    profiles[i].name = "svc" + std::to_string(i);
    profiles[i].input_len_dist.mean = in_mean[i];
    profiles[i].input_len_dist.stddev = in_sd[i];
    profiles[i].output_len_dist.mean = out_mean[i];
    profiles[i].output_len_dist.stddev = out_sd[i];
  }
  seasim::RateProfile shape;
  if (shape_kind == 1) {
    shape.kind = seasim::RateProfile::Kind::kStep;
    shape.step_time = step_time;
    shape.step_factor = step_factor;
  }
  try {
    const seasim::Trace tr = seasim::generate_trace(profiles, rate, duration, skewness, seed, shape);
    for (long i = 0; i < (long)tr.records.size() && i < cap; ++i) {
      t[i] = tr.records[i].arrival_time;
      svc[i] = std::stoi(tr.records[i].service_id.substr(3));
      in_len[i] = tr.records[i].input_len;
      out_len[i] = tr.records[i].output_len;
    }
    return (long)tr.records.size();
  } catch (const seasim::ConfigError&) {
    return -1;
  }
}

// dedicated_plan over default_cost_model() plus caller-defined models (extra_*; their time
// coefficients are copies of llama2-7b's, only min_tp / heads / weights / activation matter
// to the placement) and overrides: min_tp per model, extra (model, tp) activation entries.
// Outputs: groups (tp, node, first gpu, services <= 32 each), unplaced services, feasible.
// Returns 0, or -1 when required_tp throws (InfeasibleError).
int ref_dedicated_plan(int n_svc, const char** svc_model, int gpus_per_node, int num_nodes, double mem_gib,
                       int share_cap, int replica_cap, double kv_reserve_gib, int batch_cap, int n_extra,
                       const char** ex_id, const int* ex_layers, const int* ex_heads, const double* ex_weight_gib,
                       const int* ex_min_tp, const int* ex_ntp, const double* ex_act /* [n_extra][4 tps][2] */,
                       int n_ovr, const char** ovr_id, const int* ovr_min_tp, int n_ent, const char** ent_id,
                       const int* ent_tp, const double* ent_act /* [n_ent][2] GiB */, int* n_groups, int* g_tp,
                       int* g_node, int* g_gpu0, int* g_nsvc, int* g_svcs, int* n_unplaced, int* unplaced,
                       int* feasible) {
  seasim::CostModel cm = seasim::default_cost_model();
  auto gib = [](double g) { return g * seasim::kGiB; };
  for (int i = 0; i < n_extra; ++i) {
    cm.add_model({.model_id = ex_id[i], .num_layers = ex_layers[i], .num_heads = ex_heads[i], .head_dim = 128,
                  .dtype_bytes = 2, .weight_bytes = gib(ex_weight_gib[i]), .min_tp = ex_min_tp[i]});
    for (int k = 0; k < ex_ntp[i]; ++k) {
      const int tp = 1 << k;
      cm.add_entry(ex_id[i], tp,
                   {2.0e-3, 8.0e-5, 6.0e-3, 4.0e-4, 2.5e-7, gib(ex_act[(i * 4 + k) * 2]), gib(ex_act[(i * 4 + k) * 2 + 1])});
    }
  }
  for (int i = 0; i < n_ovr; ++i) {
    seasim::ModelSpec m = cm.model(ovr_id[i]);
    m.min_tp = ovr_min_tp[i];
    cm.add_model(m);
  }
  for (int i = 0; i < n_ent; ++i)
    cm.add_entry(ent_id[i], ent_tp[i], {2.0e-3, 8.0e-5, 6.0e-3, 4.0e-4, 2.5e-7, gib(ent_act[2 * i]), gib(ent_act[2 * i + 1])});
  seasim::GpuSpec cluster;
  cluster.mem_bytes = gib(mem_gib);
  cluster.gpus_per_node = gpus_per_node;
  cluster.num_nodes = num_nodes;
  seasim::PlacementConfig pcfg;
  pcfg.share_cap = share_cap;
  pcfg.replica_cap = replica_cap;
  pcfg.kv_reserve_bytes = gib(kv_reserve_gib);
  std::vector<seasim::ServiceProfile> profiles(n_svc);
  for (int i = 0; i < n_svc; ++i) {
    profiles[i].name = "svc" + std::to_string(i);
    profiles[i].model_id = svc_model[i];
  }
  try {
    const seasim::PlacementPlan plan = seasim::dedicated_plan(cluster, cm, profiles, pcfg, batch_cap);
    *n_groups = (int)plan.groups.size();
    for (size_t g = 0; g < plan.groups.size(); ++g) {
      g_tp[g] = plan.groups[g].tp_size;
      g_node[g] = plan.groups[g].node_id;
      g_gpu0[g] = plan.groups[g].gpu_ids.empty() ? -1 : plan.groups[g].gpu_ids[0];
      g_nsvc[g] = (int)plan.groups[g].services.size();
      for (size_t s = 0; s < plan.groups[g].services.size() && s < 32; ++s) g_svcs[g * 32 + s] = (int)plan.groups[g].services[s];
    }
    *n_unplaced = (int)plan.unplaced.size();
    for (size_t i = 0; i < plan.unplaced.size(); ++i) unplaced[i] = (int)plan.unplaced[i];
    *feasible = plan.feasible ? 1 : 0;
    return 0;
  } catch (const seasim::InfeasibleError&) {
    return -1;
  }
}

}  // extern "C"

"""The control-plane restatements the hot path is fed by, pinned to the UNMODIFIED reference
compiled here (oracle/ref_ctl.cpp -> oracle/_ref/libref_ctl.so; skipped where the reference
was not built):

* churn.generate_trace  vs seasim::generate_trace (workload.hpp:181-212, LengthDist::sample
  :33-38 with std::llround) — identical traces over seeds, rates, skewness, step shapes;
* placement.dedicated_plan vs seasim::dedicated_plan (placement.hpp:284-319, required_tp
  :37-46, can_allocate :129-156) — identical groups / unplaced / feasibility for the config-5
  services under the reference defaults and the SURVEY §8e overrides.
"""
import pytest

import oracle_py as O
from paper_2504_15720_b200 import placement as PL
from paper_2504_15720_b200.churn import ServiceProfile, generate_trace, llround, paper_services

pytestmark = pytest.mark.skipif(not O.ref_ctl_available(), reason="reference control-plane shim not built")


def _ref_trace(prof, **kw):
    return O.ref_generate_trace([(p.in_mean, p.in_sd, p.out_mean, p.out_sd) for p in prof], **kw)


@pytest.mark.parametrize("seed", [1, 7, 2025, 2 ** 63 + 5])
@pytest.mark.parametrize("skew", [1, 4])
def test_generate_trace_matches_reference(seed, skew):
    prof = paper_services(4)
    ours = generate_trace(prof, rate=20.0, duration=60.0, skewness=skew, seed=seed)
    ref = _ref_trace(prof, rate=20.0, duration=60.0, skewness=skew, seed=seed)
    assert len(ours) == len(ref) > 100
    assert [(a.t, a.svc, a.in_len, a.out_len) for a in ours] == ref


@pytest.mark.parametrize("seed", [3, 11])
def test_generate_trace_step_profile_matches_reference(seed):
    prof = paper_services(4)
    ours = generate_trace(prof, rate=8.0, duration=40.0, skewness=4, seed=seed, step_time=20.0, step_factor=2.0)
    ref = _ref_trace(prof, rate=8.0, duration=40.0, skewness=4, seed=seed, step_time=20.0, step_factor=2.0)
    assert [(a.t, a.svc, a.in_len, a.out_len) for a in ours] == ref


def test_half_integer_lengths_round_like_llround():
    """Degenerate (sd 0) lengths at .5 hit the rounding rule directly: std::llround rounds half
    away from zero; Python's round() would give 2 and 72 here."""
    prof = [ServiceProfile("a", 0, 2.5, 0.0, 71.5, 0.0), ServiceProfile("b", 0, 3.5, 0.0, 0.5, 0.0)]
    ours = generate_trace(prof, rate=5.0, duration=10.0, skewness=1, seed=9)
    ref = _ref_trace(prof, rate=5.0, duration=10.0, skewness=1, seed=9)
    assert [(a.t, a.svc, a.in_len, a.out_len) for a in ours] == ref
    assert {(a.in_len, a.out_len) for a in ours} == {(3, 72), (4, 1)}
    assert llround(2.5) == 3 and llround(-2.5) == -3


_EXTRA = [(mid, m.num_layers, m.num_heads, m.weight_gib, m.min_tp, m.activation)
          for mid, m in PL.MODELS.items() if mid in ("llama3-8b", "mistral-7b")]


def _ref_plan(services, cfg):
    return O.ref_dedicated_plan(services, cfg.gpus_per_node, cfg.num_nodes, cfg.gpu_mem_gib, cfg.share_cap,
                                cfg.replica_cap, cfg.kv_reserve_gib, cfg.batch_cap, extra_models=_EXTRA,
                                min_tp_override=cfg.min_tp_override, extra_entries=cfg.extra_tp_entries)


def _ours(services, cfg):
    try:
        plan = PL.dedicated_plan(services, cfg)
    except RuntimeError:
        return None
    return ([(g.tp_size, g.node_id, g.gpu_ids[0], list(g.services)) for g in plan.groups], list(plan.unplaced),
            plan.feasible)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_dedicated_plan_config5_overrides_match_reference(n):
    services = PL.config5_services()
    cfg = PL.config5_overrides(n)
    assert _ours(services, cfg) == _ref_plan(services, cfg)


@pytest.mark.parametrize("gpus,mem,share", [(4, 80.0, 2), (8, 80.0, 2), (8, 178.8, 2), (8, 178.8, 3), (2, 80.0, 2),
                                            (8, 40.0, 4)])
def test_dedicated_plan_reference_defaults_match_reference(gpus, mem, share):
    """Reference defaults (share_cap 2, 80 GiB GPUs) and variations, incl. the infeasible cases
    SURVEY §8e lists (2 GPUs: required_tp throws for the 70B shape)."""
    services = PL.config5_services()
    cfg = PL.PlacementConfig(share_cap=share, gpus_per_node=gpus, gpu_mem_gib=mem)
    assert _ours(services, cfg) == _ref_plan(services, cfg)


@pytest.mark.parametrize("seed", range(6))
def test_dedicated_plan_random_mixes_match_reference(seed):
    import numpy as np
    rng = np.random.default_rng(seed)
    ids = list(PL.MODELS)
    services = [ids[int(i)] for i in rng.integers(0, len(ids), int(rng.integers(1, 24)))]
    cfg = PL.PlacementConfig(share_cap=int(rng.integers(1, 6)), gpus_per_node=int(rng.choice([1, 2, 4, 8])),
                             num_nodes=int(rng.integers(1, 3)), gpu_mem_gib=float(rng.choice([40.0, 80.0, 178.8])),
                             replica_cap=int(rng.integers(0, 3)), batch_cap=int(rng.choice([8, 16, 64])))
    assert _ours(services, cfg) == _ref_plan(services, cfg)

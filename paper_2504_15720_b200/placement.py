"""Services -> GPUs for the unified KV path.

Restates the parts of the reference placement that decide which services share
one pool and at which TP size (host-side, no GPU):

* ``SharingGroup``               placement_plan.hpp:17-26
* ``required_tp``                placement.hpp:37-46  (smallest power-of-two TP >= min_tp
                                 dividing num_heads, fitting a node, with a cost entry)
* ``can_allocate``               placement.hpp:129-156 (share cap, replica cap, TP fit,
                                 per-GPU memory = Σ weights/tp + max activation + kv/tp)
* ``dedicated_plan``             placement.hpp:284-319 (first-fit dedicated groups, then
                                 join an existing group when the cap and memory allow)

plus ``rank_role`` which turns a plan into the per-process role of one rank
(its group, its TP rank, the services whose KV it holds).  The model table is
the reference's ``default_cost_model`` (cost_model.hpp:191-262) extended with the
GQA shapes of the BASELINE configs (Llama-3-8B / Mistral-7B, which the reference
would add through ``[model <id>]`` INI sections, config.hpp:295-310).
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence

GiB = 1024.0 ** 3


@dataclasses.dataclass(frozen=True)
class ModelClass:
    model_id: str
    num_layers: int
    num_heads: int       # KV heads (sizes the native block)
    num_q_heads: int
    weight_gib: float
    min_tp: int
    # tp -> (activation_base GiB, activation_per_seq GiB); presence == "has cost entry"
    activation: Dict[int, tuple]


_ACT7 = {1: (0.8, 0.03), 2: (0.5, 0.02), 4: (0.35, 0.013), 8: (0.25, 0.009)}
MODELS: Dict[str, ModelClass] = {
    "llama2-7b": ModelClass("llama2-7b", 32, 32, 32, 14.0, 1, _ACT7),
    "llama2-13b": ModelClass("llama2-13b", 40, 40, 40, 26.0, 1,
                             {1: (1.1, 0.045), 2: (0.7, 0.028), 4: (0.5, 0.018), 8: (0.35, 0.012)}),
    "llama2-70b": ModelClass("llama2-70b", 80, 64, 64, 140.0, 4, {4: (1.4, 0.055), 8: (0.9, 0.035)}),
    "opt-6.7b": ModelClass("opt-6.7b", 32, 32, 32, 13.4, 1,
                           {1: (0.8, 0.03), 2: (0.5, 0.02), 4: (0.35, 0.013), 8: (0.25, 0.009)}),
    "llama3-8b": ModelClass("llama3-8b", 32, 8, 32, 16.0, 1, _ACT7),
    "mistral-7b": ModelClass("mistral-7b", 32, 8, 32, 14.5, 1, _ACT7),
}


@dataclasses.dataclass
class SharingGroup:
    services: List[int]
    gpu_ids: List[int]
    tp_size: int = 1
    node_id: int = 0

    def serves(self, svc: int) -> bool:
        return svc in self.services


@dataclasses.dataclass
class PlacementPlan:
    groups: List[SharingGroup]
    unplaced: List[int]
    feasible: bool


@dataclasses.dataclass
class PlacementConfig:
    share_cap: int = 2              # placement.hpp:19
    replica_cap: int = 0
    kv_reserve_gib: float = 4.0
    gpus_per_node: int = 8
    num_nodes: int = 1
    gpu_mem_gib: float = 178.8      # B200 (the reference default is 80 GiB)
    batch_cap: int = 16              # [scheduler] batch_cap default (config.hpp:349)
    min_tp_override: Optional[Dict[str, int]] = None
    extra_tp_entries: Optional[Dict[str, Dict[int, tuple]]] = None


def _activation(m: ModelClass, tp: int, cfg: PlacementConfig):
    ent = dict(m.activation)
    if cfg.extra_tp_entries and m.model_id in cfg.extra_tp_entries:
        ent.update(cfg.extra_tp_entries[m.model_id])
    return ent.get(tp)


def _min_tp(m: ModelClass, cfg: PlacementConfig) -> int:
    if cfg.min_tp_override and m.model_id in cfg.min_tp_override:
        return cfg.min_tp_override[m.model_id]
    return m.min_tp


def required_tp(m: ModelClass, cfg: PlacementConfig) -> int:
    """placement.hpp:37-46"""
    tp = 1
    while tp <= cfg.gpus_per_node:
        if tp >= _min_tp(m, cfg) and m.num_heads % tp == 0 and _activation(m, tp, cfg) is not None:
            return tp
        tp *= 2
    raise RuntimeError(f"InfeasibleError: model {m.model_id} fits no TP size up to {cfg.gpus_per_node} GPUs")


def memory_footprint_gib(model_ids: Sequence[str], tp: int, kv_gib: float, cfg: PlacementConfig) -> float:
    """cost_model.hpp memory_footprint: Σ weights/tp + max activation(batch_cap) + kv/tp."""
    w = act = 0.0
    for mid in model_ids:
        m = MODELS[mid]
        w += m.weight_gib / tp
        base, per = _activation(m, tp, cfg)
        act = max(act, base + per * cfg.batch_cap)
    return w + act + kv_gib / tp


def can_allocate(group: SharingGroup, svc: int, services: Sequence[str], cfg: PlacementConfig,
                 plan: PlacementPlan) -> bool:
    """placement.hpp:129-156"""
    if group.serves(svc) or len(group.services) >= cfg.share_cap:
        return False
    if cfg.replica_cap > 0 and sum(g.serves(svc) for g in plan.groups) >= cfg.replica_cap:
        return False
    m = MODELS[services[svc]]
    if m.num_heads % group.tp_size or group.tp_size < _min_tp(m, cfg) or _activation(m, group.tp_size, cfg) is None:
        return False
    mids = []
    for s in group.services + [svc]:
        if services[s] not in mids:
            mids.append(services[s])
    return memory_footprint_gib(mids, group.tp_size, cfg.kv_reserve_gib, cfg) <= cfg.gpu_mem_gib


def dedicated_plan(services: Sequence[str], cfg: PlacementConfig) -> PlacementPlan:
    """placement.hpp:284-319: `services` lists each service's model id."""
    plan = PlacementPlan([], [], True)
    next_free = [0] * cfg.num_nodes
    for svc, mid in enumerate(services):
        tp = required_tp(MODELS[mid], cfg)
        placed = False
        for node in range(cfg.num_nodes):
            if next_free[node] + tp > cfg.gpus_per_node:
                continue
            g = SharingGroup([svc], [node * cfg.gpus_per_node + next_free[node] + k for k in range(tp)], tp, node)
            next_free[node] += tp
            plan.groups.append(g)
            placed = True
            break
        if not placed:
            for g in plan.groups:
                if can_allocate(g, svc, services, cfg, plan):
                    g.services.append(svc)
                    placed = True
                    break
        if not placed:
            plan.unplaced.append(svc)
            plan.feasible = False
    return plan


@dataclasses.dataclass
class RankRole:
    rank: int
    group_index: int
    group: SharingGroup
    tp_rank: int
    services: List[int]


def rank_role(plan: PlacementPlan, rank: int) -> Optional[RankRole]:
    """The group a GPU (= process rank) belongs to, and its position in the TP group."""
    for gi, g in enumerate(plan.groups):
        if rank in g.gpu_ids:
            return RankRole(rank, gi, g, g.gpu_ids.index(rank), list(g.services))
    return None


def config5_services(n_small: int = 15) -> List[str]:
    """Config 5: one 70B-shape service + 15 mixed services."""
    small = ["llama2-7b", "llama2-13b", "opt-6.7b", "llama3-8b"]
    return ["llama2-70b"] + [small[i % len(small)] for i in range(n_small)]


def config5_overrides(n_gpus: int) -> PlacementConfig:
    """The overrides that make config 5 feasible."""
    if n_gpus >= 8:
        return PlacementConfig(share_cap=4, gpus_per_node=8)
    if n_gpus == 4:
        return PlacementConfig(share_cap=16, gpus_per_node=4)
    if n_gpus == 2:
        return PlacementConfig(share_cap=16, gpus_per_node=2, min_tp_override={"llama2-70b": 2},
                               extra_tp_entries={"llama2-70b": {2: (2.0, 0.08)}})
    # one GPU cannot hold the 16 services' weights (~370 GiB): the 1-GPU point of the
    # scaling curve is a KV-path-only run (weights not resident), so the memory check is off
    return PlacementConfig(share_cap=16, gpus_per_node=1, min_tp_override={"llama2-70b": 1},
                           extra_tp_entries={"llama2-70b": {1: (2.8, 0.11)}}, gpu_mem_gib=1e9)

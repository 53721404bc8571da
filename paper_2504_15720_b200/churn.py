"""Config 3 — bursty multi-service churn over the unified pool (SURVEY §8d cfg 3).

A serving-iteration driver that exercises every hot-path operation the way an
engine does: Poisson arrivals in service runs (the reference trace generator,
workload.hpp:150-212), admission while pool occupancy is below a target
(70 %), chunked prefill (C tokens per iteration: grow -> KV append -> causal
prefill attention on tcgen05), decode (+1 token: grow -> append -> paged decode
attention), frees of finished requests, and preemption on CacheFull
(simulation.hpp:144-157,333-340: evict -> free_request -> re-prefill later).

Every allocator call is recorded as a KvOp (kv_cache.hpp:270-275) so the exact
stream can be replayed through the oracle / the reference to prove the GPU
block tables bit-exact.  Only the control flow lives here (Python); every
allocation, append and attention runs through libseakv.
"""
from __future__ import annotations

import dataclasses
import math
import time
from typing import Dict, List, Optional, Sequence

import torch

from .kvcache import Batch, UnifiedKvCache

M64 = (1 << 64) - 1


class Rng:
    """SplitMix64 with the reference's draw functions (common.hpp:41-74)."""

    def __init__(self, seed: int):
        self.s = seed & M64

    def next_u64(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def exponential(self, rate: float) -> float:
        return -math.log(1.0 - self.next_double()) / rate

    def gaussian(self, mean: float, sd: float) -> float:
        u1 = 1.0 - self.next_double()
        u2 = self.next_double()
        return mean + sd * math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586 * u2)


@dataclasses.dataclass
class ServiceProfile:
    name: str
    model_idx: int
    in_mean: float
    in_sd: float
    out_mean: float
    out_sd: float

    def sample(self, rng: Rng, mean: float, sd: float) -> int:  # LengthDist::sample, workload.hpp:33-38
        if sd == 0.0:
            return max(1, int(round(mean)))
        return max(1, int(round(rng.gaussian(mean, sd))))


def paper_services(n_models: int) -> List[ServiceProfile]:
    """Table 1: chat (ShareGPT 73.0 in / 426.9 out) and
    summarisation (LongBench 13186.8 in / 21.1 out), one of each per model."""
    out = []
    for m in range(n_models):
        out.append(ServiceProfile(f"chat{m}", m, 73.0, 40.0, 426.9, 200.0))
        out.append(ServiceProfile(f"summ{m}", m, 13186.8, 3000.0, 21.1, 8.0))
    return out


@dataclasses.dataclass
class Arrival:
    t: float
    svc: int
    in_len: int
    out_len: int


def generate_trace(profiles: Sequence[ServiceProfile], rate: float, duration: float, skewness: int, seed: int,
                   step_time: Optional[float] = None, step_factor: float = 1.0) -> List[Arrival]:
    """workload.hpp:181-212 with RateProfile::kStep (:150-176)."""
    arrivals, lengths = Rng(seed), Rng(seed ^ 0x5EED5EED5EED5EED)
    peak = rate * (max(1.0, step_factor) if step_time is not None else 1.0)
    t, run, out = 0.0, 0, []
    while True:
        t += arrivals.exponential(peak)
        if t >= duration:
            break
        if step_time is not None:
            factor = step_factor if t >= step_time else 1.0
            if arrivals.next_double() >= rate * factor / peak:
                continue
        svc = (run // skewness) % len(profiles)
        run += 1
        p = profiles[svc]
        out.append(Arrival(t, svc, p.sample(lengths, p.in_mean, p.in_sd), p.sample(lengths, p.out_mean, p.out_sd)))
    return out


@dataclasses.dataclass
class Req:
    rid: int
    svc: int
    model: int
    in_len: int
    out_len: int
    done: int = 0       # prompt tokens prefilled
    generated: int = 0  # output tokens generated
    phase: str = "waiting"


class ChurnEngine:
    def __init__(self, cache: UnifiedKvCache, shapes: Sequence[tuple], profiles: Sequence[ServiceProfile],
                 chunk: int = 512, occupancy: float = 0.70, max_decode: int = 512, max_prefill: int = 8,
                 layers: Optional[int] = None, stream=None, seed: int = 7):
        self.cache, self.shapes, self.profiles = cache, list(shapes), list(profiles)
        self.chunk, self.occupancy = chunk, occupancy
        self.max_decode, self.max_prefill = max_decode, max_prefill
        self.nlayers = layers or max(L for L, _, _ in shapes)
        self.stream = stream
        self.ops: List[tuple] = []  # KvOp record: (kind, id, model, tokens)
        self.waiting: List[Req] = []
        self.running: Dict[int, Req] = {}
        self.next_id = 1
        self.dtype = torch.float16
        g = torch.Generator(device="cuda").manual_seed(seed)
        M = len(shapes)
        # synthetic activations, sliced per iteration (contents are irrelevant to the KV path)
        self.q_dec = [torch.randn((max_decode, Hq, 128), generator=g, device="cuda").half() for _, _, Hq in shapes]
        self.o_dec = [torch.empty_like(x) for x in self.q_dec]
        self.kv_dec = [torch.randn((max_decode, 1, H, 128), generator=g, device="cuda").half() for _, H, _ in shapes]
        self.q_pre = [torch.randn((max_prefill, chunk, Hq, 128), generator=g, device="cuda").half()
                      for _, _, Hq in shapes]
        self.o_pre = [torch.empty_like(x) for x in self.q_pre]
        self.kv_pre = [torch.randn((max_prefill, chunk, H, 128), generator=g, device="cuda").half()
                       for _, H, _ in shapes]
        self._dec_batch: Optional[Batch] = None
        self._pre_batches: Dict[int, Batch] = {}
        self.stats = dict(iterations=0, grow_ops=0, free_ops=0, preemptions=0, alloc_s=0.0, append_ms=0.0,
                          decode_ms=0.0, prefill_ms=0.0, decode_bytes=0.0, append_bytes=0.0, data_path_ms=0.0,
                          prefill_flops=0.0,
                          occupancy_sum=0.0, finished=0, admitted=0, cache_full=0)
        self.M = M

    # -- allocator calls, recorded -----------------------------------------------------------
    def _grow(self, r: Req, tokens: int) -> bool:
        self.ops.append((0, r.rid, r.model, tokens))
        self.stats["grow_ops"] += 1
        return self.cache.try_allocate(r.rid, r.model, tokens)

    def _free(self, r: Req):
        self.ops.append((1, r.rid, r.model, 0))
        self.stats["free_ops"] += 1
        self.cache.free_request(r.rid)

    def add_arrivals(self, arrivals: Sequence[Arrival]):
        for a in arrivals:
            p = self.profiles[a.svc]
            self.waiting.append(Req(self.next_id, a.svc, p.model_idx, a.in_len, a.out_len))
            self.next_id += 1

    def _batch(self, key, groups):
        if key == "dec":
            if self._dec_batch is None:
                self._dec_batch = self.cache.batch(groups)
            else:
                self._dec_batch.reset(groups)
            return self._dec_batch
        b = self._pre_batches.get(key)
        if b is None:
            b = self._pre_batches[key] = self.cache.batch(groups)
        else:
            b.reset(groups)
        return b

    # -- steady-state start -------------------------------------------------------------------
    def warm_start(self, arrivals: Sequence[Arrival], seed: int = 11) -> int:
        """Bring the pool to the occupancy target before timing: requests from ``arrivals``
        (in order) are admitted as already prefilled -- one grow to their input length plus
        a seeded part of their output, K/V from the pool's synthetic fill -- and join the
        decode set while they fit under the target; one that does not fit joins the waiting
        queue (normal admission later).  Stops once the pool is within 5 % of the target.
        Returns the number of arrivals consumed.  The grows are recorded like every other
        allocator call."""
        cache, pool = self.cache, self.cache.pool_size()
        target = self.occupancy * pool
        rng = Rng(seed)
        used = 0
        for a in arrivals:
            if cache.allocated_blocks() >= 0.95 * target or len(self.running) >= self.max_decode:
                break
            used += 1
            p = self.profiles[a.svc]
            r = Req(self.next_id, a.svc, p.model_idx, a.in_len, a.out_len)
            self.next_id += 1
            gen = 1 + int(rng.next_double() * max(0, a.out_len - 1))
            # gen tokens generated, gen - 1 of them already fed back (their K/V cached)
            need = cache.native_blocks_for(r.in_len + gen - 1) / max(1, cache.sub_slots_per_merged(r.model))
            if cache.allocated_blocks() + need > target or not self._grow(r, r.in_len + gen - 1):
                self.waiting.append(r)
                continue
            r.phase, r.done, r.generated = "decode", r.in_len, gen
            self.running[r.rid] = r
        self.cache.flush(self.stream)
        return used

    def reset_stats(self) -> None:
        """Zero the counters (the recorded KvOp stream is kept)."""
        for k in self.stats:
            self.stats[k] = 0.0 if isinstance(self.stats[k], float) else 0

    # -- one serving iteration ------------------------------------------------------------------
    def step(self) -> dict:
        cache, st = self.cache, self.stats
        t0 = time.perf_counter()
        pool = cache.pool_size()
        # admission (FCFS) while occupancy is below target
        prefill = [r for r in self.running.values() if r.phase == "prefill"]
        while self.waiting and len(prefill) < self.max_prefill and \
                cache.allocated_blocks() < self.occupancy * pool:
            r = self.waiting.pop(0)
            r.phase, r.done, r.generated = "prefill", 0, 0
            self.running[r.rid] = r
            prefill.append(r)
            st["admitted"] += 1
        # decode growth: the last generated token is fed back, so the cache holds prompt +
        # generated tokens (+1 per step); CacheFull -> preempt (free + re-queue for re-prefill)
        decode = [r for r in self.running.values() if r.phase == "decode"][: self.max_decode]
        dec_ok = []
        for r in decode:
            if self._grow(r, r.in_len + r.generated):
                dec_ok.append(r)
            else:
                st["cache_full"] += 1
                st["preemptions"] += 1
                self._free(r)
                del self.running[r.rid]
                r.phase = "waiting"
                self.waiting.insert(0, r)
        # prefill chunk growth
        pre_ok: Dict[int, List[Req]] = {}
        for r in prefill:
            c = min(self.chunk, r.in_len - r.done)
            if self._grow(r, r.done + c):
                pre_ok.setdefault(c, []).append(r)
            else:
                st["cache_full"] += 1
        cache.flush(self.stream)
        st["alloc_s"] += time.perf_counter() - t0
        # data path over every layer index
        ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        marks = []
        span = [ev(), ev()]  # GPU time of the whole data path of this step
        span[0].record(self.stream)
        if dec_ok:
            groups = [(m, [r.rid for r in dec_ok if r.model == m]) for m in range(self.M)]
            groups = [g for g in groups if g[1]]
            b = self._batch("dec", groups)
            q = [self.q_dec[m][: len(ids)] for m, ids in groups]
            o = [self.o_dec[m][: len(ids)] for m, ids in groups]
            kv = [self.kv_dec[m][: len(ids)] for m, ids in groups]
            # one launch per layer: the new token's K/V is appended inside the decode kernel
            # (fused append); the layer loop is bracketed by one pair of events, so decode_ms
            # is the GPU span of the decode phase (host submission runs ahead of it)
            e = [ev(), ev(), ev()]
            e[0].record(self.stream)
            e[1].record(self.stream)
            for layer in range(self.nlayers):
                b.decode(q, o, layer, stream=self.stream, k=kv, v=kv)
            e[2].record(self.stream)
            marks.append(("dec", e))
            for layer in range(self.nlayers):
                kvb, _ = b.decode_bytes(layer)
                st["decode_bytes"] += kvb
        for c, rs in pre_ok.items():
            groups = [(m, [r.rid for r in rs if r.model == m]) for m in range(self.M)]
            groups = [g for g in groups if g[1]]
            b = self._batch(c, groups)
            q = [self.q_pre[m][: len(ids), :c] for m, ids in groups]
            o = [self.o_pre[m][: len(ids), :c] for m, ids in groups]
            kv = [self.kv_pre[m][: len(ids), :c] for m, ids in groups]
            q = [x.contiguous() for x in q]
            o = [torch.empty_like(x) for x in q]
            kv = [x.contiguous() for x in kv]
            for layer in range(self.nlayers):
                e = [ev(), ev(), ev()]
                e[0].record(self.stream)
                b.append(kv, kv, layer, c, self.stream)
                e[1].record(self.stream)
                b.prefill(q, o, layer, c, stream=self.stream)
                e[2].record(self.stream)
                marks.append(("pre", e))
            for r in rs:
                L, H, Hq = self.shapes[r.model]
                p0 = r.done
                st["prefill_flops"] += 4.0 * 128 * Hq * L * (c * p0 + c * (c + 1) / 2)
                st["append_bytes"] += c * L * 2 * H * 128 * 2 * 2
        span[1].record(self.stream)
        torch.cuda.synchronize()
        st["data_path_ms"] += span[0].elapsed_time(span[1])
        for kind, e in marks:
            st["append_ms"] += e[0].elapsed_time(e[1])
            st["decode_ms" if kind == "dec" else "prefill_ms"] += e[1].elapsed_time(e[2])
        # bookkeeping: finished requests are freed
        t1 = time.perf_counter()
        for r in dec_ok:
            r.generated += 1
            if r.generated >= r.out_len:
                self._free(r)
                del self.running[r.rid]
                st["finished"] += 1
        for c, rs in pre_ok.items():
            for r in rs:
                r.done += c
                if r.done >= r.in_len:
                    r.phase, r.generated = "decode", 1  # the prefill iteration emits token 1
                    if r.generated >= r.out_len:
                        self._free(r)
                        del self.running[r.rid]
                        st["finished"] += 1
        st["alloc_s"] += time.perf_counter() - t1
        st["iterations"] += 1
        st["occupancy_sum"] += cache.allocated_blocks() / max(1, pool)
        return st

    def summary(self) -> dict:
        st = self.stats
        it = max(1, st["iterations"])
        return {
            "iterations": st["iterations"], "admitted": st["admitted"], "finished": st["finished"],
            "preemptions": st["preemptions"], "cache_full": st["cache_full"],
            "grow_ops": st["grow_ops"], "free_ops": st["free_ops"],
            "alloc_ops_per_s": round((st["grow_ops"] + st["free_ops"]) / max(st["alloc_s"], 1e-9), 1),
            "mean_occupancy": round(st["occupancy_sum"] / it, 4),
            "decode_GBps": round(st["decode_bytes"] / max(st["decode_ms"], 1e-9) / 1e6, 1),
            # prefill-chunk appends (a decode step's append is fused into its decode launch)
            "append_GBps": round(st["append_bytes"] / max(st["append_ms"], 1e-9) / 1e6, 1),
            "prefill_TFLOPs": round(st["prefill_flops"] / max(st["prefill_ms"], 1e-9) / 1e9, 1),
            "decode_ms": round(st["decode_ms"], 2), "prefill_ms": round(st["prefill_ms"], 2),
            "append_ms": round(st["append_ms"], 2), "data_path_ms": round(st["data_path_ms"], 2),
        }


# ------------------------------------------------------------------ persisted formats --
TRACE_HEADER = "arrival_time,service_id,input_len,output_len"  # workload.hpp:214
OPS_HEADER = "kind,request_id,model_idx,tokens"                 # KvOp, kv_cache.hpp:270-275


def save_trace(arrivals: Sequence[Arrival], profiles: Sequence[ServiceProfile], path: str) -> None:
    """The reference's trace CSV (save_trace, workload.hpp:216-225)."""
    with open(path, "w") as f:
        f.write(TRACE_HEADER + "\n")
        for a in arrivals:
            f.write(f"{a.t:.6f},{profiles[a.svc].name},{a.in_len},{a.out_len}\n")


def load_trace(path: str, profiles: Sequence[ServiceProfile]) -> List[Arrival]:
    """load_trace (workload.hpp:227-265): header check, 4 fields, lengths >= 1, monotone time."""
    by_name = {p.name: i for i, p in enumerate(profiles)}
    out: List[Arrival] = []
    with open(path) as f:
        lines = f.read().splitlines()
    if not lines or lines[0].rstrip("\r") != TRACE_HEADER:
        raise ValueError(f"{path}:1: bad header, expected '{TRACE_HEADER}'")
    prev = -1.0
    for n, line in enumerate(lines[1:], start=2):
        line = line.rstrip("\r")
        if not line:
            continue
        parts = line.split(",")
        if len(parts) != 4:
            raise ValueError(f"{path}:{n}: expected 4 comma-separated fields")
        t, svc, il, ol = float(parts[0]), parts[1], int(parts[2]), int(parts[3])
        if il < 1 or ol < 1:
            raise ValueError(f"{path}:{n}: lengths must be >= 1")
        if t < prev:
            raise ValueError(f"{path}:{n}: non-monotone arrival_time")
        if svc not in by_name:
            raise ValueError(f"{path}:{n}: unknown service '{svc}'")
        prev = t
        out.append(Arrival(t, by_name[svc], il, ol))
    return out


def save_ops(ops: Sequence[tuple], path: str) -> None:
    """KvOp stream as CSV: kind (0 grow, 1 free), request id, model index, tokens."""
    with open(path, "w") as f:
        f.write(OPS_HEADER + "\n")
        for kind, rid, m, tok in ops:
            f.write(f"{kind},{rid},{m},{tok}\n")


def load_ops(path: str) -> List[tuple]:
    with open(path) as f:
        lines = f.read().splitlines()
    if not lines or lines[0] != OPS_HEADER:
        raise ValueError(f"{path}:1: bad header, expected '{OPS_HEADER}'")
    return [tuple(int(x) for x in line.split(",")) for line in lines[1:] if line]

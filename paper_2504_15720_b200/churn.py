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

import numpy as np
import torch

from .kvcache import KVOP_DTYPE, Batch, UnifiedKvCache

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
            return max(1, llround(mean))
        return max(1, llround(rng.gaussian(mean, sd)))


def llround(x: float) -> int:
    """std::llround: nearest integer, halfway cases away from zero (Python's round() rounds
    them to even)."""
    a = abs(x)
    r = math.floor(a)  # a - r is exact in binary floating point (x + 0.5 is not)
    r = int(r) + (1 if a - r >= 0.5 else 0)
    return r if x >= 0 else -r


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
    """Host-driven serving loop over one unified pool.  Per iteration: admission (FCFS while the
    pool is below the occupancy target), the decode step's +1-token grows and the prefill
    chunks' grows as ONE batched allocator call each (skv_replay), preemption of decode
    requests that hit CacheFull (free -> re-queue -> re-prefill from token 0,
    simulation.hpp:144-157,333-340), then per layer one fused append+decode launch and one
    ragged append + one ragged causal-prefill launch (every prefill chunk of the iteration,
    whatever its length), then the frees of finished requests.  GPU timings are resolved
    lazily (no per-iteration synchronize); the host still waits once per iteration for the
    emptied-block counts of the previous iteration's frees before its next grows."""

    def __init__(self, cache: UnifiedKvCache, shapes: Sequence[tuple], profiles: Sequence[ServiceProfile],
                 chunk: int = 512, occupancy: float = 0.70, max_decode: int = 512, max_prefill: int = 8,
                 layers: Optional[int] = None, stream=None, seed: int = 7, io: bool = False):
        self.cache, self.shapes, self.profiles = cache, list(shapes), list(profiles)
        self.io = io  # e2e: every decode step copies its per-layer q/k/v in from pinned host memory and
        #              every layer's output back (prefill activations stay device-resident)
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
        # synthetic activations, sliced per iteration (contents are irrelevant to the KV path);
        # prefill buffers are packed by request: [sum of the iteration's chunk lengths, heads, d]
        self.q_dec = [torch.randn((max_decode, Hq, 128), generator=g, device="cuda").half() for _, _, Hq in shapes]
        self.o_dec = [torch.empty_like(x) for x in self.q_dec]
        self.kv_dec = [torch.randn((max_decode, 1, H, 128), generator=g, device="cuda").half() for _, H, _ in shapes]
        self.q_pre = [torch.randn((max_prefill * chunk, Hq, 128), generator=g, device="cuda").half()
                      for _, _, Hq in shapes]
        self.o_pre = [torch.empty_like(x) for x in self.q_pre]
        self.kv_pre = [torch.randn((max_prefill * chunk, H, 128), generator=g, device="cuda").half()
                       for _, H, _ in shapes]
        if io:  # per-layer decode activations: pinned host <-> device staging
            L = self.nlayers
            self.h_q = [torch.randn((L, max_decode, Hq, 128), generator=g, device="cuda").half().cpu().pin_memory()
                        for _, _, Hq in shapes]
            self.h_kv = [torch.randn((L, max_decode, 1, H, 128), generator=g, device="cuda").half().cpu().pin_memory()
                         for _, H, _ in shapes]
            self.h_o = [torch.empty((L, max_decode, Hq, 128), dtype=torch.float16).pin_memory() for _, _, Hq in shapes]
            self.d_q = [torch.empty(x.shape, dtype=x.dtype, device="cuda") for x in self.h_q]
            self.d_kv = [torch.empty(x.shape, dtype=x.dtype, device="cuda") for x in self.h_kv]
            self.d_o = [torch.empty(x.shape, dtype=x.dtype, device="cuda") for x in self.h_o]
        self._dec_batch: Optional[Batch] = None
        self._pre_batch: Optional[Batch] = None
        self._marks: List[tuple] = []  # (kind, events) resolved by summary()
        self.stats = dict(iterations=0, grow_ops=0, free_ops=0, preemptions=0, reprefilled=0, alloc_s=0.0,
                          append_ms=0.0, decode_ms=0.0, prefill_ms=0.0, decode_bytes=0.0, append_bytes=0.0,
                          data_path_ms=0.0, prefill_flops=0.0, occupancy_sum=0.0, finished=0, admitted=0,
                          cache_full=0, prefill_launches=0, h2d_bytes=0.0, d2h_bytes=0.0)
        self.M = M
        self.preempted_ids: set = set()

    # -- allocator calls, recorded (one C-ABI call per batch) ---------------------------------
    def _replay(self, kind: int, reqs: Sequence[Req], tokens: Sequence[int]) -> np.ndarray:
        n = len(reqs)
        if n == 0:
            return np.zeros(0, dtype=bool)
        arr = np.zeros(n, dtype=KVOP_DTYPE)
        arr["kind"] = kind
        arr["model"] = [r.model for r in reqs]
        arr["id"] = [r.rid for r in reqs]
        arr["tokens"] = tokens
        self.ops.extend((kind, r.rid, r.model, int(t)) for r, t in zip(reqs, tokens))
        self.stats["grow_ops" if kind == 0 else "free_ops"] += n
        return self.cache.replay_array(arr).astype(bool)

    def _grow_many(self, reqs: Sequence[Req], tokens: Sequence[int]) -> np.ndarray:
        return self._replay(0, reqs, tokens)

    def _free_many(self, reqs: Sequence[Req]) -> None:
        self._replay(1, reqs, [0] * len(reqs))

    # single-op forms (warm start)
    def _grow(self, r: Req, tokens: int) -> bool:
        return bool(self._grow_many([r], [tokens])[0])

    def add_arrivals(self, arrivals: Sequence[Arrival]):
        for a in arrivals:
            p = self.profiles[a.svc]
            self.waiting.append(Req(self.next_id, a.svc, p.model_idx, a.in_len, a.out_len))
            self.next_id += 1

    def _batch(self, attr: str, groups):
        b = getattr(self, attr)
        if b is None:
            b = self.cache.batch(groups)
            setattr(self, attr, b)
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
        self._resolve()
        self._marks = []
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
        # decode growth (one batched call): the last generated token is fed back, so the cache
        # holds prompt + generated tokens (+1 per step); CacheFull -> preempt: free + re-queue
        # at the head of the waiting queue, re-prefilled from token 0 when re-admitted
        decode = [r for r in self.running.values() if r.phase == "decode"][: self.max_decode]
        ok = self._grow_many(decode, [r.in_len + r.generated for r in decode])
        dec_ok = [r for r, g in zip(decode, ok) if g]
        victims = [r for r, g in zip(decode, ok) if not g]
        if victims:
            st["cache_full"] += len(victims)
            st["preemptions"] += len(victims)
            self._free_many(victims)
            for r in reversed(victims):
                del self.running[r.rid]
                r.phase = "waiting"
                self.preempted_ids.add(r.rid)
                self.waiting.insert(0, r)
        # prefill chunk growth (one batched call)
        chunks = [min(self.chunk, r.in_len - r.done) for r in prefill]
        ok = self._grow_many(prefill, [r.done + c for r, c in zip(prefill, chunks)])
        pre_ok = [(r, c) for r, c, g in zip(prefill, chunks, ok) if g]
        st["cache_full"] += int(len(prefill) - len(pre_ok))
        cache.flush(self.stream)
        st["alloc_s"] += time.perf_counter() - t0
        # data path over every layer index
        ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
        span = [ev(), ev()]  # GPU span of the whole data path of this step
        span[0].record(self.stream)
        if dec_ok:
            groups = [(m, [r.rid for r in dec_ok if r.model == m]) for m in range(self.M)]
            groups = [g for g in groups if g[1]]
            b = self._batch("_dec_batch", groups)
            q = [self.q_dec[m][: len(ids)] for m, ids in groups]
            o = [self.o_dec[m][: len(ids)] for m, ids in groups]
            kv = [self.kv_dec[m][: len(ids)] for m, ids in groups]
            # one launch per layer: the new token's K/V is appended inside the decode kernel
            # (fused append); bracketed by one pair of events = GPU span of the decode phase
            e = [ev(), ev(), ev()]
            e[0].record(self.stream)
            if self.io:  # this step's q / new K,V of every layer from pinned host memory
                with torch.cuda.stream(self.stream):
                    for (m, ids) in groups:
                        n = len(ids)
                        self.d_q[m][:, :n].copy_(self.h_q[m][:, :n], non_blocking=True)
                        self.d_kv[m][:, :n].copy_(self.h_kv[m][:, :n], non_blocking=True)
                        st["h2d_bytes"] += 2.0 * (self.h_q[m][:, :n].numel() + self.h_kv[m][:, :n].numel())
            e[1].record(self.stream)
            for layer in range(self.nlayers):
                if self.io:
                    sel = [(m, len(ids), min(layer, self.shapes[m][0] - 1)) for m, ids in groups]
                    q = [self.d_q[m][li, :n] for m, n, li in sel]
                    o = [self.d_o[m][li, :n] for m, n, li in sel]
                    kv = [self.d_kv[m][li, :n] for m, n, li in sel]
                b.decode(q, o, layer, stream=self.stream, k=kv, v=kv)
            e[2].record(self.stream)
            if self.io:  # every layer's attention output back to the host
                with torch.cuda.stream(self.stream):
                    for (m, ids) in groups:
                        n = len(ids)
                        self.h_o[m][:, :n].copy_(self.d_o[m][:, :n], non_blocking=True)
                        st["d2h_bytes"] += 2.0 * self.h_o[m][:, :n].numel()
            self._marks.append(("dec", e))
            for layer in range(self.nlayers):
                st["decode_bytes"] += b.decode_bytes(layer)[0]
        if pre_ok:
            # every prefill chunk of the iteration in ONE ragged batch: per layer one append and
            # one causal-prefill launch, whatever the chunk lengths
            groups, lens = [], []
            for m in range(self.M):
                rs = [(r, c) for r, c in pre_ok if r.model == m]
                if rs:
                    groups.append((m, [r.rid for r, _ in rs]))
                    lens += [c for _, c in rs]
            tot = {m: sum(c for r, c in pre_ok if r.model == m) for m, _ in groups}
            b = self._batch("_pre_batch", groups)
            q = [self.q_pre[m][: tot[m]] for m, _ in groups]
            o = [self.o_pre[m][: tot[m]] for m, _ in groups]
            kv = [self.kv_pre[m][: tot[m]] for m, _ in groups]
            e = [ev(), ev(), ev()]
            e[0].record(self.stream)
            for layer in range(self.nlayers):
                b.append(kv, kv, layer, lens, self.stream)
            e[1].record(self.stream)
            for layer in range(self.nlayers):
                b.prefill(q, o, layer, lens, stream=self.stream)
            e[2].record(self.stream)
            self._marks.append(("pre", e))
            st["prefill_launches"] += self.nlayers
            for r, c in pre_ok:
                L, H, Hq = self.shapes[r.model]
                st["prefill_flops"] += 4.0 * 128 * Hq * L * (c * r.done + c * (c + 1) / 2)
                st["append_bytes"] += c * L * 2 * H * 128 * 2 * 2
        span[1].record(self.stream)
        self._marks.append(("span", span))
        # bookkeeping: finished requests are freed (one batched call)
        t1 = time.perf_counter()
        done = []
        for r in dec_ok:
            r.generated += 1
            if r.generated >= r.out_len:
                done.append(r)
        for r, c in pre_ok:
            r.done += c
            if r.done >= r.in_len:
                r.phase, r.generated = "decode", 1  # the prefill iteration emits token 1
                if r.rid in self.preempted_ids:
                    st["reprefilled"] += 1
                    self.preempted_ids.discard(r.rid)
                if r.generated >= r.out_len:
                    done.append(r)
        self._free_many(done)
        for r in done:
            del self.running[r.rid]
        st["finished"] += len(done)
        st["alloc_s"] += time.perf_counter() - t1
        st["iterations"] += 1
        st["occupancy_sum"] += cache.allocated_blocks() / max(1, pool)
        return st

    def _resolve(self) -> None:
        """GPU times of the recorded phases (one synchronize, after the timed region)."""
        if not self._marks:
            return
        torch.cuda.synchronize()
        st = self.stats
        for kind, e in self._marks:
            if kind == "span":
                st["data_path_ms"] += e[0].elapsed_time(e[1])
            elif kind == "dec":
                st["decode_ms"] += e[1].elapsed_time(e[2])
            else:
                st["append_ms"] += e[0].elapsed_time(e[1])
                st["prefill_ms"] += e[1].elapsed_time(e[2])
        self._marks = []

    def summary(self) -> dict:
        self._resolve()
        st = self.stats
        it = max(1, st["iterations"])
        return {
            "iterations": st["iterations"], "admitted": st["admitted"], "finished": st["finished"],
            "preemptions": st["preemptions"], "reprefilled": st["reprefilled"], "cache_full": st["cache_full"],
            "grow_ops": st["grow_ops"], "free_ops": st["free_ops"],
            "alloc_ops_per_s": round((st["grow_ops"] + st["free_ops"]) / max(st["alloc_s"], 1e-9), 1),
            "mean_occupancy": round(st["occupancy_sum"] / it, 4),
            "decode_GBps": round(st["decode_bytes"] / max(st["decode_ms"], 1e-9) / 1e6, 1),
            # prefill-chunk appends (a decode step's append is fused into its decode launch)
            "append_GBps": round(st["append_bytes"] / max(st["append_ms"], 1e-9) / 1e6, 1),
            "prefill_TFLOPs": round(st["prefill_flops"] / max(st["prefill_ms"], 1e-9) / 1e9, 1),
            "decode_ms": round(st["decode_ms"], 2), "prefill_ms": round(st["prefill_ms"], 2),
            "append_ms": round(st["append_ms"], 2), "data_path_ms": round(st["data_path_ms"], 2),
            "prefill_launches": st["prefill_launches"],
            "h2d_bytes": st["h2d_bytes"], "d2h_bytes": st["d2h_bytes"],
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

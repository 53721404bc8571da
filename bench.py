#!/usr/bin/env python
"""bench.py — unified-KV paged decode attention on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], "config 2"): 4 services sharing ONE merged-block
pool — Llama-3-8B (32L, 8 KV / 32 Q heads), Mistral-7B (same), Llama-2-13B (40L, 40H),
OPT-6.7B (32L, 32H), d=128, fp16 — 256 decode requests each (1024 total) at context
2048.  As written that KV needs ~1.0 TB, so the pool is LAYER-SLICED:
block tables come from the full-shape allocator (bit-exact, 76,460+ merged blocks),
each native block physically stores 4 layers and logical layer l reads physical
layer l % 4.  Every per-layer launch reads exactly the config's bytes (23.6 GB per
layer index, far larger than the 126 MB L2, so no L2 flush is needed).

One step = one decode iteration of all 1024 requests over all 40 layer indices:
  GPU allocator grow (+1 token each) -> per layer ONE launch covering all services that
  appends the new token's K/V and runs paged decode attention.
value = decode K/V bytes of the step / device time of the step (GB/s), max over ranks.
e2e   = the same through the C-ABI with host (pinned) buffers: H2D of q/k/v and D2H of
        the attention output inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SERVICES = [  # (name, layers, kv_heads, q_heads)
    ("llama-3-8b", 32, 8, 32),
    ("mistral-7b", 32, 8, 32),
    ("llama-2-13b", 40, 40, 40),
    ("opt-6.7b", 32, 32, 32),
]


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler over the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


SERVICES_C1 = [("llama-2-7b", 32, 32, 32), ("llama-2-13b", 40, 40, 40)]
# (name, layers, kv heads, q heads, head dim): config 2 with four different head-dim / GQA mixes
SERVICES_MIXED_D = [("llama-3.2-1b", 16, 8, 32, 64), ("llama-3-8b", 32, 8, 32, 128), ("llama-2-13b", 40, 40, 40, 128),
                    ("gemma-7b", 28, 16, 16, 256)]


class Workload:
    """services [(name, layers, kv_heads, q_heads)], per-service request contexts,
    physical layers per native block (0 = faithful all-layer layout), pool blocks."""

    def __init__(self, name, services, ctxs, phys_layers, pool_blocks, desc):
        self.name, self.services, self.ctxs = name, services, ctxs
        self.phys_layers, self.pool_blocks, self.desc = phys_layers, pool_blocks, desc
        self.nlayers = max(s[1] for s in services)


def hd(s):
    """head dim of a service tuple (name, layers, kv heads, q heads[, head dim = 128])"""
    return s[4] if len(s) > 4 else 128


def model_specs(P, services):
    return [P.ModelSpec(s[0], s[1], s[2], hd(s), 2, s[3]) for s in services]


def _subs(P, services):
    specs = model_specs(P, services)
    merged = P.plan_merged_shape(specs)
    return [int(merged // P.native_block_bytes(s)) for s in specs], merged


def _blocks(P, services, ctxs, grow):
    subs, _ = _subs(P, services)
    return sum(-(-sum((c + grow + 15) // 16 for c in cl) // sub) for sub, cl in zip(subs, ctxs)) + 64


# tokens every decode request may still grow by during one run: warm-up + timed steps of the
# device and e2e legs, the capture steps and the allocator measurement (3 x 16 + 16 steps)
def grow_reserve(args):
    return args.warmup * 2 + args.steps * 2 + 8 + 80


def make_workload(P, args):
    grow = grow_reserve(args)
    if args.workload == "config1":
        ctxs = [[args.ctx or 512] * (args.requests or 32) for _ in SERVICES_C1]
        return Workload("config1", SERVICES_C1, ctxs, 0, _blocks(P, SERVICES_C1, ctxs, grow),
                        f"config1: llama-2-7b + llama-2-13b shapes, {len(ctxs[0])} decode requests each, ctx "
                        f"{ctxs[0][0]}+, fp16, faithful all-layer merged-block pool")
    if args.workload == "config4":
        # long context, skewed lengths: seeded lognormal (median 4K tokens) capped at 32K,
        # services round-robin until the requests fill ~95 % of a ~150 GB pool
        subs, merged = _subs(P, SERVICES)
        pool = int(150e9 // merged)
        rng = np.random.default_rng(32768)
        ctxs = [[] for _ in SERVICES]
        used = [0] * len(SERVICES)  # native slots per service
        m = 0
        while True:
            c = int(min(32768, max(256, rng.lognormal(np.log(4096), 1.0))))
            trial = list(used)
            trial[m] += (c + grow + 15) // 16
            if sum(-(-u // sb) for u, sb in zip(trial, subs)) > 0.95 * pool:
                break
            used = trial
            ctxs[m].append(c)
            m = (m + 1) % len(SERVICES)
        return Workload("config4", SERVICES, ctxs, 0, pool,
                        f"config4: 4 services (config-2 shapes), {sum(map(len, ctxs))} requests, ctx lognormal "
                        f"(median 4096, max 32768; max drawn {max(max(c) for c in ctxs)}), faithful all-layer pool of "
                        f"{pool} merged blocks (~150 GB) filled to ~95 %, split-KV decode")
    nreq = args.requests or 256
    ctx = args.ctx or 2048
    if args.workload == "config2d":  # config 2 with services of different head dims
        ctxs = [[ctx] * nreq for _ in SERVICES_MIXED_D]
        return Workload("config2d", SERVICES_MIXED_D, ctxs, args.phys_layers,
                        _blocks(P, SERVICES_MIXED_D, ctxs, grow),
                        f"config2-mixed-head-dims: 4 services (llama-3.2-1b d64 GQA4, llama-3-8b d128 GQA4, "
                        f"llama-2-13b d128 MHA, gemma-7b d256 MHA) x {nreq} decode requests, ctx {ctx}+, one "
                        f"unified pool; {args.phys_layers} physical layers per native block, 40 layer-index "
                        f"launches per step")
    ctxs = [[ctx] * nreq for _ in SERVICES]
    blocks = _blocks(P, SERVICES, ctxs, grow)
    if args.phys_layers == 0:  # SURVEY §8d run (B): every layer stored, requests cut to fit one B200
        return Workload("config2", SERVICES, ctxs, 0, blocks,
                        f"config2-capacity-faithful: 4 services (llama-3-8b, mistral-7b, llama-2-13b, opt-6.7b) x "
                        f"{nreq} decode requests, ctx {ctx}+, one unified all-layer pool of {blocks} merged blocks, "
                        f"40 layer-index launches per step")
    return Workload("config2", SERVICES, ctxs, args.phys_layers, blocks,
                    f"config2-layer-sliced: 4 services (llama-3-8b, mistral-7b, llama-2-13b, opt-6.7b) x {nreq} "
                    f"decode requests, ctx {ctx}+, one unified pool; {args.phys_layers} physical layers per native "
                    f"block (logical l -> l % {args.phys_layers}), 40 layer-index launches per step")


def add_tp_shard(P, wl, args, tp):
    """N >= 2: one 70B-shape service (reference llama2-70b: 80 layers, 64 KV heads, Q7) is
    head-sharded over tp = min(N, 4) ranks.  Each rank's pool holds its 64/tp KV heads as one
    more service — native block = 16*80*2*(64/tp)*128*2 B, exactly native_block_bytes(70B, tp)
    (kv_cache.hpp:17-22) — and replays the same op stream, so block tables are identical on the
    tp ranks with no communication.  16*tp requests per group keep the per-rank bytes constant
    as N grows (weak scaling)."""
    h = 64 // tp
    nreq = 16 * tp
    ctx = args.ctx or 2048
    wl.services = list(wl.services) + [(f"llama2-70b/tp{tp}", 80, h, h)]
    wl.ctxs = list(wl.ctxs) + [[ctx] * nreq]
    grow = grow_reserve(args)
    wl.pool_blocks = _blocks(P, wl.services, wl.ctxs, grow)
    wl.nlayers = 80
    wl.desc += (f"; plus a llama2-70b-shape service head-sharded over tp={tp} ranks ({nreq} requests per tp group, "
                f"{h} KV/Q heads per rank, W_o row slice + NCCL AllReduce of the [B, 8192] output per layer; "
                f"80 layer-index launches per step)")
    return wl


def setup(P, torch, args, device, tp_shard=0):
    wl = make_workload(P, args)
    if tp_shard:
        add_tp_shard(P, wl, args, tp_shard)
    models = model_specs(P, wl.services)
    ctx_max = max(max(c) for c in wl.ctxs if c) + grow_reserve(args)
    nreq_total = sum(len(c) for c in wl.ctxs)
    cache = P.UnifiedKvCache(models, 16, 1, wl.pool_blocks, device=device, dtype=P.FP16,
                             phys_layers=wl.phys_layers, max_requests=nreq_total + 16,
                             max_blocks_per_request=(ctx_max + 15) // 16 + 1, allocate_storage=True)
    ns = len(wl.services)
    groups = [(m, []) for m in range(ns)]
    ops = []
    rid = 1
    for r in range(max(len(c) for c in wl.ctxs)):  # interleaved arrival order across services
        for m in range(ns):
            if r < len(wl.ctxs[m]):
                ops.append((0, rid, m, wl.ctxs[m][r]))
                groups[m][1].append(rid)
                rid += 1
    granted = cache.replay(ops)
    assert granted.all(), "pool too small for the workload"
    # a dedicated (non-blocking) stream: the legacy default stream would serialise
    # the e2e leg's copy stream against compute
    stream = torch.cuda.Stream(device=device)
    torch.cuda.set_stream(stream)
    cache.set_stream(stream)
    cache.synth_fill(20250421, 1.0, stream)
    batch = cache.batch(groups)
    g = torch.Generator(device=device).manual_seed(1)
    sizes = [len(ids) for _, ids in groups]
    q = [torch.randn((n, s[3], hd(s)), generator=g, device=device).half() for n, s in zip(sizes, wl.services)]
    out = [torch.empty_like(x) for x in q]
    k = [torch.randn((n, 1, s[2], hd(s)), generator=g, device=device).half() * 0.5 for n, s in zip(sizes, wl.services)]
    v = [torch.randn((n, 1, s[2], hd(s)), generator=g, device=device).half() * 0.5 for n, s in zip(sizes, wl.services)]
    torch.cuda.synchronize(device)
    return wl, cache, batch, q, out, k, v, stream


def step_device(batch, q, out, k, v, stream, nlayers, epilogue=None, timed=False):
    """One decode step: allocator grow (+1 token per request), then per layer one fused
    launch that appends the new K/V token and runs paged decode attention (then, with a
    head-sharded service, its output projection + AllReduce)."""
    batch.grow(1)
    for layer in range(nlayers):
        batch.decode(q, out, layer, stream=stream, k=k, v=v)
        if epilogue:
            epilogue(layer, out, timed)


def capture_step_graph(torch, cache, batch, q, out, k, v, stream, nlayers):
    """CUDA graph of one decode step's whole device work: the allocator's device half (decode-
    step grow ops generated on the device from its own request state + the placement kernel,
    skv_batch_grow_launch), the decode plan kernel, then per layer the fused append + decode
    launch.  Each replay follows the host mirror of the same step (batch.grow_mirror(1): the
    exact try_allocate answers and CacheStats, no upload).  Returns None if capture is not
    possible."""
    try:
        assert batch.grow_mirror(1), "decode step not fully granted"
        batch.grow_launch(1, stream=stream)  # eager once: sizes the batch's grow buffers
        for layer in range(nlayers):
            batch.decode(q, out, layer, stream=stream, k=k, v=v)
        torch.cuda.synchronize()
        assert batch.grow_mirror(1), "decode step not fully granted"
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            batch.grow_launch(1, stream=stream)
            for layer in range(nlayers):
                batch.decode(q, out, layer, stream=stream, k=k, v=v)
        g.replay()  # the captured step
        torch.cuda.synchronize()
        return g
    except Exception as e:  # noqa: BLE001 - report and fall back to eager launches
        print(f"# graph capture unavailable, eager launches: {e}", file=sys.stderr)
        torch.cuda.synchronize()
        return None


def step_bytes(batch, nlayers):
    kv = tot = 0.0
    for layer in range(nlayers):
        a, b = batch.decode_bytes(layer)
        kv += a
        tot += b
    return kv, tot


def profiled_traffic(wl, args):
    """dram__bytes_read.sum + dram__bytes_write.sum per decode launch from the committed ncu
    capture of this same workload (profiles/r01_decode_traffic_config2.csv: single-pass
    metrics, so ncu did not save/restore the 122 GB pool), or None."""
    path = os.path.join(ROOT, "profiles", "r01_decode_traffic_config2.csv")
    if wl.name != "config2" or (args.requests or 256) != 256 or (args.ctx or 2048) != 2048 or not os.path.exists(path):
        return None, None
    import csv
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    tot = {}
    for r in rows[hi + 1:]:
        if len(r) > 5 and r[h.index("Metric Name")].startswith("dram__bytes_"):
            tot[r[0]] = tot.get(r[0], 0.0) + float(r[h.index("Metric Value")].replace(",", ""))
    return (sum(tot.values()) / len(tot) if tot else None), os.path.relpath(path, ROOT)


def run_gpu(args):
    import torch

    import paper_2504_15720_b200 as P

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SKV_BENCH_SHARE_GPU=1 + SKV_BENCH_BACKEND=gloo: every rank on GPU 0 (functional test
    # of the N-rank path on a 1-GPU box; the numbers are then meaningless)
    if os.environ.get("SKV_BENCH_SHARE_GPU") == "1":
        local = 0
    backend = os.environ.get("SKV_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    # N >= 2: a 70B-shape service head-sharded over tp = min(N, 4) ranks joins every rank's
    # pool; its per-layer output reduction is the data path's only collective
    tp = min(world, 4) if world > 1 and not args.no_tp_group else 0
    if tp and world % tp:
        raise SystemExit(f"--gpus {world}: not a multiple of the tp group size {tp}")
    pg = None
    if tp:
        for g0 in range(0, world, tp):  # every rank creates every subgroup, same order
            grp = dist.new_group(list(range(g0, g0 + tp)))
            if g0 <= rank < g0 + tp:
                pg = grp
    wl, cache, batch, q, out, k, v, stream = setup(P, torch, args, local, tp_shard=tp)
    NLAYERS = wl.nlayers
    red_dev = "cuda" if backend == "nccl" else "cpu"
    shard_g = len(wl.services) - 1 if tp else None
    ar_events = []
    if tp:
        L70 = wl.services[shard_g][1]
        B70 = len(wl.ctxs[shard_g])
        gen = torch.Generator(device=local).manual_seed(70)
        w_o = (torch.randn((q[shard_g].shape[1] * 128, 8192), generator=gen, device=local) / 90).half()
        y70 = torch.empty((B70, 8192), device=local, dtype=torch.float16)

    def tp_epilogue(layer, outs, timed=False, y=None):
        """70B shard: row-parallel W_o slice (cuBLAS) and NCCL AllReduce over the tp group."""
        if not tp or layer >= L70:
            return
        y = y70 if y is None else y
        torch.matmul(outs[shard_g].view(B70, -1), w_o, out=y)
        if timed:
            e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            e[0].record(stream)
        dist.all_reduce(y, op=dist.ReduceOp.SUM, group=pg)
        if timed:
            e[1].record(stream)
            ar_events.append(e)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # ---- device-resident timed region (value) ------------------------------------------
    for _ in range(args.warmup):
        step_device(batch, q, out, k, v, stream, NLAYERS, tp_epilogue)
    barrier()
    # the collective is not captured: with a tp group the step runs eagerly
    graph = None if (args.no_graph or tp) else capture_step_graph(torch, cache, batch, q, out, k, v, stream, NLAYERS)
    kv_total = all_total = 0.0
    launches0 = cache.kernel_launches()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        t0.record(stream)
        for st in range(args.steps):  # no host sync inside the timed region
            if graph is not None:
                if batch.grow_mirror(1):  # host mirror; the device half is in the graph
                    graph.replay()
                else:  # CacheFull somewhere: the per-request host path, eager launches
                    step_device(batch, q, out, k, v, stream, NLAYERS, tp_epilogue, timed=True)
            else:
                step_device(batch, q, out, k, v, stream, NLAYERS, tp_epilogue, timed=True)
            kvb, totb = step_bytes(batch, NLAYERS)  # host mirror: exact context of this step
            kv_total += kvb
            all_total += totb
        t1.record(stream)
        barrier()
    launches_timed = cache.kernel_launches() - launches0
    graph_launches = 0
    if graph is not None:  # the graph's kernels bypass the pool's launch counter
        graph_launches = args.steps * (NLAYERS + 2)  # device grow (op generation + placement), plan, decodes
    # per-launch decode timing for the roofline: a CUDA graph of the step's NLAYERS fused
    # append+decode launches (same contexts, no grow; re-appending the same token is
    # idempotent) replayed back to back on the launching stream, bracketed by events
    dgraph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(dgraph, stream=stream):
        for layer in range(NLAYERS):
            batch.decode(q, out, layer, stream=stream, k=k, v=v)
    dgraph.replay()
    torch.cuda.synchronize()
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nrep = 3
    d0.record(stream)
    for _ in range(nrep):
        dgraph.replay()
    d1.record(stream)
    torch.cuda.synchronize()
    dec_ms = d0.elapsed_time(d1)
    dec_bytes = step_bytes(batch, NLAYERS)[1] * nrep
    n_launch = nrep * NLAYERS
    launches = launches_timed + graph_launches
    elapsed_ms = max_over_ranks(t0.elapsed_time(t1))
    kv_all = sum_over_ranks(kv_total)
    value = kv_all / (elapsed_ms / 1e3) / 1e9
    # a head-sharded request is served by its tp ranks together: count it once per group
    n_tok = sum(len(c) for c in wl.ctxs) - (len(wl.ctxs[shard_g]) * (tp - 1) / tp if tp else 0)
    tokens_s = sum_over_ranks(float(n_tok * args.steps)) / (elapsed_ms / 1e3)
    ar_ms = sum(a.elapsed_time(b) for a, b in ar_events)
    hbm, peak_kind = peaks()
    achieved = dec_bytes / (dec_ms / 1e3) / 1e9  # algorithmic bytes / decode launch time
    traffic, traffic_src = profiled_traffic(wl, args)
    layer0_bytes = batch.decode_bytes(0)[1]

    # ---- allocator: decode-step growth of the whole batch ----------------------------------
    # (a) the step path: host mirror (exact try_allocate answers + CacheStats, no upload) and
    #     the device half (op generation + placement kernel) as the graph runs it
    torch.cuda.synchronize()
    na = 16
    n_ops = na * sum(len(c) for c in wl.ctxs)
    host_s = 0.0
    gg = None
    try:  # the device half of `na` consecutive steps as one graph (as nodes of the step graph run)
        assert batch.grow_mirror(1)
        batch.grow_launch(1, stream=stream)
        torch.cuda.synchronize()
        gg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gg, stream=stream):
            for _ in range(na):
                batch.grow_launch(1, stream=stream)
    except Exception as e:  # noqa: BLE001
        print(f"# allocator graph unavailable: {e}", file=sys.stderr)
    dev_ms = 0.0
    for rep in range(3):
        for i in range(na):  # host halves of the na steps (exact answers + CacheStats)
            h0 = time.perf_counter()
            ok = batch.grow_mirror(1)
            host_s += time.perf_counter() - h0
            assert ok
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):  # keep the GPU busy while the host submits
            torch.cuda._sleep(200000)
        e0.record(stream)
        if gg is not None:
            gg.replay()
        else:
            for i in range(na):
                batch.grow_launch(1, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        dev_ms += e0.elapsed_time(e1)
    n_ops = 3 * na * sum(len(c) for c in wl.ctxs)
    mirror_ns = host_s / n_ops * 1e9
    device_ns = dev_ms * 1e6 / n_ops
    n_ops = na * sum(len(c) for c in wl.ctxs)
    # (b) the per-request host path (any CacheFull case): host mirror + op upload + placement
    a0 = time.perf_counter()
    aev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(na)]
    for i in range(na):
        batch.grow(1)  # host mirror: the grant / CacheFull answer, no device round trip
        with torch.cuda.stream(stream):
            torch.cuda._sleep(200000)
        aev[i][0].record(stream)
        cache.flush(stream)  # GPU placement: op upload + grow_kernel
        aev[i][1].record(stream)
    torch.cuda.synchronize()
    alloc_ns = (time.perf_counter() - a0) / n_ops * 1e9 - 200000 / 1.9e9 * na / n_ops * 1e9  # minus the spin
    alloc_gpu_ns = sum(e0.elapsed_time(e1) for e0, e1 in aev) * 1e6 / n_ops

    # ---- e2e through the C-ABI with host buffers -----------------------------------------
    # Every step copies its inputs (q, k, v of every layer: [NLAYERS, B, H, d] per group)
    # from pinned host memory and reads every layer's attention output back, in 4 chunks
    # of layers: the H2D of chunk c+1 (h2d stream) overlaps the attention of chunk c, whose
    # outputs go back (d2h stream) while chunk c+1 runs; within a chunk the launches stay
    # back to back (no event between them, so programmatic dependent launch still
    # overlaps them).  Device buffers are double-buffered by step parity.
    glayers = [wl.services[m][1] for m, _ in batch.groups]  # each service copies only its own layers

    def pinned_like(x, nl):
        return torch.empty((nl,) + tuple(x.shape), dtype=x.dtype, pin_memory=True)

    hq = [pinned_like(x, nl) for x, nl in zip(q, glayers)]
    hk = [pinned_like(x, nl) for x, nl in zip(k, glayers)]
    hv = [pinned_like(x, nl) for x, nl in zip(v, glayers)]
    ho = [pinned_like(x, nl) for x, nl in zip(out, glayers)]
    if tp:  # the reduced 70B output of every layer comes back too
        ho.append(torch.empty((L70, B70, 8192), dtype=torch.float16, pin_memory=True))
    for hs, ds in ((hq, q), (hk, k), (hv, v)):
        for a, b in zip(hs, ds):
            a.copy_(b.unsqueeze(0).expand_as(a).cpu())
    h2d = sum(x.numel() * x.element_size() for x in hq + hk + hv)
    d2h = sum(x.numel() * x.element_size() for x in ho)
    glayers_o = glayers + ([L70] if tp else [])
    h2d_stream = torch.cuda.Stream(device=local)
    d2h_stream = torch.cuda.Stream(device=local)
    dq = [[torch.empty(x.shape, dtype=x.dtype, device=local) for x in hq] for _ in range(2)]
    dk = [[torch.empty(x.shape, dtype=x.dtype, device=local) for x in hk] for _ in range(2)]
    dv = [[torch.empty(x.shape, dtype=x.dtype, device=local) for x in hv] for _ in range(2)]
    do = [[torch.empty(x.shape, dtype=x.dtype, device=local) for x in ho] for _ in range(2)]
    CH = -(-NLAYERS // 4)  # layers per copy chunk
    chunks = [range(c, min(NLAYERS, c + CH)) for c in range(0, NLAYERS, CH)]
    in_ev = [torch.cuda.Event() for _ in chunks]   # chunk c's inputs are on the device
    out_ev = [torch.cuda.Event() for _ in chunks]  # chunk c's attention is done
    comp_ev = [torch.cuda.Event() for _ in range(2)]       # step done with buffer set j
    d2h_ev = [torch.cuda.Event() for _ in range(2)]        # buffer set j's outputs drained
    for e in comp_ev + d2h_ev:
        e.record(stream)
    e2e_step = [0]

    def step_e2e():
        j = e2e_step[0] & 1
        e2e_step[0] += 1
        with torch.cuda.stream(h2d_stream):
            h2d_stream.wait_event(comp_ev[j])  # step i-2 is done with buffer set j
            for ci, ls in enumerate(chunks):
                for a, b, nl in zip(dq[j] + dk[j] + dv[j], hq + hk + hv, glayers * 3):
                    if ls.start < nl:
                        a[ls.start:min(ls.stop, nl)].copy_(b[ls.start:min(ls.stop, nl)], non_blocking=True)
                in_ev[ci].record(h2d_stream)
        batch.grow(1)
        stream.wait_event(d2h_ev[j])  # output set j drained to host
        for ci, ls in enumerate(chunks):
            stream.wait_event(in_ev[ci])
            for layer in ls:
                sel = [min(layer, nl - 1) for nl in glayers]  # groups past their last layer are skipped
                outs = [x[s] for x, s in zip(do[j], sel)]
                batch.decode([x[s] for x, s in zip(dq[j], sel)], outs, layer, stream=stream,
                             k=[x[s] for x, s in zip(dk[j], sel)], v=[x[s] for x, s in zip(dv[j], sel)])
                if tp and layer < L70:
                    tp_epilogue(layer, outs, y=do[j][-1][layer])
            out_ev[ci].record(stream)
            with torch.cuda.stream(d2h_stream):
                d2h_stream.wait_event(out_ev[ci])
                for a, b, nl in zip(ho, do[j], glayers_o):
                    if ls.start < nl:
                        a[ls.start:min(ls.stop, nl)].copy_(b[ls.start:min(ls.stop, nl)], non_blocking=True)
        comp_ev[j].record(stream)
        d2h_ev[j].record(d2h_stream)

    for _ in range(args.warmup):
        step_e2e()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kv_e2e = 0.0
    e0.record(stream)
    for _ in range(args.steps):
        step_e2e()
        kv_e2e += step_bytes(batch, NLAYERS)[0]
    stream.wait_stream(d2h_stream)  # the last step's outputs are on the host
    e1.record(stream)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    e2e_value = sum_over_ranks(kv_e2e) / (e2e_ms / 1e3) / 1e9

    result = {
        "metric": "unified-KV paged decode attention HBM GB/s (mixed services)",
        "value": round(value, 1),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(elapsed_ms / args.steps, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp16",
        "data": "synthetic (SplitMix64 K/V pool, randn q/k/v); no checkpoints",
        "tokens_per_s": round(tokens_s, 1),
        "config": {
            "workload": wl.desc,
            "requests": sum(len(c) for c in wl.ctxs) * world,
            "ctx_mean": round(float(np.mean([c for cl in wl.ctxs for c in cl])), 1),
            "pool_blocks": cache.pool_size(),
            "merged_block_bytes": cache.merged_block_bytes(),
            "pool_gb": round(cache.storage()[1] / 1e9, 2),
            "l2": "inputs larger than L2 (>= 0.6 GB K/V per layer launch vs 126 MB L2); no flush",
            "parallelism": (f"placement-sharded replicas x{world} (tp=1 groups, no collective)" if not tp else
                            f"config-2 replica per rank (tp=1, no collective) + llama2-70b shape head-sharded in "
                            f"{world // tp} tp={tp} group(s) (NCCL AllReduce of its output per layer)"),
            "cuda_graph": graph is not None,
        },
        "e2e": {"value": round(e2e_value, 1), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e2e_ms / args.steps, 3)},
        "roofline": {"bound": "hbm", "kernel": "skv decode_kernel (KV append + split-KV combine fused)",
                     "achieved": round(achieved, 1), "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": traffic, "traffic_source": traffic_src,
                     "traffic_note": "4-service layer launch (layers 0-31); algorithmic bytes of that launch "
                                     f"~{layer0_bytes:.4g}",
                     "avg_launch_ms": round(dec_ms / n_launch, 4),
                     "timing": f"CUDA events around {nrep} replays of a graph of the step's {NLAYERS} decode "
                               "launches (inter-kernel gaps included)",
                     "bytes_per_launch": round(dec_bytes / n_launch, 1)},
        "allocator": {"ns_per_grow_op": round(mirror_ns + device_ns, 2), "host_mirror_ns_per_op": round(mirror_ns, 2),
                      "device_ns_per_op": round(device_ns, 2),
                      "host_path_ns_per_grow_op": round(alloc_ns, 2), "host_path_gpu_ns_per_grow_op": round(alloc_gpu_ns, 2),
                      "note": "ns_per_grow_op = host mirror (skv_batch_grow_mirror, wall) + device half "
                              "(skv_batch_grow_launch: op generation + placement in one kernel; CUDA events around a "
                              "graph of 16 consecutive steps' launches, as they run as nodes of the step graph) per "
                              "decode-step grow op; host_path_*: batch.grow(1) + flush (op upload + grow_kernel) wall "
                              "incl. sync, the fallback when a step hits CacheFull"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if tp:
        result["allreduce"] = {"group_size": tp, "groups": world // tp, "backend": backend,
                               "bytes_per_layer": int(y70.numel() * 2), "layers_per_step": L70,
                               "ms_per_step_rank0": round(ar_ms / args.steps, 4),
                               "per_layer_ms_rank0": round(ar_ms / max(1, len(ar_events)), 4),
                               "note": "CUDA events around dist.all_reduce on the compute stream (rank 0), "
                                       "timed steps only"}
    cache.synchronize()  # surfaces any device-side invariant flag raised during the runs
    if rank == 0 and not args.no_parity:
        result["parity"] = headline_parity(torch, cache, batch, q, k, v, stream, NLAYERS)
    if rank == 0 and not args.no_prefill:
        # chunked prefill (tcgen05) measured in the same run, so the driver sees the tensor-pipe path
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                tpk, tpk_kind = float(json.load(f)["bf16_tflops"]), "measured (burst, cuBLAS bf16)"
        except Exception:  # noqa: BLE001
            tpk, tpk_kind = 2250.0, "fallback (nominal dense bf16)"
        pf = {"kernel": PREFILL_KERNEL, "peak": tpk, "peak_kind": tpk_kind, "unit": "TFLOP/s", "bound": "tensor",
              "ncu": PREFILL_NCU}
        for key, (R_, ctx_, C_) in (("long_chunk", (4, 16384, 2048)), ("config3_chunk", (8, 2048, 512))):
            s_ = prefill_sample(P, torch, local, R_, ctx_, C_)
            s_["frac"] = round(s_["tflops"] / tpk, 4)
            pf[key] = s_
        result["prefill"] = pf
    if rank == 0 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(cache, batch, q, args)
    if rank == 0 and world == 1 and not args.no_faithful and args.workload == "config2" and args.phys_layers > 0:
        # SURVEY §8d run (B) in the same driver run: the layer-sliced pool is released, then the
        # capacity-faithful config 2 (every layer stored, 38 requests per service, ~152 GB) is timed
        try:
            batch.close()
            cache.close()
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
            result["capacity_faithful"] = faithful_sample()
            if not args.no_config4:  # BASELINE configs[3]: long contexts (lognormal, <= 32K), ~150 GB faithful pool
                result["config4"] = faithful_sample(["--workload", "config4"])
            # BASELINE configs[0]: 7B + 13B shapes, 64 requests at ctx 512 (the small-launch case)
            result["config1"] = faithful_sample(["--workload", "config1"])
            # BASELINE configs[2]: 8 services, bursty trace, alloc/append/free churn at 70 % occupancy
            result["config3"] = faithful_sample(["--workload", "config3"])
        except Exception as e:  # noqa: BLE001  (the headline line is printed regardless)
            result["other_configs_error"] = f"{type(e).__name__}: {e}"[:300]
    if rank == 0:
        print(json.dumps(result), flush=True)
    if dist:
        dist.destroy_process_group()


def faithful_sample(workload=("--workload", "config2", "--phys-layers", "0", "--requests", "38"), steps=5, warmup=3,
                    timeout=600):
    """A faithful-pool workload (default: config 2 with every layer stored) in a child process,
    after the parent released its pool; returns the headline numbers of the child's line."""
    import subprocess

    cmd = [sys.executable, os.path.abspath(__file__), *workload, "--steps", str(steps), "--warmup", str(warmup),
           "--no-prefill", "--no-cpu-baseline", "--no-faithful"]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=dict(os.environ, WORLD_SIZE="1"))
        line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
        d = json.loads(line)
    except Exception as e:  # noqa: BLE001
        return {"error": f"{type(e).__name__}: {e}"[:300]}
    try:  # a sample never breaks the main line
        rf = d.get("roofline", {}) or {}
        cfg = d.get("config", {}) or {}
        out = {"value": d.get("value"), "unit": d.get("unit"), "ms_per_step": d.get("ms_per_step"), "steps": steps,
               "e2e": (d.get("e2e") or {}).get("value"), "roofline_frac": rf.get("frac"), "achieved": rf.get("achieved"),
               "peak": rf.get("peak"), "pool_gb": cfg.get("pool_gb"), "requests": cfg.get("requests"),
               "parity_max_abs": (d.get("parity") or {}).get("max_abs"), "clocks": d.get("clocks"),
               "workload": cfg.get("workload"), "cmd": " ".join(cmd[1:])}
        if "churn" in d:
            out["churn"] = {k: d["churn"][k] for k in ("iterations", "preemptions", "reprefilled", "cache_full",
                                                        "mean_occupancy", "decode_GBps", "prefill_TFLOPs",
                                                        "alloc_ops_per_s") if k in d["churn"]}
        return out
    except Exception as e:  # noqa: BLE001
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def headline_parity(torch, cache, batch, q, k, v, stream, nlayers, per_end=2, tol=2e-3):
    """Oracle check of the measured code path at the measured size (run after the timed
    regions): the same fused append+decode launch over the WHOLE batch at layers 0, 31 and the
    last layer, then the fp32 CPU oracle (oracle/attn_oracle.c; checker only) on a sample of
    its rows — the first and last `per_end` requests of every service, which covers both
    (request, kv head)s that were run as one piece and the last n_cut ones that were cut into
    pieces merged in-kernel."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_py as O

    layers = sorted({0, min(31, nlayers - 1), nlayers - 1})
    outs = {}
    for layer in layers:
        o = [torch.full_like(x, float("nan")) for x in q]
        batch.decode(q, o, layer, stream=stream, k=k, v=v)
        outs[layer] = o
    info = batch.plan_info()
    torch.cuda.synchronize()
    groups = batch.groups
    picks = [sorted(set(range(min(per_end, len(ids)))) | set(range(max(0, len(ids) - per_end), len(ids))))
             for _, ids in groups]
    hkv = [cache.layout(m).kv_heads for m, _ in groups]
    # (request, kv head) index in batch order: the last n_cut of them were cut
    first_rh, acc = [], 0
    for (m, ids), h in zip(groups, hkv):
        first_rh.append(acc)
        acc += len(ids) * h
    cut_from = info["sum_hkv"] - info["n_cut"]
    blocks = sorted({int(b) for (m, ids), pk in zip(groups, picks) for i in pk
                     for b in cache.block_table_np(ids[i])[:, 0]})
    remap = {b: j for j, b in enumerate(blocks)}
    img = cache.read_blocks(np.array(blocks, dtype=np.int32))
    worst, n_rows, cut_rows = 0.0, 0, 0
    for gi, ((m, ids), pk) in enumerate(zip(groups, picks)):
        lay = cache.layout(m)
        olay = O.layout(lay.merged_stride, lay.native_stride, lay.layer_stride, lay.head_stride, lay.kv_stride,
                        lay.tpb, lay.head_dim, lay.kv_heads, lay.q_heads, lay.phys_layers, lay.dtype)
        tabs = [cache.block_table_np(ids[i]) for i in pk]
        tt = np.zeros((len(pk), max(len(t) for t in tabs), 2), np.int32)
        for j, t in enumerate(tabs):
            tt[j, :len(t), 0] = [remap[int(b)] for b in t[:, 0]]
            tt[j, :len(t), 1] = t[:, 1]
        ctx = np.array([cache.request_tokens(ids[i]) for i in pk], np.int64)
        qh = q[gi][pk].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
        G = lay.q_heads // lay.kv_heads
        for layer in layers:
            if layer >= cache.models[m].num_layers:
                continue
            ref = O.decode_attention(olay, img, layer, tt, ctx, qh, 1.0 / np.sqrt(lay.head_dim))
            got = outs[layer][gi][pk].float().cpu().numpy()
            worst = max(worst, float(np.abs(got - ref).max()) if not np.isnan(got).any() else float("inf"))
            n_rows += got.shape[0] * got.shape[1]
            cut_rows += sum(G for i in pk for h in range(lay.kv_heads)
                            if first_rh[gi] + i * lay.kv_heads + h >= cut_from)
    return {"max_abs": worst, "tol": tol, "ok": bool(worst <= tol), "n_rows": n_rows, "rows_in_cut_pieces": cut_rows,
            "layers": layers, "requests_per_service": [len(pk) for pk in picks],
            "schedule": info, "oracle": "oracle/attn_oracle.c (fp32, OpenMP)",
            "note": "fused append+decode launch over the whole measured batch; first/last requests of each service"}


def _sample_image(cache, batch_groups, per_group):
    """Compact host image holding only the sampled requests' merged blocks."""
    import oracle_py as O  # noqa: F401  (checker only; never on the product path)

    samp = []
    blocks = set()
    for m, ids in batch_groups:
        for rid in ids[:per_group]:
            bt = cache.block_table_np(rid)
            samp.append((m, rid, bt))
            blocks.update(bt[:, 0].tolist())
    blocks = sorted(blocks)
    remap = {b: i for i, b in enumerate(blocks)}
    img = cache.read_blocks(np.array(blocks, dtype=np.int32))
    return samp, remap, img


def cpu_baseline(cache, batch, q, args, budget_s=None):
    """fp32 CPU oracle (oracle/attn_oracle.c, OpenMP over all host cores) on a bounded
    sample of the same workload: the first few requests of every service, layer 0."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_py as O

    budget_s = budget_s or args.cpu_seconds
    groups = batch.groups
    per = args.cpu_requests
    samp, remap, img = _sample_image(cache, groups, per)
    cores = os.cpu_count() or 1
    work = []
    nbytes = 0.0
    for m, ids in groups:
        lay = cache.layout(m)
        olay = O.layout(lay.merged_stride, lay.native_stride, lay.layer_stride, lay.head_stride, lay.kv_stride,
                        lay.tpb, lay.head_dim, lay.kv_heads, lay.q_heads, lay.phys_layers, lay.dtype)
        rows = [s for s in samp if s[0] == m]
        width = max(len(s[2]) for s in rows)
        tabs = np.zeros((len(rows), width, 2), np.int32)
        ctx = np.zeros(len(rows), np.int64)
        for i, (_, rid, bt) in enumerate(rows):
            tabs[i, :len(bt), 0] = [remap[b] for b in bt[:, 0]]
            tabs[i, :len(bt), 1] = bt[:, 1]
            ctx[i] = cache.request_tokens(rid)
        qh = q[m][:len(rows)].view(__import__("torch").int16).cpu().numpy().view(np.uint16)
        work.append((olay, tabs, ctx, qh))
        nbytes += float(ctx.sum()) * lay.kv_heads * lay.head_dim * 2 * 2
    t0 = time.perf_counter()
    reps = 0
    while True:
        for olay, tabs, ctx, qh in work:
            O.decode_attention(olay, img, 0, tabs, ctx, qh, 1.0 / np.sqrt(olay.head_dim), nthreads=cores)
        reps += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": round(nbytes * reps / dt / 1e9, 3), "unit": "GB/s", "cores": cores, "kind": "port",
            "sample": f"fp32 oracle decode, layer 0, first {per} requests of each of the 4 services at ctx "
                      f"~{int(np.mean([c for c in (cache.request_tokens(r) for _, ids in groups for r in ids[:per])]))}, "
                      f"{reps} reps in {dt:.1f} s (attention has no reference implementation; "
                      "oracle/attn_oracle.c)"}


def run_churn(args):
    """Config 3: 8 services (4 shapes x {chat, summarisation}) on one faithful pool, bursty
    Poisson trace (skewness 4, rate step x2 halfway), chunked prefill C=512, 70 % occupancy."""
    import torch

    import paper_2504_15720_b200 as P
    from paper_2504_15720_b200.churn import ChurnEngine, generate_trace, paper_services

    torch.cuda.set_device(0)
    models = [P.ModelSpec(n, L, H, 128, 2, Hq) for n, L, H, Hq in SERVICES]
    merged = P.plan_merged_shape(models)
    pool = int(args.pool_gb * 1e9 // merged)
    cache = P.UnifiedKvCache(models, 16, 1, pool, allocate_storage=True, max_requests=8192,
                             max_blocks_per_request=2048)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    cache.set_stream(stream)
    cache.synth_fill(3, 1.0, stream)
    shapes = [(L, H, Hq) for _, L, H, Hq in SERVICES]
    prof = paper_services(len(SERVICES))
    iters = args.steps * 10 + args.warmup * 10
    dt = 0.1
    trace = generate_trace(prof, rate=args.rate, duration=iters * dt, skewness=4, seed=2025,
                           step_time=iters * dt / 2, step_factor=2.0)
    eng = ChurnEngine(cache, shapes, prof, chunk=512, occupancy=args.occupancy, max_decode=1024, max_prefill=8,
                      stream=stream, io=True)
    # steady state first: the pool is brought to the occupancy target with already-prefilled
    # requests from the head of the trace, then warm-up iterations run untimed
    k = eng.warm_start(trace)
    t = 0.0
    n_warm = args.warmup * 10

    def advance():
        nonlocal t, k
        t += dt
        new = []
        while k < len(trace) and trace[k].t <= t:
            new.append(trace[k])
            k += 1
        eng.add_arrivals(new)
        eng.step()

    for _ in range(n_warm):
        advance()
    torch.cuda.synchronize()
    eng.reset_stats()
    launches0 = cache.kernel_launches()
    with Clocks(0) as clk:
        w0 = time.perf_counter()
        for _ in range(iters - n_warm):
            advance()
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    summ = eng.summary()
    n_it = iters - n_warm
    e2e = {"value": round(eng.stats["decode_bytes"] / wall / 1e9, 1), "unit": "GB/s",
           "h2d_bytes_per_step": int(summ["h2d_bytes"] / n_it), "d2h_bytes_per_step": int(summ["d2h_bytes"] / n_it),
           "iteration_ms_wall": round(wall / n_it * 1e3, 3),
           "gpu_busy_frac": round(summ["data_path_ms"] / (wall * 1e3), 4),
           "prefill_TFLOPs_wall": round(eng.stats["prefill_flops"] / wall / 1e12, 1),
           "note": "wall clock of the whole host-driven loop (admission, batched allocator calls, every launch, "
                   "decode q/k/v of every layer H2D from pinned memory and every layer's output D2H); decode "
                   "bytes / wall time, so prefill and allocator time count against it"}
    res = {
        "metric": "unified-KV paged decode attention HBM GB/s under churn (config 3)",
        "value": summ["decode_GBps"], "unit": "GB/s", "n_gpus": 1, "steps": iters - n_warm, "warmup": n_warm,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp16",
        "data": "synthetic trace (reference generate_trace semantics) + synthetic K/V",
        "config": {"workload": f"config3: 8 services (4 shapes x chat/summarisation, PAPER Table 1 lengths), "
                               f"Poisson rate {args.rate}/s, skewness 4, rate x2 at half time, chunk 512, "
                               f"occupancy target {args.occupancy} (pool filled with {k} prefilled trace requests, then "
                               f"{n_warm} untimed iterations), faithful pool {pool} merged blocks ({args.pool_gb} GB)"},
        "churn": summ, "e2e": e2e, "gpu_launches": int(cache.kernel_launches() - launches0),
        "clocks": clk.summary(),
        "note": "eager, host-driven engine (allocator decisions on the host each iteration, one batched C-ABI "
                "call per grow/free set); value = decode bytes / GPU span of each iteration's decode phase (one "
                "fused append+decode launch per layer); prefill = one ragged append + one ragged causal-prefill "
                "launch per layer; churn.data_path_ms is the GPU span of each whole step",
    }
    print(json.dumps(res), flush=True)


SHAPES_C5 = {  # reference model id -> (layers, kv heads, q heads); 70B keeps the reference's 64 KV heads (Q7)
    "llama2-70b": (80, 64, 64), "llama2-7b": (32, 32, 32), "llama2-13b": (40, 40, 40),
    "opt-6.7b": (32, 32, 32), "llama3-8b": (32, 8, 32),
}


def run_config5(args):
    """Config 5: 16 services (one 70B shape + 15 mixed) placed on N GPUs by the reference
    placement (placement.dedicated_plan with the SURVEY §8e overrides).  Each process (one
    GPU) owns one sharing group's unified pool at the group's TP size; per layer ONE decode
    launch covers every service of the group.  A head-sharded (tp > 1) group also projects
    the 70B service's partial attention output through its W_o row slice and sums it over
    the group with NCCL AllReduce -- the only collective of the data path.  Total work is
    fixed as N grows (strong scaling)."""
    import torch
    import torch.distributed as dist

    import paper_2504_15720_b200 as P
    from paper_2504_15720_b200 import placement as PL

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SKV_BENCH_SHARE_GPU=1: every rank on GPU 0 (functional test of the N-rank path on a
    # 1-GPU box; use SKV_BENCH_BACKEND=gloo then)
    dev = 0 if os.environ.get("SKV_BENCH_SHARE_GPU") == "1" else local
    torch.cuda.set_device(dev)
    backend = os.environ.get("SKV_BENCH_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    services = PL.config5_services()
    plan = PL.dedicated_plan(services, PL.config5_overrides(world))
    assert plan.feasible, f"config5 placement infeasible on {world} GPUs: unplaced {plan.unplaced}"
    tp_groups = {}
    for gi, g in enumerate(plan.groups):  # every rank creates every subgroup, same order
        if world > 1 and g.tp_size > 1:
            tp_groups[gi] = dist.new_group(g.gpu_ids)
    role = PL.rank_role(plan, rank)
    nreq = args.requests or 16
    ctx = args.ctx or 2048
    grow = args.warmup * 2 + args.steps * 2 + 8
    kv_total = 0.0
    elapsed_ms = 0.0
    ar_ms = 0.0
    n_ar = 0
    launches = 0
    if role is not None:
        g = role.group
        tp = g.tp_size
        names = [services[s] for s in role.services]
        models = [P.ModelSpec(f"{n}#{s}", SHAPES_C5[n][0], SHAPES_C5[n][1], 128, 2, SHAPES_C5[n][2])
                  for n, s in zip(names, role.services)]
        merged = P.plan_merged_shape(models, 16, tp)
        subs = [int(merged // P.native_block_bytes(m, 16, tp)) for m in models]
        pool = sum(-(-nreq * ((ctx + grow + 15) // 16) // sb) for sb in subs) + 64
        cache = P.UnifiedKvCache(models, 16, tp, pool, device=dev, dtype=P.FP16, phys_layers=args.phys_layers,
                                 max_requests=nreq * len(models) + 16,
                                 max_blocks_per_request=(ctx + grow + 15) // 16 + 1, allocate_storage=True)
        groups = [(m, []) for m in range(len(models))]
        ops, rid = [], 1
        for r in range(nreq):
            for m in range(len(models)):
                ops.append((0, rid, m, ctx))
                groups[m][1].append(rid)
                rid += 1
        assert cache.replay(ops).all(), "pool too small"
        stream = torch.cuda.Stream(device=dev)
        torch.cuda.set_stream(stream)
        cache.set_stream(stream)
        cache.synth_fill(5 + role.group_index, 1.0, stream)
        batch = cache.batch(groups)
        gen = torch.Generator(device=dev).manual_seed(1)
        shp = [SHAPES_C5[n] for n in names]
        q = [torch.randn((nreq, Hq // tp, 128), generator=gen, device=dev).half() for _, _, Hq in shp]
        out = [torch.empty_like(x) for x in q]
        k = [torch.randn((nreq, 1, H // tp, 128), generator=gen, device=dev).half() * 0.5 for _, H, _ in shp]
        v = [torch.randn((nreq, 1, H // tp, 128), generator=gen, device=dev).half() * 0.5 for _, H, _ in shp]
        big = [i for i, n in enumerate(names) if n == "llama2-70b"]
        hidden = 8192
        w_o = (torch.randn((64 // tp * 128, hidden), generator=gen, device=dev) / 90).half() if big else None
        y = torch.empty((nreq, hidden), device=dev, dtype=torch.float16) if big else None
        pg = tp_groups.get(role.group_index)
        nl = max(L for L, _, _ in shp)
        ev_ar = []

        def step(timed):
            batch.grow(1)
            for layer in range(nl):
                batch.decode(q, out, layer, stream=stream, k=k, v=v)
                if big and layer < shp[big[0]][0]:
                    torch.matmul(out[big[0]].view(nreq, -1), w_o, out=y)  # partial row-parallel output
                    if pg is not None:
                        e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                        e[0].record(stream)
                        dist.all_reduce(y, op=dist.ReduceOp.SUM, group=pg)
                        e[1].record(stream)
                        if timed:
                            ev_ar.append(e)

        for _ in range(args.warmup):
            step(False)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = cache.kernel_launches()
        t0.record(stream)
        for _ in range(args.steps):
            step(True)
            kv_total += step_bytes(batch, nl)[0]
        t1.record(stream)
        torch.cuda.synchronize()
        launches = cache.kernel_launches() - l0
        elapsed_ms = t0.elapsed_time(t1)
        ar_ms = sum(a.elapsed_time(b) for a, b in ev_ar)
        n_ar = len(ev_ar)
    if world > 1:
        dist.barrier()
        t = torch.tensor([elapsed_ms, kv_total, float(launches)], dtype=torch.float64,
                         device=dev if backend == "nccl" else "cpu")
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        elapsed_ms, kv_all, launches = float(mx[0]), float(t[1]), int(t[2])
    else:
        kv_all = kv_total
    if rank == 0:
        hbm, peak_kind = peaks()
        value = kv_all / (elapsed_ms / 1e3) / 1e9
        desc = "; ".join(f"group {gi}: gpus {g.gpu_ids} tp{g.tp_size} services "
                         f"{[services[s] for s in g.services]}" for gi, g in enumerate(plan.groups))
        print(json.dumps({
            "metric": "unified-KV paged decode attention HBM GB/s (mixed services)", "value": round(value, 1),
            "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(elapsed_ms / args.steps, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "fp16", "data": "synthetic",
            "config": {"workload": f"config5: 16 services (llama2-70b shape head-sharded + 15 mixed), reference "
                                   f"dedicated_plan with SURVEY 8e overrides; {nreq} decode requests per service at "
                                   f"ctx {ctx}+; layer-sliced pools ({args.phys_layers} physical layers)",
                       "placement": desc, "backend": backend},
            "frac_of_hbm_x_n": round(value / (hbm * world), 4), "peak": hbm, "peak_kind": peak_kind,
            "allreduce": {"per_layer_ms_rank0": round(ar_ms / max(1, n_ar), 4), "count_rank0": n_ar},
            "gpu_launches": launches,
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()


# head dim 128 runs the ping-pong kernel (skv_prefill.cu prefill_pp_kernel; SKV_PREFILL_PP=0: the
# one-tile-per-CTA prefill_kernel<T, 128>)
PREFILL_KERNEL = ("skv prefill_pp_kernel<T> (cta_group::2 tcgen05.mma, two query tiles per CTA, TMA, TMEM)"
                  if os.environ.get("SKV_PREFILL_PP", "1") != "0" else
                  "skv prefill_kernel<T, 128> (cta_group::2 tcgen05.mma, TMA, TMEM)")
PREFILL_NCU = "profiles/r02_ncu_prefill_pp.txt (tensor pipe active % of cycles)"


def prefill_sample(P, torch, device, R, ctx, C, steps=10, warmup=3, services=None, check=True):
    """Chunked prefill (tcgen05 CTA-pair kernel) on its own pool: the config-2 services, R
    requests each, the last C tokens of a ctx-token context attending causally (layer 0),
    timed with CUDA events on the launching stream (useful causal flops); plus an fp32-oracle
    check of the last 64 query rows of each service's first request."""
    services = services or SERVICES
    models = model_specs(P, services)
    cache = P.UnifiedKvCache(models, 16, 1, len(services) * R * (ctx // 16 + 2) + 64, device=device,
                             phys_layers=2, allocate_storage=True)
    groups, rid = [], 1
    for m in range(len(services)):
        ids = []
        for _ in range(R):
            assert cache.try_allocate(rid, m, ctx)
            ids.append(rid)
            rid += 1
        groups.append((m, ids))
    stream = torch.cuda.Stream(device=device)
    cache.set_stream(stream)
    cache.synth_fill(1, 1.0, stream)
    b = cache.batch(groups)
    gen = torch.Generator(device=device).manual_seed(3)
    with torch.cuda.stream(stream):
        qs = [torch.randn((R, C, s[3], hd(s)), generator=gen, device=device).half() for s in services]
        outs = [torch.empty_like(x) for x in qs]
    flops = sum(4.0 * hd(s) * s[3] * R * (C * (ctx - C) + C * (C + 1) / 2) for s in services)
    for _ in range(warmup):
        b.prefill(qs, outs, 0, C, stream=stream)
    torch.cuda.synchronize(device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(device) as clk:
        e0.record(stream)
        for _ in range(steps):
            b.prefill(qs, outs, 0, C, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize(device)
    ms = e0.elapsed_time(e1) / steps
    res = {"tflops": round(flops / (ms * 1e-3) / 1e12, 1), "ms_per_launch": round(ms, 4),
           "shape": f"{len(services)} services x {R} requests, last {C} of {ctx} tokens (causal)",
           "clocks": clk.summary()}
    if check:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle_py as O
        worst, nq = 0.0, min(64, C)
        for (m, ids), q, o in zip(groups, qs, outs):
            bt = cache.block_table_np(ids[0])
            img = cache.read_blocks(bt[:, 0])
            tab = np.stack([np.arange(len(bt), dtype=np.int32), bt[:, 1]], axis=1)[None]
            lay = cache.layout(m)
            olay = O.layout(lay.merged_stride, lay.native_stride, lay.layer_stride, lay.head_stride, lay.kv_stride,
                            16, lay.head_dim, lay.kv_heads, lay.q_heads, lay.phys_layers, lay.dtype)
            qh = q[0, C - nq:].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
            ref = O.prefill_attention(olay, img, 0, tab, np.array([ctx - nq], np.int64), np.array([nq], np.int64),
                                      qh.reshape(nq, -1, lay.head_dim), 1.0 / np.sqrt(lay.head_dim))
            got = o[0, C - nq:].float().cpu().numpy().reshape(ref.shape)
            worst = max(worst, float(np.abs(got - ref).max()))
        res["parity"] = {"max_abs": worst, "tol": 2e-3, "ok": bool(worst <= 2e-3),
                         "rows": f"last {nq} query tokens of the first request of each service"}
    b.close()
    cache.close()
    return res


def run_prefill(args):
    """Chunked-prefill attention on tcgen05, one line in the bench format:
    the four config-2 services, R requests each, the last C tokens of a CTX-token context
    attending causally (layer 0), default R=4, CTX=16384, C=2048.  value = useful causal
    TFLOP/s, roofline against the measured dense bf16 peak; e2e copies q from pinned host
    memory and the output back every step."""
    import numpy as np
    import torch

    import paper_2504_15720_b200 as P

    torch.cuda.set_device(0)
    R = args.requests or 4
    ctx = args.ctx or 16384
    C = args.chunk
    models = [P.ModelSpec(n, L, H, 128, 2, Hq) for n, L, H, Hq in SERVICES]
    cache = P.UnifiedKvCache(models, 16, 1, 4 * R * (ctx // 16 + 2) + 64, phys_layers=2, allocate_storage=True)
    groups, rid = [], 1
    for m in range(len(SERVICES)):
        ids = []
        for _ in range(R):
            assert cache.try_allocate(rid, m, ctx)
            ids.append(rid)
            rid += 1
        groups.append((m, ids))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    cache.set_stream(stream)
    cache.synth_fill(1, 1.0, stream)
    b = cache.batch(groups)
    gen = torch.Generator(device="cuda").manual_seed(3)
    qs = [torch.randn((R, C, Hq, 128), generator=gen, device="cuda").half() for _, _, _, Hq in SERVICES]
    outs = [torch.empty_like(x) for x in qs]
    p0 = ctx - C
    flops = sum(4.0 * 128 * Hq * R * (C * p0 + C * (C + 1) / 2) for _, _, _, Hq in SERVICES)
    launches0 = cache.kernel_launches()
    for _ in range(args.warmup):
        b.prefill(qs, outs, 0, C, stream=stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(0) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            b.prefill(qs, outs, 0, C, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    tflops = flops / (ms * 1e-3) / 1e12
    launches = cache.kernel_launches() - launches0 - args.warmup
    # e2e: every step copies each service's q from pinned host memory and its output back;
    # per-service launches on the compute stream overlap service s's prefill with the H2D of
    # s+1 (copy-in stream) and the D2H of s-1 (copy-out stream)
    hq = [x.cpu().pin_memory() for x in qs]
    ho = [torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in outs]
    sb = [cache.batch([g]) for g in groups]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    s_in.wait_stream(stream)
    s_out.wait_stream(stream)
    done = [None] * len(groups)
    for _ in range(args.steps):
        for i in range(len(groups)):
            with torch.cuda.stream(s_in):
                if done[i] is not None:
                    s_in.wait_event(done[i])  # q_i is free once the previous step's prefill_i ran
                qs[i].copy_(hq[i], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(s_in)
            stream.wait_event(ev_in)
            if done[i] is not None:
                stream.wait_stream(s_out)  # out_i of the previous step copied out
            sb[i].prefill([qs[i]], [outs[i]], 0, C, stream=stream)
            done[i] = torch.cuda.Event()
            done[i].record(stream)
            s_out.wait_event(done[i])
            with torch.cuda.stream(s_out):
                ho[i].copy_(outs[i], non_blocking=True)
    stream.wait_stream(s_out)
    t1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = t0.elapsed_time(t1) / args.steps
    io_bytes = sum(x.numel() * 2 for x in qs)
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peak, peak_kind = float(json.load(f)["bf16_tflops"]), "measured (burst, cuBLAS bf16)"
    except Exception:
        peak, peak_kind = 2250.0, "fallback (nominal dense bf16)"
    # CPU baseline: the fp32 oracle on a bounded sample (first request of each service, 32 q tokens)
    cpu = None
    if not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle_py as O
        cores = os.cpu_count() or 1
        img = cache.read_blocks(np.arange(cache.pool_size(), dtype=np.int32))
        qn_tok = 32
        done, cflops, t_start = 0, 0.0, time.perf_counter()
        while time.perf_counter() - t_start < args.cpu_seconds / 2 or done == 0:
            for (m, ids), q in zip(groups, qs):
                Lh = cache.layout(m)
                lay = O.layout(Lh.merged_stride, Lh.native_stride, Lh.layer_stride, Lh.head_stride, Lh.kv_stride,
                               16, 128, Lh.kv_heads, Lh.q_heads, Lh.phys_layers, 0)
                tab = np.array([cache.block_table(ids[0])], np.int32)
                qh = q[0, C - qn_tok:].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
                qh = qh.reshape(qn_tok, -1, 128)
                O.prefill_attention(lay, img, 0, tab, np.array([ctx - qn_tok], np.int64),
                                    np.array([qn_tok], np.int64), qh, 1.0 / np.sqrt(128.0), nthreads=cores)
                Hq = SERVICES[m][3]
                cflops += 4.0 * 128 * Hq * (qn_tok * (ctx - qn_tok) + qn_tok * (qn_tok + 1) / 2)
            done += 1
        dt = time.perf_counter() - t_start
        cpu = {"value": round(cflops / dt / 1e12, 6), "unit": "TFLOP/s", "cores": cores, "kind": "port",
               "sample": f"fp32 oracle causal prefill of the last {qn_tok} tokens of one request per service at "
                         f"ctx {ctx}, {done} reps in {dt:.1f} s (oracle/attn_oracle.c; the reference has no attention)"}
    res = {
        "metric": "chunked-prefill attention TFLOP/s (unified pool, tcgen05)", "value": round(tflops, 1),
        "unit": "TFLOP/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp16",
        "data": "synthetic (SplitMix64 K/V pool, randn q)",
        "config": {"workload": f"prefill: 4 services (config-2 shapes) x {R} requests, last {C} tokens of a "
                               f"{ctx}-token context, causal, layer 0; useful (causal) flops only",
                   "l2": "K/V per step larger than L2; no flush"},
        "e2e": {"value": round(flops / (e2e_ms * 1e-3) / 1e12, 1), "unit": "TFLOP/s",
                "h2d_bytes_per_step": int(io_bytes), "d2h_bytes_per_step": int(io_bytes),
                "ms_per_step": round(e2e_ms, 4),
                "note": "per-service launches, H2D / D2H on their own streams overlapping the other services' prefill"},
        "roofline": {"bound": "tensor", "kernel": PREFILL_KERNEL,
                     "achieved": round(tflops, 1), "peak": peak, "peak_kind": peak_kind, "unit": "TFLOP/s",
                     "frac": round(tflops / peak, 4), "traffic": None,
                     "ncu": PREFILL_NCU},
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    if cpu:
        res["cpu_baseline"] = cpu
    print(json.dumps(res), flush=True)


def run_reference(args):
    """Reference arm: the reference's own CPU path for this workload on the host cores —
    the reference has no attention, so the fp32 oracle port stands in for decode and the
    unmodified reference allocator (oracle/_ref) replays the step's allocation ops."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_py as O

    services = {"config1": SERVICES_C1, "config2d": SERVICES_MIXED_D}.get(args.workload, SERVICES)
    ctx_default = {"config1": 512, "config4": 4096}.get(args.workload, 2048)
    args.ctx = args.ctx or ctx_default
    cores = os.cpu_count() or 1
    # synthetic host pool for a bounded sample: per service `per` requests at ctx
    per = args.cpu_requests
    models = [(s[1], s[2], hd(s), 2) for s in services]
    allocator = O.RefCache(models, pool=200000) if O.ref_available() else O.OracleCache(models, pool=200000)
    kind = "reference" if O.ref_available() else "port"
    rid = 1
    ids = {m: [] for m in range(len(services))}
    for r in range(per):
        for m in range(len(services)):
            assert allocator.try_allocate(rid, m, args.ctx)
            ids[m].append(rid)
            rid += 1
    merged = int(O.plan_merged_shape(models))
    rng = np.random.default_rng(0)
    work = []
    nbytes = 0.0
    used = sorted({b for m in ids for i in ids[m] for b, _ in allocator.block_table(i)})
    remap = {b: k for k, b in enumerate(used)}
    # 4 physical layers like the GPU arm; image holds only the used blocks
    Lp = args.phys_layers
    stride = 0
    lays = []
    for m, s in enumerate(services):
        L, H, Hq, d = s[1], s[2], s[3], hd(s)
        layer_stride = H * 2 * 16 * d * 2
        native = min(Lp, L) * layer_stride
        lays.append((L, H, Hq, layer_stride, native, d))
    sub = [int(merged // (16 * s[1] * 2 * s[2] * hd(s) * 2)) for s in services]
    stride = max(s * l[4] for s, l in zip(sub, lays))
    stride = (stride + 1023) // 1024 * 1024
    img = rng.integers(0, 0x3C00, size=len(used) * stride // 2, dtype=np.uint16).view(np.uint8)
    for m, (L, H, Hq, layer_stride, native, d) in enumerate(lays):
        olay = O.layout(stride, native, layer_stride, 2 * 16 * d * 2, 16 * d * 2, 16, d, H, Hq, min(Lp, L), 0)
        tabs = np.array([[(remap[b], s) for b, s in allocator.block_table(i)] for i in ids[m]], np.int32)
        ctx = np.full(len(ids[m]), args.ctx, np.int64)
        qh = rng.integers(0, 0x3C00, size=(len(ids[m]), Hq, d), dtype=np.uint16)
        work.append((olay, tabs, ctx, qh))
        nbytes += float(ctx.sum()) * H * d * 2 * 2
    # allocator: one decode step of grows for the sampled requests, timed separately
    def one_step():
        t = time.perf_counter()
        for olay, tabs, ctx, qh in work:
            O.decode_attention(olay, img, 0, tabs, ctx, qh, 1.0 / np.sqrt(olay.head_dim), nthreads=cores)
        return time.perf_counter() - t

    for _ in range(min(args.warmup, 1)):
        one_step()
    times = [one_step() for _ in range(args.steps)]
    dt = sum(times)
    value = nbytes * len(times) / dt / 1e9
    # allocator: the decode-step op stream of the workload's request count (every request
    # +1 token per step, 64 steps), replayed through the reference allocator single-threaded
    # (kv_cache.hpp:45); the array is built before the timer starts
    n_alloc_req = args.requests or {"config1": 32, "config3": 64, "config4": 32}.get(args.workload, 256)
    nsteps = 64
    acache = (O.RefCache if kind == "reference" else O.OracleCache)(models, pool=400000)
    aops = [(0, 1 + r * len(services) + m, m, args.ctx) for r in range(n_alloc_req) for m in range(len(services))]
    acache.replay(aops)
    ops = [(0, 1 + r * len(services) + m, m, args.ctx + s_ + 1) for s_ in range(nsteps)
           for r in range(n_alloc_req) for m in range(len(services))]
    arr = O.ops_array(ops)
    t = time.perf_counter()
    acache.replay_array(arr, len(ops))
    alloc_ns = (time.perf_counter() - t) / max(1, len(ops)) * 1e9
    res = {
        "impl": "reference",
        "metric": "unified-KV paged decode attention HBM GB/s (mixed services)",
        "value": round(value, 3), "unit": "GB/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / len(times) * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic", "config": {"workload": f"{args.workload} decode, bounded CPU sample", "ctx": args.ctx,
                                        "requests_per_service": per},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": f"fp32 oracle decode (no reference attention exists), {per} requests per "
                                   f"service at ctx {args.ctx}, 1 layer per step; allocator: {kind} "
                                   f"replay of {len(ops)} decode-step grows, {alloc_ns:.1f} ns/op"},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "allocator_ns_per_op": round(alloc_ns, 2), "allocator_kind": kind,
    }
    print(json.dumps(res), flush=True)


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch this script as N ranks (one process per
    GPU, torch.distributed.run on 127.0.0.1); rank 0 prints the JSON line."""
    import socket

    env = dict(os.environ)
    if args.share_gpu:
        env["SKV_BENCH_SHARE_GPU"] = "1"
        env.setdefault("SKV_BENCH_BACKEND", "gloo")
    elif args.impl == "ours":
        try:
            import torch
            have = torch.cuda.device_count()
        except Exception:  # noqa: BLE001
            have = 0
        if have < args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} but this box has {have} GPU(s); use --share-gpu "
                                       "for a functional dry run"}), flush=True)
            return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config2",
                    choices=["config1", "config2", "config2d", "config3", "config4", "config5", "prefill"])
    ap.add_argument("--chunk", type=int, default=2048, help="prefill workload: chunk length")
    ap.add_argument("--rate", type=float, default=20.0, help="config3 arrival rate (requests/s)")
    ap.add_argument("--pool-gb", dest="pool_gb", type=float, default=100.0, help="config3 pool size")
    ap.add_argument("--occupancy", type=float, default=0.70, help="config3 admission occupancy target")
    ap.add_argument("--requests", type=int, default=0, help="decode requests per service (0 = workload default)")
    ap.add_argument("--ctx", type=int, default=0, help="context length (0 = workload default)")
    ap.add_argument("--phys-layers", dest="phys_layers", type=int, default=None,
                    help="physical layers per native block (0 = all; default 4, config2d 2)")
    ap.add_argument("--cpu-seconds", dest="cpu_seconds", type=float, default=12.0,
                    help="CPU-baseline sample duration (bounded sample of the workload)")
    ap.add_argument("--cpu-requests", dest="cpu_requests", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", dest="no_cpu_baseline", action="store_true")
    ap.add_argument("--no-tp-group", dest="no_tp_group", action="store_true",
                    help="N>1: run config-2 replicas only (no head-sharded 70B service)")
    ap.add_argument("--share-gpu", dest="share_gpu", action="store_true",
                    help="dry run of the N-rank path on a box with fewer GPUs: every rank on GPU 0, gloo "
                         "(functional only; the numbers are meaningless)")
    ap.add_argument("--no-faithful", dest="no_faithful", action="store_true",
                    help="skip the other-config samples (capacity-faithful config 2, configs 4, 1, 3) in the default line")
    ap.add_argument("--no-config4", dest="no_config4", action="store_true",
                    help="skip only the config-4 sample in the default line")
    ap.add_argument("--no-prefill", dest="no_prefill", action="store_true",
                    help="skip the chunked-prefill sample in the decode line")
    ap.add_argument("--no-parity", dest="no_parity", action="store_true",
                    help="skip the post-timing oracle check of a sample of the measured launch")
    ap.add_argument("--no-graph", dest="no_graph", action="store_true",
                    help="eager launches instead of a CUDA graph per step")
    args = ap.parse_args()
    if args.phys_layers is None:  # config2d: the d=64 service packs 25 sub-slots, so slice finer to fit
        args.phys_layers = 2 if args.workload == "config2d" else 4
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None and int(env_world) != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={env_world}: launch one rank per GPU "
                                   f"(torchrun --nproc-per-node {args.gpus}) or drop --gpus"}), flush=True)
        sys.exit(2)
    if env_world is None and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "config3":
        run_churn(args)
    elif args.workload == "config5":
        run_config5(args)
    elif args.workload == "prefill":
        run_prefill(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()

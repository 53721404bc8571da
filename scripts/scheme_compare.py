"""Merged vs split scheme on the same GPU kernels.

For the paper's pairs (A-B = service A sharing the pool with B; L7 = Llama-2-7B shape,
L13 = Llama-2-13B shape) and config 1's batch (R decode requests per service at ctx):
 - decode: one full decode step (all layers, fused append) per scheme, CUDA-graph replay
 - allocation: GPU time of one decode-step grow (+1 token for every request, the step
   that crosses a 16-token boundary, so every request claims a native block)
 - block-table size: live entries and device bytes
usage: python scripts/scheme_compare.py [R] [ctx]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2504_15720_b200 as P

SHAPES = {"L7": ("llama-2-7b", 32, 32, 32), "L13": ("llama-2-13b", 40, 40, 40)}


def run(pair, R, ctx):
    names = pair.split("-")
    specs = [SHAPES[n] for n in names]
    models = [P.ModelSpec(f"{n}#{i}", L, H, 128, 2, Hq) for i, (n, L, H, Hq) in enumerate(specs)]
    nblk = (ctx + 64 + 15) // 16
    split_blocks = sum(R * nblk * L * H for _, L, H, _ in specs) + 64
    merged = P.plan_merged_shape(models)
    subs = [int(merged // P.native_block_bytes(m)) for m in models]
    pool = sum(-(-R * nblk // s) for s in subs) + 16
    res = {"pair": pair, "requests_per_service": R, "ctx": ctx}
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    for scheme in ("merged", "split"):
        if scheme == "merged":
            c = P.UnifiedKvCache(models, 16, 1, pool, allocate_storage=True, max_requests=2 * R + 8,
                                 max_blocks_per_request=nblk + 1)
        else:
            c = P.SplitKvCache(models, 16, 1, split_blocks, max_requests=2 * R + 8, max_blocks_per_request=nblk + 1)
        c.set_stream(stream)
        groups, rid = [(m, []) for m in range(len(models))], 1
        for r in range(R):
            for m in range(len(models)):
                if scheme == "merged":
                    assert c.try_allocate(rid, m, ctx)
                else:
                    assert c.grow([rid], [m], [ctx]).all()
                groups[m][1].append(rid)
                rid += 1
        c.synth_fill(7, 1.0, stream)
        b = c.batch(groups)
        q = [torch.randn((R, Hq, 128), device="cuda").half() for _, _, _, Hq in specs]
        o = [torch.empty_like(x) for x in q]
        k = [torch.randn((R, 1, H, 128), device="cuda").half() for _, _, H, _ in specs]
        v = [torch.randn((R, 1, H, 128), device="cuda").half() for _, _, H, _ in specs]
        nl = max(L for _, L, _, _ in specs)
        # allocation: grow to the next block boundary, then time the step that claims blocks
        for _ in range((16 - ctx % 16) % 16):
            b.grow(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        b.grow(1)  # every request crosses into a new native block
        if scheme == "merged":
            c.flush(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        grow_ms = e0.elapsed_time(e1)
        for layer in range(nl):
            b.decode(q, o, layer, stream=stream, k=k, v=v)  # plan for this context
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for layer in range(nl):
                b.decode(q, o, layer, stream=stream, k=k, v=v)
        g.replay()
        torch.cuda.synchronize()
        reps = 5
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        step_ms = e0.elapsed_time(e1) / reps
        kv = sum(b.decode_bytes(layer)[0] for layer in range(nl))
        if scheme == "merged":
            entries = c.table_entries()
            table_dev = (2 * R) * (nblk + 1) * 8
        else:
            entries = c.table_entries()
            table_dev = (2 * R + 8) * nl * max(H for _, _, H, _ in specs) * (nblk + 1) * 8
        res[scheme] = {"decode_step_ms": round(step_ms, 4), "decode_GBps": round(kv / step_ms / 1e6, 1),
                       "grow_step_ms": round(grow_ms, 4), "live_table_entries": int(entries),
                       "table_device_bytes": int(table_dev)}
        del b, g
        c.close()
    res["split_over_merged"] = {"decode_time": round(res["split"]["decode_step_ms"] / res["merged"]["decode_step_ms"], 4),
                                "grow_time": round(res["split"]["grow_step_ms"] / max(1e-9, res["merged"]["grow_step_ms"]), 2),
                                "table_entries": round(res["split"]["live_table_entries"] /
                                                       max(1, res["merged"]["live_table_entries"]), 1)}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    R = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    for pair in ("L7-L7", "L7-L13", "L13-L7"):
        run(pair, R, ctx)

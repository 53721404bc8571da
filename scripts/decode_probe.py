"""Decode launch timing sweep: services x requests x ctx on a faithful pool, per split_tokens.

usage: python scripts/decode_probe.py [config1|config2s] [ctx] [requests/service] [splits...]
Prints one JSON line per split setting: ms per decode launch (layer 0), GB/s of algorithmic bytes.
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2504_15720_b200 as P

SETS = {
    "config1": [("llama-2-7b", 32, 32, 32), ("llama-2-13b", 40, 40, 40)],
    "13b": [("llama-2-13b", 40, 40, 40)],
    "7b": [("llama-2-7b", 32, 32, 32)],
    "config2s": [("llama-3-8b", 32, 8, 32), ("mistral-7b", 32, 8, 32), ("llama-2-13b", 40, 40, 40),
                 ("opt-6.7b", 32, 32, 32)],
}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "config1"
    ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 520
    R = int(sys.argv[3]) if len(sys.argv) > 3 else 32
    splits = [int(x) for x in sys.argv[4:]] or [0]
    serv = SETS[name]
    models = [P.ModelSpec(n, L, H, 128, 2, Hq) for n, L, H, Hq in serv]
    merged = P.plan_merged_shape(models)
    subs = [int(merged // P.native_block_bytes(m)) for m in models]
    pool = sum(-(-R * ((ctx + 15) // 16) // s) for s in subs) + 16
    cache = P.UnifiedKvCache(models, 16, 1, pool, allocate_storage=True, phys_layers=1,
                             max_requests=R * len(serv) + 8, max_blocks_per_request=ctx // 16 + 2)
    groups = [(m, []) for m in range(len(serv))]
    rid = 1
    for r in range(R):
        for m in range(len(serv)):
            assert cache.try_allocate(rid, m, ctx)
            groups[m][1].append(rid)
            rid += 1
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    cache.set_stream(s)
    cache.synth_fill(1, 1.0, s)
    b = cache.batch(groups)
    q = [torch.randn((R, Hq, 128), device="cuda").half() for _, _, _, Hq in serv]
    out = [torch.empty_like(x) for x in q]
    nbytes = b.decode_bytes(0)[1]
    for sp in splits:
        for _ in range(5):
            b.decode(q, out, 0, split_tokens=sp, stream=s)
        reps = 50
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                b.decode(q, out, 0, split_tokens=sp, stream=s)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(json.dumps({"set": name, "ctx": ctx, "R": R, "split": sp, "ms": round(ms, 4),
                          "GBps": round(nbytes / ms / 1e6, 1), "bytes": nbytes}), flush=True)


if __name__ == "__main__":
    main()

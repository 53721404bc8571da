"""Per-warp timeline of one decode launch (SKV_TRACE=1): start / after-wait / end spread.

usage: SKV_TRACE=1 python scripts/decode_trace.py <set> <ctx> <R> [split]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
os.environ.setdefault("SKV_TRACE", "1")
import paper_2504_15720_b200 as P
from decode_probe import SETS


def main():
    name, ctx, R = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    split = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    serv = SETS[name]
    models = [P.ModelSpec(n, L, H, 128, 2, Hq) for n, L, H, Hq in serv]
    merged = P.plan_merged_shape(models)
    subs = [int(merged // P.native_block_bytes(m)) for m in models]
    pool = sum(-(-R * ((ctx + 15) // 16) // s) for s in subs) + 16
    cache = P.UnifiedKvCache(models, 16, 1, pool, allocate_storage=True, phys_layers=2,
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
    k = [torch.randn((R, 1, H, 128), device="cuda").half() for _, _, H, _ in serv]
    v = [torch.randn((R, 1, H, 128), device="cuda").half() for _, _, H, _ in serv]
    out = [torch.empty_like(x) for x in q]
    nbytes = b.decode_bytes(0)[1]
    for i in range(6):
        b.decode(q, out, i % 2, split_tokens=split, stream=s, k=k, v=v)
    torch.cuda.synchronize()
    t = b.decode_trace().astype(np.int64)
    t0 = t[:, 0].min()
    st, wt, en = t[:, 0] - t0, t[:, 1] - t0, t[:, 2] - t0
    tiles, items = t[:, 3] >> 32, t[:, 3] & 0xffffffff
    span = en.max()
    busy = (en - wt).sum() / (len(t) * (span - np.median(wt)))
    pct = lambda x: [int(np.percentile(x, p)) for p in (0, 10, 50, 90, 100)]  # noqa: E731
    print(json.dumps({"set": name, "ctx": ctx, "R": R, "split": split, "warps": len(t), "span_us": span / 1e3,
                      "GBps_span": round(nbytes / span, 1), "start_ns_pct": pct(st), "wait_ns_pct": pct(wt),
                      "end_ns_pct": pct(en), "tiles_pct": pct(tiles), "items_pct": pct(items),
                      "busy_frac": round(float(busy), 3)}))
    # end-time histogram (10 bins)
    h, e = np.histogram(en, bins=10)
    print("end hist:", list(zip([int(x) for x in e[:-1]], h.tolist())))


if __name__ == "__main__":
    main()

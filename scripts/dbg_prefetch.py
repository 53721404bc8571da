"""Debug: churn-style eager decode loop (events around each launch), per-launch sum vs total."""
import os
import sys
import torch
sys.path.insert(0, ".")
import paper_2504_15720_b200 as P

serv = [(32, 8, 32), (40, 40, 40), (32, 32, 32)]
models = [P.ModelSpec(f"s{i}", L, H, 128, 2, Hq) for i, (L, H, Hq) in enumerate(serv)]
cache = P.UnifiedKvCache(models, 16, 1, 2000, allocate_storage=True, max_blocks_per_request=200)
groups, rid = [], 1
for m in range(3):
    ids = []
    for r in range(10):
        assert cache.try_allocate(rid, m, 300 + 97 * r)
        ids.append(rid)
        rid += 1
    groups.append((m, ids))
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
cache.set_stream(s)
cache.synth_fill(1, 1.0, s)
b = cache.batch(groups)
q = [torch.randn((10, Hq, 128), device="cuda").half() for _, _, Hq in serv]
o = [torch.empty_like(x) for x in q]
kv = [torch.randn((10, 1, H, 128), device="cuda").half() for _, H, _ in serv]
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
import time
gap = float(os.environ.get("GAP_US", "0")) * 1e-6
for it in range(4):
    b.grow(1)
    marks = []
    t0, t1 = ev(), ev()
    t0.record(s)
    for layer in range(40):
        e = [ev(), ev()]
        e[0].record(s)
        b.decode(q, o, layer, stream=s, k=kv, v=kv)
        e[1].record(s)
        if gap:
            t_end = time.perf_counter() + gap
            while time.perf_counter() < t_end:
                pass
        marks.append(e)
    t1.record(s)
    torch.cuda.synchronize()
    print(os.environ.get("SKV_NO_PREFETCH", "0"), "sum of per-launch ms", round(sum(a.elapsed_time(c) for a, c in marks), 3),
          "total ms", round(t0.elapsed_time(t1), 3))

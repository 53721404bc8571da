"""Quick prefill timing: 4 config-2 services (head dim D), R requests each, context CTX, chunk Q (last Q tokens).
Usage: prefill_probe.py R CTX Q [reps] [D]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2504_15720_b200 as P

SERV = [("llama-3-8b", 32, 8, 32), ("mistral-7b", 32, 8, 32), ("llama-2-13b", 40, 40, 40), ("opt-6.7b", 32, 32, 32)]


def main(R=8, CTX=2048, Q=512, reps=10, D=128):
    models = [P.ModelSpec(n, L, H, D, 2, Hq) for n, L, H, Hq in SERV]
    cache = P.UnifiedKvCache(models, 16, 1, 4 * R * (CTX // 16 + 2) + 64, phys_layers=2, allocate_storage=True)
    groups = []
    rid = 1
    for m in range(4):
        ids = []
        for _ in range(R):
            assert cache.try_allocate(rid, m, CTX)
            ids.append(rid)
            rid += 1
        groups.append((m, ids))
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    cache.set_stream(s)
    cache.synth_fill(1, 1.0, s)
    b = cache.batch(groups)
    qs = [torch.randn((R, Q, Hq, D), device="cuda").half() for _, _, _, Hq in SERV]
    outs = [torch.empty_like(x) for x in qs]
    p0 = CTX - Q
    flops = sum(4 * D * Hq * R * (Q * p0 + Q * (Q + 1) / 2) for _, _, _, Hq in SERV)
    for _ in range(3):
        b.prefill(qs, outs, 0, Q, stream=s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        b.prefill(qs, outs, 0, Q, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"R": R, "ctx": CTX, "q_len": Q, "head_dim": D, "ms": ms, "tflops": flops / ms / 1e9,
                      "frac_of_1644": flops / ms / 1e9 / 1644.2}))


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:]])

"""Measured B200 decode-attention coefficients for the reference cost model.

The reference prices a decode iteration as decode_fixed + decode_per_seq * B +
decode_per_context_token * (total context tokens) (cost_model.hpp:116-124); the last
term is exactly the paged-attention KV read this repository implements.  For each
reference model class (and TP size) this measures, on one B200, the time of one full
decode step of the unified-pool kernel (all layers, CUDA-graph replay) at two context
lengths and fits the per-context-token slope.  It writes the reference's own INI
[cost <model> tp=<n>] sections (config.hpp:311-328) with decode_per_context_token
replaced by the measurement and every other coefficient (GEMM-dominated, not on this
path) kept from default_cost_model (cost_model.hpp:191-262), so the reference simulator
can be run with B200-measured attention cost.
usage: python scripts/calibrate_cost.py [out.ini]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2504_15720_b200 as P

# reference default_cost_model: (layers, kv heads, q heads), {tp: coefficients}
# coefficients: prefill_fixed, prefill_per_token, decode_fixed, decode_per_seq,
#               decode_per_context_token, activation_base_gb, activation_per_seq_gb
REF = {
    "llama2-7b": ((32, 32, 32), {1: (2.0e-3, 8.0e-5, 6.0e-3, 4.0e-4, 2.5e-7, 0.8, 0.03),
                                 2: (5.0e-3, 4.8e-5, 7.5e-3, 2.4e-4, 1.4e-7, 0.5, 0.02),
                                 4: (9.0e-3, 2.8e-5, 1.0e-2, 1.4e-4, 0.8e-7, 0.35, 0.013),
                                 8: (1.4e-2, 1.8e-5, 1.4e-2, 0.9e-4, 0.5e-7, 0.25, 0.009)}),
    "llama2-13b": ((40, 40, 40), {1: (2.5e-3, 1.45e-4, 9.0e-3, 6.5e-4, 4.2e-7, 1.1, 0.045),
                                  2: (5.5e-3, 8.7e-5, 1.1e-2, 3.9e-4, 2.3e-7, 0.7, 0.028),
                                  4: (1.0e-2, 5.2e-5, 1.4e-2, 2.3e-4, 1.3e-7, 0.5, 0.018),
                                  8: (1.6e-2, 3.2e-5, 1.9e-2, 1.5e-4, 0.8e-7, 0.35, 0.012)}),
    "llama2-70b": ((80, 64, 64), {4: (1.8e-2, 2.6e-4, 2.6e-2, 9.0e-4, 5.5e-7, 1.4, 0.055),
                                  8: (2.6e-2, 1.5e-4, 3.3e-2, 5.6e-4, 3.2e-7, 0.9, 0.035)}),
    "opt-6.7b": ((32, 32, 32), {1: (1.9e-3, 7.6e-5, 5.7e-3, 3.8e-4, 2.4e-7, 0.8, 0.03),
                                2: (4.8e-3, 4.6e-5, 7.2e-3, 2.3e-4, 1.35e-7, 0.5, 0.02),
                                4: (8.6e-3, 2.7e-5, 9.6e-3, 1.35e-4, 0.77e-7, 0.35, 0.013),
                                8: (1.35e-2, 1.7e-5, 1.35e-2, 0.87e-4, 0.48e-7, 0.25, 0.009)}),
}
KEYS = ["prefill_fixed", "prefill_per_token", "decode_fixed", "decode_per_seq", "decode_per_context_token",
        "activation_base_gb", "activation_per_seq_gb"]


def step_ms(shape, tp, R, ctx):
    L, H, Hq = shape
    m = P.ModelSpec("m", L, H, 128, 2, Hq)
    nblk = (ctx + 32 + 15) // 16
    cache = P.UnifiedKvCache([m], 16, tp, R * nblk + 8, allocate_storage=True, phys_layers=4,
                             max_requests=R + 8, max_blocks_per_request=nblk + 1)
    for r in range(R):
        assert cache.try_allocate(r + 1, 0, ctx)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    cache.set_stream(s)
    cache.synth_fill(3, 1.0, s)
    b = cache.batch([(0, list(range(1, R + 1)))])
    hq, hk = Hq // tp, H // tp
    q = torch.randn((R, hq, 128), device="cuda").half()
    o = torch.empty_like(q)
    k = torch.randn((R, 1, hk, 128), device="cuda").half()
    for layer in range(L):
        b.decode([q], [o], layer, stream=s, k=[k], v=[k])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for layer in range(L):
            b.decode([q], [o], layer, stream=s, k=[k], v=[k])
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(5):
        g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    del g, b
    cache.close()
    torch.cuda.set_stream(torch.cuda.default_stream())
    return ms


def main(out_path):
    R, c1, c2 = 64, 1024, 4096
    lines = ["# B200-measured decode attention cost (scripts/calibrate_cost.py): decode_per_context_token",
             "# is the unified-pool paged decode kernel's time per context token of a full decode step",
             "# (all layers, per-rank heads at tp); other coefficients: reference default_cost_model."]
    rows = []
    for mid, (shape, entries) in REF.items():
        for tp, coeffs in entries.items():
            t1, t2 = step_ms(shape, tp, R, c1), step_ms(shape, tp, R, c2)
            per_tok = (t2 - t1) / 1e3 / (R * (c2 - c1))
            vals = list(coeffs)
            rows.append({"model": mid, "tp": tp, "reference_s": vals[4], "b200_s": per_tok,
                         "speedup": round(vals[4] / per_tok, 2), "step_ms_ctx1k": round(t1, 3),
                         "step_ms_ctx4k": round(t2, 3)})
            vals[4] = per_tok
            lines.append(f"\n[cost {mid} tp={tp}]")
            lines += [f"{k_} = {v:.6g}" for k_, v in zip(KEYS, vals)]
            print(json.dumps(rows[-1]), flush=True)
    with open(out_path, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "b200_cost.ini")

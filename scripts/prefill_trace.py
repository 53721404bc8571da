"""Per-role wait profile of the warp-specialised prefill kernels (build: make SKV_EXTRA=-DSKV_PF_TRACE; run with SKV_TRACE=1).

usage: SKV_TRACE=1 python scripts/prefill_trace.py R CTX Q
Prints the mean fraction of each CTA's cycles spent in each wait.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
os.environ.setdefault("SKV_TRACE", "1")
import paper_2504_15720_b200 as P

SERV = [("llama-3-8b", 32, 8, 32), ("mistral-7b", 32, 8, 32), ("llama-2-13b", 40, 40, 40), ("opt-6.7b", 32, 32, 32)]
R, CTX, Q = (int(x) for x in sys.argv[1:4])
models = [P.ModelSpec(n, L, H, 128, 2, Hq) for n, L, H, Hq in SERV]
cache = P.UnifiedKvCache(models, 16, 1, 4 * R * (CTX // 16 + 2) + 64, phys_layers=2, allocate_storage=True)
groups, rid = [], 1
for m in range(4):
    ids = []
    for _ in range(R):
        assert cache.try_allocate(rid, m, CTX)
        ids.append(rid)
        rid += 1
    groups.append((m, ids))
cache.synth_fill(1, 1.0)
b = cache.batch(groups)
qs = [torch.randn((R, Q, Hq, 128), device="cuda").half() for _, _, _, Hq in SERV]
outs = [torch.empty_like(x) for x in qs]
for _ in range(2):
    b.prefill(qs, outs, 0, Q)
torch.cuda.synchronize()
t = b.decode_trace(1 << 20).reshape(-1, 16).astype(np.float64)
t = t[t[:, 13] > 0]
tot = t[:, 13]
names = ["load:kv_empty", "mma:q_full", "mma:kv_full", "mma:p_full_A", "mma:p_full_B",
         "smA:s_full", "smA:pv_corr", "smA:pv_last", "-", "smB:s_full", "smB:pv_corr", "smB:pv_last"]
if os.environ.get("SEAKV_PREFILL_V", "10") == "10":  # CTA pairs: softmax halves c=0/1 of the same rows
    names = ["load:kv_empty", "mma:q_full", "mma:kv_full", "mma:p_full", "mma:issue",
             "sm0:s_full", "sm0:pv_corr", "sm0:pv_last", "sm0:max_xchg", "sm1:s_full", "sm1:pv_corr", "sm1:pv_last",
             "sm1:max_xchg", "-", "-", "mma:descs"]
if os.environ.get("SKV_PREFILL_PP", "1") != "0":  # ping-pong kernel (two query tiles per CTA)
    names = ["load:kv_empty", "mma:q_full", "mma:kv_full", "mma:p_full_A", "mma:p_full_B",
             "smA:s_full", "smA:o_done", "-", "-", "smB:s_full", "smB:o_done", "-", "-", "-", "-", "mma:issue"]
res = {n: round(float((t[:, i] / tot).mean()), 4) for i, n in enumerate(names) if n != "-"}
res["ctas"] = int(len(t))
res["mean_cta_us_at_1.9GHz"] = round(float(tot.mean()) / 1.9e3, 1)
res["mean_n_kt"] = round(float(t[:, 14].mean()), 1)
print(json.dumps(res))

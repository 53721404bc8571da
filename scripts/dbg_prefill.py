"""Debug: prefill output NaN/error map vs the oracle for one small case."""
import sys
import numpy as np
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests"); sys.path.insert(0, "oracle")
import oracle_py as O
import paper_2504_15720_b200 as P
from test_gpu_decode import build_pool, host_image, oracle_layout, tables_of

shapes = [(2, 2, 2)]
ctx, q_len = int(sys.argv[1]), int(sys.argv[2])
cache, groups = build_pool(shapes, [[ctx]])
gen = torch.Generator(device="cuda").manual_seed(11)
q = (torch.rand((1, q_len, 2, 128), generator=gen, device="cuda") * 2 - 1).half()
o = torch.full_like(q, float("nan"))
b = cache.batch(groups)
b.prefill([q], [o], 1, q_len)
torch.cuda.synchronize()
img = host_image(cache)
ref = O.prefill_attention(oracle_layout(cache, 0), img, 1, tables_of(cache, groups[0][1]), np.array([ctx - q_len]),
                          np.array([q_len]), q.view(torch.int16).cpu().numpy().view(np.uint16).reshape(q_len, 2, 128),
                          1.0 / np.sqrt(128.0))
got = o.float().cpu().numpy().reshape(q_len, 2, 128)
nan = np.isnan(got)
print("nan rows:", sorted(set(np.nonzero(nan)[0].tolist()))[:40], "count", nan.any(axis=(1, 2)).sum())
err = np.nan_to_num(np.abs(got - ref), nan=99)
bad = np.nonzero(err.max(axis=(1, 2)) > 2e-3)[0]
print("bad rows:", bad[:40].tolist(), "n", len(bad), "max err", float(err.max()))

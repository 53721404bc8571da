import sys, numpy as np, torch
sys.path[:0] = ['.', 'oracle', 'tests']
import oracle_py as O
import paper_2504_15720_b200 as P
from paper_2504_15720_b200.tp import head_slice
from test_gpu_decode import oracle_layout, tables_of
import test_gpu_tp as T
g = torch.Generator(device="cuda").manual_seed(3)
# poison freed memory first, like the earlier test did
junk = torch.full((1 << 28,), float("nan"), device="cuda").half(); del junk
kv = [[(torch.randn((c, T.H, 2, T.D), generator=g, device="cuda") * 0.5).half() for _ in range(T.L)] for c in T.CTX]
q = torch.randn((len(T.CTX), T.HQ, T.D), generator=g, device="cuda").half()
for tp, r in ((1, 0), (2, 0), (2, 1)):
    c = T._pool(tp, r, kv)
    ids = [i + 1 for i in range(len(T.CTX))]
    b = c.batch([(0, ids)])
    hs = head_slice(T.HQ, tp, r)
    ql = q[:, hs].contiguous()
    o = torch.empty_like(ql)
    for layer in range(T.L):
        b.decode([ql], [o], layer)
        torch.cuda.synchronize()
        img = c.read_blocks(np.arange(c.pool_size()))
        ref = O.decode_attention(oracle_layout(c, 0), img, layer, tables_of(c, ids), np.array(T.CTX, np.int64),
                                 ql.view(torch.int16).cpu().numpy().view(np.uint16), 1 / np.sqrt(128))
        got = o.float().cpu().numpy()
        bad = np.argwhere(~np.isfinite(got))
        print("tp", tp, "rank", r, "layer", layer, "maxerr", np.nanmax(np.abs(got - ref)), "nan_in_ref", np.isnan(ref).sum(),
              "nan rows", sorted(set(map(tuple, bad[:, :2].tolist())))[:10])

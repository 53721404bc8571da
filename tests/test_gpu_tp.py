"""Head-sharded (tp=2) service on the GPU kernels: two rank-local pools (tp_size=2)
plus an unsharded pool on one GPU, identical K/V written through the append
kernel; Σ_ranks (local decode · W_o row slice) must equal the unsharded result.
(The cross-GPU AllReduce itself is covered with gloo in test_multi_gloo.py; this
run has one GPU.)"""
import numpy as np
import pytest

import paper_2504_15720_b200 as P
from paper_2504_15720_b200.tp import HeadShardedDecode, gpu_attend, head_slice

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

L, H, HQ, D, HID = 2, 8, 16, 128, 512
CTX = [37, 100, 16, 250, 129]


def _pool(tp, tp_rank, kv):
    cache = P.UnifiedKvCache([P.ModelSpec("big", L, H, D, 2, HQ), P.ModelSpec("small", 2, 4, D, 2, 4)], 16, tp, 128,
                             allocate_storage=True)
    for i, c in enumerate(CTX):
        assert cache.try_allocate(i + 1, 0, c)
        assert cache.try_allocate(100 + i, 1, 2 * c + 3)
    hs = head_slice(H, tp, tp_rank)
    for i, c in enumerate(CTX):  # write each request's full context through the append kernel
        b = cache.batch([(0, [i + 1])])
        for layer in range(L):
            k = kv[i][layer][:c, hs, 0].contiguous()[None]
            v = kv[i][layer][:c, hs, 1].contiguous()[None]
            b.append([k], [v], layer, n_new=c)
    return cache


def test_tp2_shards_sum_to_unsharded():
    g = torch.Generator(device="cuda").manual_seed(3)
    kv = [[(torch.randn((c, H, 2, D), generator=g, device="cuda") * 0.5).half() for _ in range(L)] for c in CTX]
    q = torch.randn((len(CTX), HQ, D), generator=g, device="cuda").half()
    w_o = torch.randn((HQ * D, HID), generator=g, device="cuda") / 32
    full = _pool(1, 0, kv)
    shards = [_pool(2, r, kv) for r in range(2)]
    for r in range(2):
        assert all(np.array_equal(shards[r].block_table_np(i + 1), full.block_table_np(i + 1)) for i in range(len(CTX)))
    ids = [i + 1 for i in range(len(CTX))]
    fb = full.batch([(0, ids)])
    ref_step = HeadShardedDecode(w_o, HQ, D, 1, 0, attend=gpu_attend(fb, 0, 1))
    for layer in range(L):
        y_full = ref_step(q, layer)
        y = torch.zeros_like(y_full)
        for r in range(2):
            sb = shards[r].batch([(0, ids)])
            step = HeadShardedDecode(w_o, HQ, D, 2, r, attend=gpu_attend(sb, 0, 1))
            y += step.partial(q[:, step.q_heads].contiguous(), layer)  # AllReduce(sum) over the TP group
        torch.cuda.synchronize()
        assert (y - y_full).abs().max().item() <= 1e-3 * max(1.0, y_full.abs().max().item())


@pytest.mark.parametrize("tp", [2, 4])
def test_tp_shards_reduced_vs_fp32_oracle(tp):
    """The head-sharded path end to end against the fp32 oracle (not against the unsharded
    CUDA path): each of the tp rank-local pools (tp_size=tp) runs the CUDA decode for its heads
    and its W_o row slice; the sum over ranks (what the AllReduce computes) must match
    concat_r(oracle attention of rank r) @ W_o in fp32.  Bound: every attention element is
    within 2e-3 of the oracle (fp16 tolerance), so |dy[:, c]| <= 2e-3 * sum_i |W_o[i, c]|."""
    import oracle_py as O

    g = torch.Generator(device="cuda").manual_seed(5 + tp)
    kv = [[(torch.randn((c, H, 2, D), generator=g, device="cuda") * 0.5).half() for _ in range(L)] for c in CTX]
    q = torch.randn((len(CTX), HQ, D), generator=g, device="cuda").half()
    w_o = torch.randn((HQ * D, HID), generator=g, device="cuda") / 32
    ids = [i + 1 for i in range(len(CTX))]
    shards = [_pool(tp, r, kv) for r in range(tp)]
    bound = 2e-3 * w_o.abs().sum(0).max().item() + 1e-4
    for layer in range(L):
        y = torch.zeros((len(CTX), HID), device="cuda")
        o_ref = []
        for r in range(tp):
            sb = shards[r].batch([(0, ids)])
            step = HeadShardedDecode(w_o, HQ, D, tp, r, attend=gpu_attend(sb, 0, 1))
            ql = q[:, step.q_heads].contiguous()
            y += step.partial(ql, layer)  # AllReduce(sum) over the TP group
            c = shards[r]
            lay = c.layout(0)
            olay = O.layout(lay.merged_stride, lay.native_stride, lay.layer_stride, lay.head_stride, lay.kv_stride,
                            16, D, lay.kv_heads, lay.q_heads, lay.phys_layers, 0)
            tabs = [c.block_table_np(i) for i in ids]
            tt = np.zeros((len(ids), max(len(t) for t in tabs), 2), np.int32)
            for j, t in enumerate(tabs):
                tt[j, :len(t)] = t
            img = c.read_blocks(np.arange(c.pool_size(), dtype=np.int32))
            o_ref.append(O.decode_attention(olay, img, layer, tt, np.array(CTX, np.int64),
                                            ql.view(torch.int16).cpu().numpy().view(np.uint16), 1 / np.sqrt(D)))
        torch.cuda.synchronize()
        y_ref = np.concatenate(o_ref, axis=1).reshape(len(CTX), -1) @ w_o.cpu().numpy()
        err = float(np.abs(y.cpu().numpy() - y_ref).max())
        assert err <= bound, (err, bound)

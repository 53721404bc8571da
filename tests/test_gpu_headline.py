"""Parity of the decode code path the headline runs, at the headline's schedule branches
(VERDICT r01 "missing #3"): the fp32 oracle (oracle/attn_oracle.c) against the fused
append+decode launch over a whole batch, on the branches plan_kernel takes at config-2 and
config-4 sizes (DESIGN.md §5 "Work list"):

* no chunking (sum of (request, kv head)s >= 1.5 per warp slot = 1776 on 148 SMs) with
  0 < n_cut < sum_hkv: the last n_cut (request, kv head)s are cut into a leading piece and
  two trailing pieces merged in-kernel, the others run as one piece;
* config-4 long contexts (up to 32K tokens, MHA and GQA) with split-KV chunking.

Rows are sampled (first / last requests of every service) so the host image stays small.
"""
import numpy as np
import pytest

import oracle_py as O
import paper_2504_15720_b200 as P

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

CFG2 = [(32, 8, 32), (32, 8, 32), (40, 40, 40), (32, 32, 32)]  # (layers, kv heads, q heads)


def _pool(shapes, ctxs, phys_layers=1, dtype=P.FP16):
    models = [P.ModelSpec(f"s{i}", L, H, 128, 2, Hq) for i, (L, H, Hq) in enumerate(shapes)]
    merged = P.plan_merged_shape(models)
    subs = [int(merged // P.native_block_bytes(m)) for m in models]
    blocks = sum(-(-sum((c + 16) // 16 + 1 for c in cl) // s) for s, cl in zip(subs, ctxs)) + 16
    cache = P.UnifiedKvCache(models, 16, 1, blocks, dtype=dtype, phys_layers=phys_layers, allocate_storage=True)
    groups, rid, order = [(m, []) for m in range(len(shapes))], 1, []
    for r in range(max(len(c) for c in ctxs)):  # interleaved arrivals across services
        for m, cl in enumerate(ctxs):
            if r < len(cl):
                order.append((0, rid, m, cl[r]))
                groups[m][1].append(rid)
                rid += 1
    assert cache.replay(order).all()
    cache.synth_fill(77, 1.0)
    return cache, groups


def _check_sampled(cache, groups, q, outs, layer, picks, tol):
    blocks = sorted({int(b) for (m, ids), pk in zip(groups, picks) for i in pk
                     for b in cache.block_table_np(ids[i])[:, 0]})
    remap = {b: j for j, b in enumerate(blocks)}
    img = cache.read_blocks(np.array(blocks, dtype=np.int32))
    worst = 0.0
    for gi, ((m, ids), pk) in enumerate(zip(groups, picks)):
        if not pk or layer >= cache.models[m].num_layers:
            continue
        L = cache.layout(m)
        lay = O.layout(L.merged_stride, L.native_stride, L.layer_stride, L.head_stride, L.kv_stride, L.tpb,
                       L.head_dim, L.kv_heads, L.q_heads, L.phys_layers, L.dtype)
        tabs = [cache.block_table_np(ids[i]) for i in pk]
        tt = np.zeros((len(pk), max(len(t) for t in tabs), 2), np.int32)
        for j, t in enumerate(tabs):
            tt[j, :len(t), 0] = [remap[int(b)] for b in t[:, 0]]
            tt[j, :len(t), 1] = t[:, 1]
        ctx = np.array([cache.request_tokens(ids[i]) for i in pk], np.int64)
        ref = O.decode_attention(lay, img, layer, tt, ctx,
                                 q[gi][pk].contiguous().view(torch.int16).cpu().numpy().view(np.uint16),
                                 1.0 / np.sqrt(L.head_dim))
        got = outs[gi][pk].float().cpu().numpy()
        assert not np.isnan(got).any()
        worst = max(worst, float(np.abs(got - ref).max()))
    assert worst <= tol, worst
    return worst


def _qkv(groups, shapes, seed, dtype=torch.float16):
    g = torch.Generator(device="cuda").manual_seed(seed)
    q = [(torch.rand((len(ids), Hq, 128), generator=g, device="cuda") * 2 - 1).to(dtype)
         for (m, ids), (_, _, Hq) in zip(groups, shapes)]
    k = [(torch.rand((len(ids), 1, H, 128), generator=g, device="cuda") - 0.5).to(dtype)
         for (m, ids), (_, H, _) in zip(groups, shapes)]
    v = [(torch.rand((len(ids), 1, H, 128), generator=g, device="cuda") - 0.5).to(dtype)
         for (m, ids), (_, H, _) in zip(groups, shapes)]
    return q, k, v


@pytest.mark.parametrize("layer", [0, 31, 39])
def test_no_chunk_branch_cut_and_uncut_pieces(layer):
    """Config-2 shapes, 32 requests per service (sum_hkv = 2816 >= 1776, contexts ~1.1K so
    pieces are >= 64 tiles and n_cut = 2 * 1184 = 2368 < 2816): one fused launch, step +1.
    The first 448 (request, kv head)s — all of Llama-3-8B's and Mistral's first 24 requests —
    run as one piece each, the rest are cut."""
    rng = np.random.default_rng(layer)
    ctxs = [[int(x) for x in rng.integers(1030, 1200, 32)] for _ in CFG2]
    cache, groups = _pool(CFG2, ctxs)
    b = cache.batch(groups)
    assert b.grow(1) == 128
    q, k, v = _qkv(groups, CFG2, 3 + layer)
    outs = [torch.full_like(x, float("nan")) for x in q]
    b.decode(q, outs, layer, k=k, v=v)
    torch.cuda.synchronize()
    info = b.plan_info()
    assert info["sum_hkv"] == 32 * 88 and info["split_tokens"] >= 1 << 30
    assert 0 < info["n_cut"] < info["sum_hkv"], info
    # the cut (request, kv head)s are the last n_cut in batch order; sampling the first 3 and
    # last 3 requests of every service covers both kinds, within Mistral's group too
    assert 32 * 8 + 3 * 8 <= info["sum_hkv"] - info["n_cut"] <= 32 * 8 + 29 * 8
    picks = [sorted({0, 1, 2, len(ids) - 3, len(ids) - 2, len(ids) - 1}) for _, ids in groups]
    _check_sampled(cache, groups, q, outs, layer, picks, 2e-3)


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_config4_long_context_split_kv(dtype):
    """Config-4 style: skewed contexts up to 32K tokens for every service (MHA 13B / OPT
    included: their P.V rounds P to 16 bits, so this bounds that error at the longest context);
    few requests, so leading pieces are chunked across warps (split-KV) and merged in-kernel."""
    ctxs = [[32768, 1500], [20000, 64], [32768, 4095], [9000, 32768]]
    dt = P.FP16 if dtype == "fp16" else P.BF16
    cache, groups = _pool(CFG2, ctxs, dtype=dt)
    b = cache.batch(groups)
    tdt = torch.float16 if dtype == "fp16" else torch.bfloat16
    q, k, v = _qkv(groups, CFG2, 9, tdt)
    for layer in (0, 39):
        b.grow(1)
        outs = [torch.full_like(x, float("nan")) for x in q]
        b.decode(q, outs, layer, k=k, v=v)
        torch.cuda.synchronize()
        info = b.plan_info()
        assert info["split_tokens"] < 1 << 30 and info["n_cut"] > 0, info
        _check_sampled(cache, groups, q, outs, layer, [[0, 1]] * 4, 2e-3 if dtype == "fp16" else 1e-2)

"""Decode-attention and KV-append parity on the GPU against the fp32 CPU oracle
(oracle/attn_oracle.c), reading K/V through the GPU allocator's block tables.

Tolerances (north star): fp16 max-abs <= 2e-3, bf16 <= 1e-2 against fp32.
"""
import numpy as np
import pytest

import oracle_py as O
import paper_2504_15720_b200 as P

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TOL = {P.FP16: 2e-3, P.BF16: 1e-2}


def tdtype(dt):
    return torch.float16 if dt == P.FP16 else torch.bfloat16


def build_pool(shapes, ctxs, pool_blocks=None, dtype=P.FP16, phys_layers=0, seed=1234, amp=1.0):
    """shapes: [(layers, kv_heads, q_heads)], ctxs: per model list of context lengths."""
    models = [P.ModelSpec(f"s{i}", L, H, 128, 2, Hq) for i, (L, H, Hq) in enumerate(shapes)]
    need = sum(len(c) * (max(c) // 16 + 2) for c in ctxs) + 8
    cache = P.UnifiedKvCache(models, 16, 1, pool_blocks or need, dtype=dtype, phys_layers=phys_layers,
                             allocate_storage=True, max_blocks_per_request=4096)
    groups = []
    rid = 1
    order = []
    for mi, cl in enumerate(ctxs):
        ids = []
        for t in cl:
            ids.append(rid)
            order.append((rid, mi, t))
            rid += 1
        groups.append((mi, ids))
    # interleave services so merged blocks of different models alternate
    order.sort(key=lambda x: (x[0] % 3, x[0]))
    for r, mi, t in order:
        assert cache.try_allocate(r, mi, t)
    cache.synth_fill(seed, amp)
    return cache, groups


def host_image(cache):
    return cache.read_blocks(np.arange(cache.pool_size(), dtype=np.int32))


def oracle_layout(cache, m):
    L = cache.layout(m)
    return O.layout(L.merged_stride, L.native_stride, L.layer_stride, L.head_stride, L.kv_stride, L.tpb,
                    L.head_dim, L.kv_heads, L.q_heads, L.phys_layers, L.dtype)


def tables_of(cache, ids):
    tabs = [cache.block_table_np(i) for i in ids]
    width = max(1, max(len(t) for t in tabs))
    out = np.zeros((len(ids), width, 2), dtype=np.int32)
    for k, t in enumerate(tabs):
        out[k, :len(t)] = t
    return out


def run_decode_check(shapes, ctxs, layer=0, dtype=P.FP16, split=0, phys_layers=0, qamp=1.0, seed=7):
    cache, groups = build_pool(shapes, ctxs, dtype=dtype, phys_layers=phys_layers)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    qs, outs = [], []
    for (mi, ids), (L, H, Hq) in zip(groups, shapes):
        q = (torch.rand((len(ids), Hq, 128), generator=gen, device="cuda") * 2 - 1) * qamp
        qs.append(q.to(tdtype(dtype)).contiguous())
        outs.append(torch.full((len(ids), Hq, 128), float("nan"), device="cuda", dtype=tdtype(dtype)))
    b = cache.batch(groups)
    b.decode(qs, outs, layer, split_tokens=split)
    torch.cuda.synchronize()
    img = host_image(cache)
    worst = 0.0
    for (mi, ids), q, o, (L, H, Hq) in zip(groups, qs, outs, shapes):
        if layer >= L:
            continue
        ctx = np.array([ctxs[mi][k] for k in range(len(ids))], dtype=np.int64)
        ref = O.decode_attention(oracle_layout(cache, mi), img, layer, tables_of(cache, ids), ctx,
                                 q.view(torch.int16).cpu().numpy().view(np.uint16), 1.0 / np.sqrt(128.0))
        got = o.float().cpu().numpy()
        err = float(np.nanmax(np.abs(got - ref))) if got.size else 0.0
        assert not np.isnan(got).any()
        worst = max(worst, err)
    assert worst <= TOL[dtype], worst
    return worst


def test_config1_shapes_fp16():
    """7B (32L,32H) + 13B (40L,40H) sharing one pool; ctx 512 (config 1, fewer requests)."""
    run_decode_check([(32, 32, 32), (40, 40, 40)], [[512] * 3, [512] * 3], layer=5)


def test_gqa_and_mha_mixed_config2_shapes():
    """Llama-3-8B / Mistral (8 KV, 32 Q heads) + 13B + OPT in one launch (config 2 shapes)."""
    run_decode_check([(32, 8, 32), (32, 8, 32), (40, 40, 40), (32, 32, 32)],
                     [[300, 17], [1, 64], [129, 40], [255, 16]], layer=31)


def test_layers_beyond_shorter_models_are_skipped():
    run_decode_check([(4, 8, 32), (6, 4, 4)], [[33, 70], [100]], layer=5)


@pytest.mark.parametrize("ctx", [1, 15, 16, 17, 31, 32, 33, 257])
def test_ragged_context_lengths(ctx):
    run_decode_check([(2, 4, 16), (3, 2, 2)], [[ctx, ctx + 3], [ctx]], layer=1)


def test_split_kv_long_context():
    run_decode_check([(2, 8, 32), (2, 4, 4)], [[4000, 1111], [3000]], layer=1, split=512)


def test_split_kv_automatic():
    run_decode_check([(2, 2, 8)], [[5000]], layer=0)


def test_bf16():
    run_decode_check([(4, 8, 32), (4, 4, 4)], [[700, 33], [99, 1000]], layer=2, dtype=P.BF16)


def test_gqa_ratio_2_and_8():
    run_decode_check([(2, 8, 16), (2, 2, 16)], [[90, 300], [200]], layer=0)


def test_peaky_queries_stress_online_softmax():
    run_decode_check([(2, 8, 32), (2, 4, 4)], [[600], [800, 5]], layer=1, qamp=8.0)


def test_layer_sliced_pool():
    """phys_layers=2: logical layer l reads physical layer l % 2 (SURVEY Q6 run A)."""
    run_decode_check([(32, 8, 32), (40, 40, 40)], [[200], [150]], layer=37, phys_layers=2)


def test_append_then_decode_matches_oracle():
    shapes = [(3, 8, 32), (3, 4, 4)]
    ctxs = [[40, 7], [16]]
    cache, groups = build_pool(shapes, ctxs)
    b = cache.batch(groups)
    assert b.grow(1) == 3  # decode step: one new token each
    gen = torch.Generator(device="cuda").manual_seed(3)
    ks = [(torch.rand((len(ids), 1, H, 128), generator=gen, device="cuda") - 0.5).half()
          for (mi, ids), (L, H, Hq) in zip(groups, shapes)]
    vs = [(torch.rand((len(ids), 1, H, 128), generator=gen, device="cuda") - 0.5).half()
          for (mi, ids), (L, H, Hq) in zip(groups, shapes)]
    before = host_image(cache)
    b.append(ks, vs, layer=2, n_new=1)
    torch.cuda.synchronize()
    after = host_image(cache)
    # oracle: scatter into the host image of `before`
    for (mi, ids), k, v in zip(groups, ks, vs):
        pos = np.array([ctxs[mi][j] for j in range(len(ids))], dtype=np.int64)
        O.append(oracle_layout(cache, mi), before, 2, tables_of(cache, ids), pos,
                 k.view(torch.int16).cpu().numpy().view(np.uint16), v.view(torch.int16).cpu().numpy().view(np.uint16))
    assert np.array_equal(before, after)
    # and decode over the grown context sees the appended token
    qs = [torch.randn((len(ids), Hq, 128), generator=gen, device="cuda").half() for (mi, ids), (L, H, Hq) in
          zip(groups, shapes)]
    outs = [torch.empty_like(q) for q in qs]
    b.decode(qs, outs, 2)
    torch.cuda.synchronize()
    for (mi, ids), q, o in zip(groups, qs, outs):
        ctx = np.array([ctxs[mi][j] + 1 for j in range(len(ids))], dtype=np.int64)
        ref = O.decode_attention(oracle_layout(cache, mi), after, 2, tables_of(cache, ids), ctx,
                                 q.view(torch.int16).cpu().numpy().view(np.uint16), 1.0 / np.sqrt(128.0))
        assert np.abs(o.float().cpu().numpy() - ref).max() <= 2e-3


def test_synth_fill_matches_oracle_generator():
    cache, groups = build_pool([(2, 2, 2)], [[16]], seed=99, amp=1.0)
    img = host_image(cache)[:4096].view(np.float16).astype(np.float32)
    ref = np.array([O.synth_value(99, i, 1.0) for i in range(2048)], dtype=np.float32).astype(np.float16)
    assert np.array_equal(img, ref.astype(np.float32))


def test_decode_is_repeatable_and_launch_count():
    cache, groups = build_pool([(2, 8, 32), (2, 4, 4)], [[100, 200], [300]])
    b = cache.batch(groups)
    qs = [torch.randn((2, 32, 128), device="cuda").half(), torch.randn((1, 4, 128), device="cuda").half()]
    o1 = [torch.empty_like(q) for q in qs]
    o2 = [torch.empty_like(q) for q in qs]
    n0 = cache.kernel_launches()
    b.decode(qs, o1, 1)
    b.decode(qs, o2, 1)
    torch.cuda.synchronize()
    assert all(torch.equal(a, c) for a, c in zip(o1, o2))
    assert cache.kernel_launches() > n0


def test_unwritten_tail_slots_with_nan_are_ignored():
    """A recycled block still holds the previous owner's bytes (here NaN) past the new
    request's context: masked tail tokens must not leak into the output (0*NaN)."""
    cache = P.UnifiedKvCache([P.ModelSpec("a", 2, 4, 128, 2, 8)], 16, 1, 8, allocate_storage=True)
    assert cache.try_allocate(1, 0, 48)
    b1 = cache.batch([(0, [1])])
    nan = torch.full((1, 48, 4, 128), float("nan"), device="cuda").half()
    for layer in range(2):
        b1.append([nan], [nan], layer, n_new=48)
    torch.cuda.synchronize()
    del b1
    cache.free_request(1)
    assert cache.try_allocate(2, 0, 37)  # reuses blocks 0..2; tokens 37..47 keep NaN
    b2 = cache.batch([(0, [2])])
    g = torch.Generator(device="cuda").manual_seed(0)
    k = torch.randn((1, 37, 4, 128), generator=g, device="cuda").half()
    v = torch.randn((1, 37, 4, 128), generator=g, device="cuda").half()
    b2.append([k], [v], 1, n_new=37)
    q = torch.randn((1, 8, 128), generator=g, device="cuda").half()
    out = torch.empty_like(q)
    b2.decode([q], [out], 1)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    kk, vv = k[0].float(), v[0].float()  # [37, 4, 128]
    for h in range(8):
        s = (kk[:, h // 2] @ q[0, h].float()) / np.sqrt(128.0)
        ref = torch.softmax(s, 0) @ vv[:, h // 2]
        assert (out[0, h].float() - ref).abs().max().item() <= 2e-3


@pytest.mark.parametrize("split", [0, 32])
def test_fused_append_decode_equals_append_then_decode(split):
    """decode(k=, v=) appends the step's token inside the decode launch: pool bytes and
    outputs identical to append(n_new=1) followed by decode (incl. split-KV, where only
    the item holding position ctx-1 writes), and within tolerance of the oracle."""
    shapes = [(3, 8, 32), (3, 4, 4), (4, 2, 16)]
    ctxs = [[40, 7, 300], [16, 1], [129, 64]]
    res = []
    for fused in (False, True):
        cache, groups = build_pool(shapes, ctxs, seed=77)
        b = cache.batch(groups)
        assert b.grow(1) == 7
        gen = torch.Generator(device="cuda").manual_seed(5)
        ks = [(torch.rand((len(ids), 1, H, 128), generator=gen, device="cuda") - 0.5).half()
              for (mi, ids), (L, H, Hq) in zip(groups, shapes)]
        vs = [(torch.rand((len(ids), 1, H, 128), generator=gen, device="cuda") - 0.5).half()
              for (mi, ids), (L, H, Hq) in zip(groups, shapes)]
        qs = [torch.randn((len(ids), Hq, 128), generator=gen, device="cuda").half()
              for (mi, ids), (L, H, Hq) in zip(groups, shapes)]
        outs = [torch.empty_like(q) for q in qs]
        n0 = cache.kernel_launches()
        if fused:
            b.decode(qs, outs, 2, split_tokens=split, k=ks, v=vs)
        else:
            b.append(ks, vs, 2, n_new=1)
            b.decode(qs, outs, 2, split_tokens=split)
        torch.cuda.synchronize()
        res.append((host_image(cache), [o.clone() for o in outs], cache.kernel_launches() - n0, cache, groups, qs))
    (img0, out0, n_sep, _, _, _), (img1, out1, n_fused, cache, groups, qs) = res
    assert np.array_equal(img0, img1)
    assert all(torch.equal(a, c) for a, c in zip(out0, out1))
    assert n_fused == n_sep - 1
    for (mi, ids), q, o in zip(groups, qs, out1):
        ctx = np.array([ctxs[mi][j] + 1 for j in range(len(ids))], dtype=np.int64)
        ref = O.decode_attention(oracle_layout(cache, mi), img1, 2, tables_of(cache, ids), ctx,
                                 q.view(torch.int16).cpu().numpy().view(np.uint16), 1.0 / np.sqrt(128.0))
        assert np.abs(o.float().cpu().numpy() - ref).max() <= 2e-3


@pytest.mark.parametrize("split", [0, 32])
def test_back_to_back_fused_launches_match_serialised(split):
    """Layer after layer of fused append+decode launched back to back (programmatic
    dependent launch lets launch l+1 prefetch K/V while l drains; counters alternate
    between two sets) gives the same pool and outputs as the same launches each followed
    by a device synchronisation, over two decode steps, eager and as a CUDA graph."""
    shapes = [(4, 8, 32), (3, 4, 4)]
    ctxs = [[40, 300, 17], [64, 1]]

    def run(mode):
        cache, groups = build_pool(shapes, ctxs, seed=5, phys_layers=1)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        torch.cuda.set_stream(s)
        cache.set_stream(s)
        b = cache.batch(groups)
        gen = torch.Generator(device="cuda").manual_seed(11)
        outs_all = []
        graph = None
        for step in range(2):
            b.grow(1)
            cache.flush()
            ks = [[(torch.rand((len(ids), 1, H, 128), generator=gen, device="cuda") - 0.5).half()
                   for (mi, ids), (L, H, Hq) in zip(groups, shapes)] for _ in range(4)]
            vs = [[(torch.rand((len(ids), 1, H, 128), generator=gen, device="cuda") - 0.5).half()
                   for (mi, ids), (L, H, Hq) in zip(groups, shapes)] for _ in range(4)]
            qs = [[torch.randn((len(ids), Hq, 128), generator=gen, device="cuda").half()
                   for (mi, ids), (L, H, Hq) in zip(groups, shapes)] for _ in range(4)]
            outs = [[torch.empty_like(q) for q in ql] for ql in qs]
            if mode == "graph":
                b.decode(qs[0], outs[0], 0, split_tokens=split, k=ks[0], v=vs[0])  # plan outside
                torch.cuda.synchronize()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=s):
                    for layer in range(4):
                        b.decode(qs[layer], outs[layer], layer, split_tokens=split, k=ks[layer], v=vs[layer],
                                 stream=s)
                graph.replay()
            else:
                for layer in range(4):
                    b.decode(qs[layer], outs[layer], layer, split_tokens=split, k=ks[layer], v=vs[layer])
                    if mode == "sync":
                        torch.cuda.synchronize()
            torch.cuda.synchronize()
            outs_all.append([[o.clone() for o in ol] for ol in outs])
        torch.cuda.synchronize()
        torch.cuda.set_stream(torch.cuda.default_stream())
        return host_image(cache), outs_all

    img_s, out_s = run("sync")
    for mode in ("eager", "graph"):
        img, out = run(mode)
        assert np.array_equal(img, img_s), mode
        for a_step, b_step in zip(out, out_s):
            for layer, (a_l, b_l) in enumerate(zip(a_step, b_step)):
                # groups whose model has <= layer layers are skipped (output untouched)
                assert all(torch.equal(x, y) for x, y, (L, _, _) in zip(a_l, b_l, shapes) if layer < L), mode


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6, 7, 8])
def test_decode_randomised_services(seed):
    """Randomised mixes: 1-4 services with random layer counts, KV heads and GQA ratios
    (1, 2, 4, 8), 1-40 requests each with ragged contexts (1-3000 tokens, some split-KV),
    fp16 or bf16, sliced or faithful pool."""
    rng = np.random.default_rng(200 + seed)
    shapes, ctxs = [], []
    for _ in range(int(rng.integers(1, 5))):
        L = int(rng.integers(1, 5))
        H = int(rng.choice([1, 2, 4, 8]))
        G = int(rng.choice([1, 2, 4, 8]))
        shapes.append((L, H, H * G))
        ctxs.append([int(rng.integers(1, 3000)) for _ in range(int(rng.integers(1, 41)))])
    layer = int(rng.integers(0, max(L for L, _, _ in shapes)))
    dtype = P.BF16 if seed % 4 == 0 else P.FP16
    phys = 2 if seed % 3 == 0 else 0
    run_decode_check(shapes, ctxs, layer=layer, dtype=dtype, phys_layers=phys, seed=seed,
                     split=int(rng.choice([0, 0, 64])))

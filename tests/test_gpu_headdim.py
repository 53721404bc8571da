"""Services with different head dims in ONE pool and ONE launch (north star: "different
layer counts, head counts, GQA ratios and head dims"; reference head_dim is a per-model
field, cost_model.hpp:23, that scales the native block, kv_cache.hpp:17-22).

* allocator: bit-exact with the oracle (native bytes scale with d);
* append: byte-exact against the oracle scatter for d = 64, 128, 256;
* decode: one launch over d = 64 / 128 / 256 groups with GQA 1-8, ragged contexts, split-KV,
  fp16 <= 2e-3 and bf16 <= 1e-2 against the fp32 oracle;
* fused append+decode == append then decode, byte for byte.
"""
import numpy as np
import pytest

import oracle_py as O
import paper_2504_15720_b200 as P

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TOL = {P.FP16: 2e-3, P.BF16: 1e-2}
# (layers, kv heads, q heads, head dim): Llama-3.2-1B-like (d 64, GQA 4), Llama-3-8B (d 128,
# GQA 4), Llama-2-13B (d 128 MHA), Gemma-7B-like (d 256 MHA), Gemma-2-9B-like (d 256, GQA 2)
MIXED = [(16, 8, 32, 64), (32, 8, 32, 128), (40, 40, 40, 128), (28, 16, 16, 256), (42, 8, 16, 256)]


def tdt(dt):
    return torch.float16 if dt == P.FP16 else torch.bfloat16


def build(shapes, ctxs, dtype=P.FP16, phys_layers=0, seed=4242):
    models = [P.ModelSpec(f"s{i}", L, H, d, 2, Hq) for i, (L, H, Hq, d) in enumerate(shapes)]
    merged = P.plan_merged_shape(models)
    subs = [int(merged // P.native_block_bytes(m)) for m in models]
    blocks = sum(-(-sum(c // 16 + 2 for c in cl) // s) for s, cl in zip(subs, ctxs)) + 8
    cache = P.UnifiedKvCache(models, 16, 1, blocks, dtype=dtype, phys_layers=phys_layers, allocate_storage=True)
    oracle = O.OracleCache([(L, H, d, 2) for L, H, _, d in shapes], pool=blocks)
    groups, rid, ops = [(m, []) for m in range(len(shapes))], 1, []
    for r in range(max(len(c) for c in ctxs)):
        for m, cl in enumerate(ctxs):
            if r < len(cl):
                ops.append((0, rid, m, cl[r]))
                groups[m][1].append(rid)
                rid += 1
    assert cache.replay(ops).all()
    for _, r, m, t in ops:
        assert oracle.try_allocate(r, m, t)
    cache.synth_fill(seed, 1.0)
    return cache, groups, oracle


def olay(cache, m):
    L = cache.layout(m)
    return O.layout(L.merged_stride, L.native_stride, L.layer_stride, L.head_stride, L.kv_stride, L.tpb, L.head_dim,
                    L.kv_heads, L.q_heads, L.phys_layers, L.dtype)


def tables(cache, ids):
    tabs = [cache.block_table_np(i) for i in ids]
    out = np.zeros((len(ids), max(1, max(len(t) for t in tabs)), 2), np.int32)
    for k, t in enumerate(tabs):
        out[k, :len(t)] = t
    return out


def image(cache):
    return cache.read_blocks(np.arange(cache.pool_size(), dtype=np.int32))


def u16(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def decode_check(shapes, ctxs, layer, dtype=P.FP16, split=0, phys_layers=0, seed=3, fused=False):
    cache, groups, oracle = build(shapes, ctxs, dtype, phys_layers)
    for (m, ids) in groups:  # allocator: identical tables although native bytes differ by d
        for i in ids:
            assert np.array_equal(cache.block_table_np(i), oracle.block_table_np(i))
    assert cache.stats() == oracle.stats()
    b = cache.batch(groups)
    g = torch.Generator(device="cuda").manual_seed(seed)
    qs = [((torch.rand((len(ids), Hq, d), generator=g, device="cuda") * 2 - 1)).to(tdt(dtype))
          for (m, ids), (L, H, Hq, d) in zip(groups, shapes)]
    outs = [torch.full_like(q, float("nan")) for q in qs]
    kw = {}
    if fused:
        assert b.grow(1) == sum(len(c) for c in ctxs)
        kw["k"] = [(torch.rand((len(ids), 1, H, d), generator=g, device="cuda") - 0.5).to(tdt(dtype))
                   for (m, ids), (L, H, Hq, d) in zip(groups, shapes)]
        kw["v"] = [(torch.rand((len(ids), 1, H, d), generator=g, device="cuda") - 0.5).to(tdt(dtype))
                   for (m, ids), (L, H, Hq, d) in zip(groups, shapes)]
    b.decode(qs, outs, layer, split_tokens=split, **kw)
    torch.cuda.synchronize()
    img = image(cache)
    worst = 0.0
    for (m, ids), q, o, (L, H, Hq, d) in zip(groups, qs, outs, shapes):
        if layer >= L:
            continue
        ctx = np.array([cache.request_tokens(i) for i in ids], np.int64)
        ref = O.decode_attention(olay(cache, m), img, layer, tables(cache, ids), ctx, u16(q), 1.0 / np.sqrt(d))
        got = o.float().cpu().numpy()
        assert not np.isnan(got).any(), (m, d)
        worst = max(worst, float(np.abs(got - ref).max()))
    assert worst <= TOL[dtype], worst
    return cache, groups, outs, img


def test_mixed_head_dims_one_launch():
    decode_check(MIXED, [[300, 17, 1], [64, 129], [1000], [255, 16, 33], [700, 2]], layer=10)


def test_mixed_head_dims_bf16_sliced_pool():
    decode_check(MIXED, [[40, 2000], [1], [77, 500], [1200], [15, 16, 17]], layer=27, dtype=P.BF16, phys_layers=2)


@pytest.mark.parametrize("d", [64, 256])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_each_gqa_ratio_per_head_dim(d, G):
    decode_check([(2, 4, 4 * G, d), (2, 2, 2, 128)], [[1, 15, 16, 17, 250, 3000], [99]], layer=1, seed=G)


@pytest.mark.parametrize("split", [0, 64])
def test_mixed_head_dims_split_kv_long_context(split):
    """Few long requests: leading pieces chunked across warps, partial (m, l, o) merged in-kernel
    (workspace rows of d floats per head)."""
    decode_check([(2, 4, 16, 64), (2, 8, 8, 256), (2, 2, 8, 128)], [[9000], [12000, 40], [5000]], layer=1,
                 split=split)


def test_mixed_head_dims_fused_append():
    decode_check(MIXED, [[300, 17], [64, 129], [1000], [255, 16], [700, 2]], layer=3, fused=True)


def test_append_byte_exact_per_head_dim():
    shapes = [(3, 4, 8, 64), (3, 2, 2, 256), (3, 4, 4, 128)]
    ctxs = [[40, 7], [16, 33], [5]]
    cache, groups, _ = build(shapes, ctxs)
    b = cache.batch(groups)
    g = torch.Generator(device="cuda").manual_seed(9)
    n_new = 5
    ks = [(torch.rand((len(ids), n_new, H, d), generator=g, device="cuda") - 0.5).half()
          for (m, ids), (L, H, Hq, d) in zip(groups, shapes)]
    vs = [(torch.rand((len(ids), n_new, H, d), generator=g, device="cuda") - 0.5).half()
          for (m, ids), (L, H, Hq, d) in zip(groups, shapes)]
    before = image(cache)
    b.append(ks, vs, layer=2, n_new=n_new)
    torch.cuda.synchronize()
    after = image(cache)
    for (m, ids), k, v in zip(groups, ks, vs):
        pos = np.array([cache.request_tokens(i) - n_new for i in ids], np.int64)
        O.append(olay(cache, m), before, 2, tables(cache, ids), pos, u16(k), u16(v))
    assert np.array_equal(before, after)


def test_fused_equals_separate_mixed_head_dims():
    shapes = [(3, 4, 16, 64), (3, 2, 4, 256), (3, 4, 4, 128), (3, 8, 8, 256)]
    ctxs = [[40, 7, 300], [16, 1], [129], [64, 2000]]
    res = []
    for fused in (False, True):
        cache, groups, _ = build(shapes, ctxs, seed=77)
        b = cache.batch(groups)
        b.grow(1)
        g = torch.Generator(device="cuda").manual_seed(5)
        ks = [(torch.rand((len(ids), 1, H, d), generator=g, device="cuda") - 0.5).half()
              for (m, ids), (L, H, Hq, d) in zip(groups, shapes)]
        vs = [(torch.rand((len(ids), 1, H, d), generator=g, device="cuda") - 0.5).half()
              for (m, ids), (L, H, Hq, d) in zip(groups, shapes)]
        qs = [torch.randn((len(ids), Hq, d), generator=g, device="cuda").half()
              for (m, ids), (L, H, Hq, d) in zip(groups, shapes)]
        outs = [torch.empty_like(q) for q in qs]
        if fused:
            b.decode(qs, outs, 2, k=ks, v=vs)
        else:
            b.append(ks, vs, 2, n_new=1)
            b.decode(qs, outs, 2)
        torch.cuda.synchronize()
        res.append((image(cache), [o.clone() for o in outs]))
    assert np.array_equal(res[0][0], res[1][0])
    assert all(torch.equal(a, c) for a, c in zip(res[0][1], res[1][1]))


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_randomised_mixed_head_dims(seed):
    rng = np.random.default_rng(900 + seed)
    shapes, ctxs = [], []
    for _ in range(int(rng.integers(2, 6))):
        H = int(rng.choice([1, 2, 4, 8]))
        shapes.append((int(rng.integers(1, 5)), H, H * int(rng.choice([1, 2, 4, 8])), int(rng.choice([64, 128, 256]))))
        ctxs.append([int(rng.integers(1, 2500)) for _ in range(int(rng.integers(1, 20)))])
    layer = int(rng.integers(0, max(s[0] for s in shapes)))
    decode_check(shapes, ctxs, layer, dtype=P.BF16 if seed % 2 else P.FP16, seed=seed, fused=bool(seed % 3 == 0),
                 split=int(rng.choice([0, 0, 48])))


# ---------------------------------------------------------------------------- prefill ---
def prefill_check(shapes, ctxs, q_lens, layer, dtype=P.FP16, seed=11, qamp=1.0):
    """q_lens: per-request chunk lengths (batch order) or one int for all."""
    cache, groups, _ = build(shapes, ctxs, dtype)
    g = torch.Generator(device="cuda").manual_seed(seed)
    nreq = [len(ids) for _, ids in groups]
    lens = [q_lens] * sum(nreq) if isinstance(q_lens, int) else list(q_lens)
    per, k = [], 0
    for n in nreq:
        per.append(lens[k:k + n])
        k += n
    qs, outs = [], []
    for (m, ids), (L, H, Hq, d), pl in zip(groups, shapes, per):
        shape = (len(ids), q_lens, Hq, d) if isinstance(q_lens, int) else (sum(pl), Hq, d)
        qs.append(((torch.rand(shape, generator=g, device="cuda") * 2 - 1) * qamp).to(tdt(dtype)))
        outs.append(torch.full(shape, float("nan"), device="cuda", dtype=tdt(dtype)))
    b = cache.batch(groups)
    b.prefill(qs, outs, layer, q_lens)
    torch.cuda.synchronize()
    img = image(cache)
    worst = 0.0
    for (m, ids), q, o, (L, H, Hq, d), pl in zip(groups, qs, outs, shapes, per):
        if layer >= L:
            continue
        ctx = np.array([cache.request_tokens(i) for i in ids], np.int64)
        ql = np.array(pl, np.int64)
        qn = u16(q).reshape(-1, Hq, d)
        ref = O.prefill_attention(olay(cache, m), img, layer, tables(cache, ids), ctx - ql, ql, qn, 1.0 / np.sqrt(d))
        got = o.float().cpu().numpy().reshape(-1, Hq, d)
        assert not np.isnan(got).any(), d
        worst = max(worst, float(np.abs(got - ref).max()))
    assert worst <= TOL[dtype], worst
    return worst


@pytest.mark.parametrize("d", [64, 256])
@pytest.mark.parametrize("G", [1, 4])
def test_prefill_head_dim(d, G):
    prefill_check([(2, 2, 2 * G, d)], [[700, 300]], 256 if G == 1 else 64, layer=1)


def test_prefill_mixed_head_dims_one_call():
    """d = 64, 128, 256 services in one prefill call (one tcgen05 launch per head dim)."""
    prefill_check([(2, 4, 16, 64), (2, 4, 4, 128), (2, 2, 4, 256), (3, 8, 8, 256)],
                  [[513, 200], [1000], [77, 1500], [300]], 33, layer=1)


@pytest.mark.parametrize("dtype", ["fp16", "bf16"])
def test_prefill_per_request_q_len(dtype):
    """Ragged chunks in one launch: each request's own chunk length (1 .. 700), q/out packed
    by request within each group (the config-3 last-chunk case without a launch per length)."""
    shapes = [(2, 8, 32, 128), (2, 4, 4, 128), (2, 2, 4, 64), (2, 2, 2, 256)]
    ctxs = [[1000, 40, 600], [129, 700], [513, 16], [300, 301]]
    q_lens = [512, 1, 300, 129, 700, 100, 16, 1, 257]
    prefill_check(shapes, ctxs, q_lens, layer=0, dtype=P.FP16 if dtype == "fp16" else P.BF16)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_prefill_randomised_head_dims(seed):
    rng = np.random.default_rng(500 + seed)
    shapes, ctxs, lens = [], [], []
    for _ in range(int(rng.integers(1, 4))):
        H = int(rng.choice([1, 2, 4]))
        shapes.append((2, H, H * int(rng.choice([1, 2, 4, 8])), int(rng.choice([64, 128, 256]))))
        cl = [int(rng.integers(1, 1500)) for _ in range(int(rng.integers(1, 5)))]
        ctxs.append(cl)
        lens += [int(rng.integers(1, c + 1)) for c in cl]
    prefill_check(shapes, ctxs, lens, layer=1, dtype=P.BF16 if seed == 2 else P.FP16, seed=seed)


def test_append_ragged_counts_byte_exact():
    """skv_append_args.n_news: each request appends its own number of tokens in one launch
    (k / v packed by request), byte-exact against the oracle scatter."""
    shapes = [(3, 4, 8, 64), (3, 2, 2, 256), (3, 4, 4, 128)]
    ctxs = [[40, 7], [16, 33], [50]]
    cache, groups, _ = build(shapes, ctxs)
    b = cache.batch(groups)
    g = torch.Generator(device="cuda").manual_seed(19)
    counts = [17, 3, 16, 1, 50]  # batch order
    before = image(cache)
    ks, vs, k = [], [], 0
    for (m, ids), (L, H, Hq, d) in zip(groups, shapes):
        n = sum(counts[k:k + len(ids)])
        k += len(ids)
        ks.append((torch.rand((n, H, d), generator=g, device="cuda") - 0.5).half())
        vs.append((torch.rand((n, H, d), generator=g, device="cuda") - 0.5).half())
    b.append(ks, vs, 1, counts)
    torch.cuda.synchronize()
    after = image(cache)
    k = 0
    for (m, ids), kk, vv in zip(groups, ks, vs):
        off = 0
        for i in ids:
            n = counts[k]
            k += 1
            pos = np.array([cache.request_tokens(i) - n], np.int64)
            O.append(olay(cache, m), before, 1, tables(cache, [i]), pos, u16(kk[off:off + n][None]),
                     u16(vv[off:off + n][None]))
            off += n
    assert np.array_equal(before, after)


def test_prefill_long_context_bf16_gqa():
    """A 64-token chunk at 16K / 9K context (ping-pong items walking ~130 K/V tiles), bf16."""
    prefill_check([(1, 2, 8, 128)], [[16384, 9000]], 64, layer=0, dtype=P.BF16)


def test_prefill_peaky_ragged_rescale_path():
    """Large-magnitude q (the running max jumps inside tiles: O, l and already stored P chunks are
    rescaled) with ragged chunk lengths crossing ping-pong item boundaries."""
    prefill_check([(2, 2, 8, 128), (2, 4, 4, 128)], [[900, 300], [1500]], [300, 77, 640], layer=1, qamp=6.0)

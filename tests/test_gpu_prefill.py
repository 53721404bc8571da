"""Chunked-prefill attention (tcgen05 tensor cores) vs the fp32 CPU oracle.

Each request's last q_len tokens attend causally to every key at or before their
own position (keys already appended to the pool).  fp16 max-abs <= 2e-3 (bf16
<= 1e-2) against oracle/attn_oracle.c:skvo_prefill_attention."""
import numpy as np
import pytest

import oracle_py as O
import paper_2504_15720_b200 as P

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from test_gpu_decode import TOL, build_pool, host_image, oracle_layout, tables_of, tdtype  # noqa: E402


def run_prefill_check(shapes, ctxs, q_len, layer=0, dtype=P.FP16, qamp=1.0, seed=11):
    cache, groups = build_pool(shapes, ctxs, dtype=dtype)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    qs, outs = [], []
    for (mi, ids), (L, H, Hq) in zip(groups, shapes):
        q = (torch.rand((len(ids), q_len, Hq, 128), generator=gen, device="cuda") * 2 - 1) * qamp
        qs.append(q.to(tdtype(dtype)).contiguous())
        outs.append(torch.full((len(ids), q_len, Hq, 128), float("nan"), device="cuda", dtype=tdtype(dtype)))
    b = cache.batch(groups)
    b.prefill(qs, outs, layer, q_len)
    torch.cuda.synchronize()
    img = host_image(cache)
    worst = 0.0
    for (mi, ids), q, o, (L, H, Hq) in zip(groups, qs, outs, shapes):
        if layer >= L:
            continue
        ctx = np.array(ctxs[mi], dtype=np.int64)
        qn = q.view(torch.int16).cpu().numpy().view(np.uint16).reshape(len(ids) * q_len, Hq, 128)
        ref = O.prefill_attention(oracle_layout(cache, mi), img, layer, tables_of(cache, ids), ctx - q_len,
                                  np.full(len(ids), q_len, np.int64), qn, 1.0 / np.sqrt(128.0))
        got = o.float().cpu().numpy().reshape(len(ids) * q_len, Hq, 128)
        assert not np.isnan(got).any()
        worst = max(worst, float(np.abs(got - ref).max()))
    assert worst <= TOL[dtype], worst
    return worst


def test_prefill_mha_first_chunk():
    """p = 0: pure causal self-attention of a 128-token chunk (one q tile, one key tile)."""
    run_prefill_check([(2, 2, 2)], [[128]], q_len=128, layer=1)


def test_prefill_mha_chunk_with_prefix():
    run_prefill_check([(2, 2, 2)], [[700]], q_len=256, layer=0)


def test_prefill_gqa_folded_rows():
    """G=4: a 128-row tile holds 32 tokens x 4 query heads sharing one KV head."""
    run_prefill_check([(2, 2, 8)], [[300, 90]], q_len=64, layer=1)


def test_prefill_ragged_and_unaligned():
    run_prefill_check([(2, 4, 4), (3, 2, 8)], [[513, 200], [77]], q_len=33, layer=0)


def test_prefill_mixed_services_config3_chunk():
    """Config-3 style: chunk C=512 for an MHA and a GQA service in one launch."""
    run_prefill_check([(2, 8, 32), (2, 4, 4)], [[1500], [1024, 600]], q_len=512, layer=1)


def test_prefill_bf16():
    run_prefill_check([(2, 2, 4)], [[400]], q_len=160, layer=0, dtype=P.BF16)


def test_prefill_peaky():
    run_prefill_check([(2, 2, 2)], [[300]], q_len=100, layer=0, qamp=6.0)


def test_prefill_single_token_equals_decode():
    """q_len = 1 is a decode step: both kernels agree with each other."""
    shapes = [(2, 4, 16)]
    cache, groups = build_pool(shapes, [[257, 31]])
    q = torch.randn((2, 1, 16, 128), device="cuda").half()
    o1 = torch.empty_like(q)
    o2 = torch.empty((2, 16, 128), device="cuda").half()
    b = cache.batch(groups)
    b.prefill([q], [o1], 1, 1)
    b.decode([q.view(2, 16, 128)], [o2], 1)
    torch.cuda.synchronize()
    assert (o1.view(2, 16, 128).float() - o2.float()).abs().max().item() <= 2e-3


def test_prefill_gqa8_llama70b_ratio():
    """G=8 (Llama-2/3-70B real GQA): 16 tokens x 8 heads per 128-row tile."""
    run_prefill_check([(2, 2, 16)], [[333, 64]], q_len=48, layer=1)


def test_prefill_long_prefix_many_tiles():
    run_prefill_check([(2, 2, 2)], [[4100]], q_len=300, layer=0)


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6])
def test_prefill_randomised_services(seed):
    """Randomised mixes: 1-3 services with random layer counts, KV heads and GQA ratios
    (1, 2, 4, 8), ragged contexts, a random chunk length (1-300), fp16 or bf16."""
    rng = np.random.default_rng(100 + seed)
    n_svc = int(rng.integers(1, 4))
    q_len = int(rng.choice([1, 7, 64, 100, 129, 256, 300]))
    shapes, ctxs = [], []
    for _ in range(n_svc):
        L = int(rng.integers(1, 4))
        H = int(rng.choice([1, 2, 4]))
        G = int(rng.choice([1, 2, 4, 8]))
        shapes.append((L, H, H * G))
        ctxs.append([int(q_len + rng.integers(0, 900)) for _ in range(int(rng.integers(1, 4)))])
    layer = int(rng.integers(0, min(L for L, _, _ in shapes)))
    dtype = P.BF16 if seed % 3 == 0 else P.FP16
    run_prefill_check(shapes, ctxs, q_len=q_len, layer=layer, dtype=dtype, seed=seed)


@pytest.mark.parametrize("q_len,G", [(129, 1), (385, 1), (513, 1), (200, 2), (97, 8)])
def test_prefill_pingpong_partial_items(q_len, G):
    """Ping-pong kernel items are four 128-row query tiles (A: rows 0-255, B: 256-511 of the
    item); chunks ending inside A or B leave whole tiles of tail rows (masked, never stored)."""
    run_prefill_check([(2, 2, 2 * G)], [[q_len + 700, q_len + 33]], q_len=q_len, layer=1)


def test_prefill_one_tile_kernel_still_matches(tmp_path):
    """SKV_PREFILL_PP=0 selects the one-query-tile-per-CTA kernel for head dim 128 (read once per
    process): run a few of this module's checks in a fresh interpreter with it set."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, SKV_PREFILL_PP="0")
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", os.path.join(here, "test_gpu_prefill.py"),
                        "-k", "gqa_folded or ragged or randomised_services or peaky or bf16"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]

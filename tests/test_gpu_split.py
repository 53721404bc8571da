"""Split scheme on the GPU (reference SplitCacheCounter,
kv_cache.hpp:277-348): accounting identical to the oracle / reference
compare_schemes on seeded op streams; decode through per-(request, layer, head)
tables matches the fp32 numpy twin and is bit-identical to the merged pool holding
the same K/V."""
import numpy as np
import pytest

import oracle_py as O
import paper_2504_15720_b200 as P

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

D = 128


def _models(shapes):
    return [P.ModelSpec(f"s{i}", L, H, D, 2, Hq) for i, (L, H, Hq) in enumerate(shapes)]


def _ops(rng, M, n, max_tok=700):
    live, ops, nxt = {}, [], 1
    for _ in range(n):
        if live and rng.random() < 0.2:
            rid = int(rng.choice(list(live)))
            ops.append((1, rid, 0, 0))
            del live[rid]
        elif live and rng.random() < 0.5:
            rid = int(rng.choice(list(live)))
            m, t = live[rid]
            t += int(rng.integers(1, 40))
            live[rid] = (m, t)
            ops.append((0, rid, m, t))
        else:
            m = int(rng.integers(0, M))
            t = int(rng.integers(0, max_tok))
            live[nxt] = (m, t)
            ops.append((0, nxt, m, t))
            nxt += 1
    return ops


@pytest.mark.parametrize("seed", [1, 2])
def test_split_accounting_matches_compare_schemes(seed):
    shapes = [(4, 4, 8), (6, 2, 2), (3, 8, 8)]
    ops = _ops(np.random.default_rng(seed), len(shapes), 400)
    sp = P.SplitKvCache(_models(shapes), 16, 1, 1 << 16, max_requests=512, max_blocks_per_request=64)
    for kind, rid, m, t in ops:
        if kind == 0:
            assert sp.grow([rid], [m], [t]).all()
        else:
            sp.free([rid])
    got = sp.stats()
    models = [(L, H, D, 2) for L, H, _ in shapes]
    libs = ["oracle"] + (["ref"] if O.ref_available() else [])
    for lib in libs:
        _, split = O.compare_schemes(models, ops, pool=1 << 16, lib=lib)
        assert got["block_table_entries"] == split["block_table_entries"], lib
        assert got["native_reads_writes"] == split["native_reads_writes"], lib
        assert got["internal_fragmentation_bytes"] == split["internal_fragmentation_bytes"], lib
    # every live request's split ids are distinct blocks
    torch.cuda.synchronize()
    live = {}
    for kind, rid, m, t in ops:
        if kind == 0:
            live[rid] = (m, t)
        else:
            live.pop(rid, None)
    seen = set()
    for rid, (m, t) in live.items():
        L, H, _ = shapes[m]
        for layer in range(L):
            for h in range(H):
                ids = sp.block_ids(rid, layer, h)
                assert len(ids) == (t + 15) // 16
                seen.update(ids.tolist())
    used = sum(((t + 15) // 16) * shapes[m][0] * shapes[m][1] for m, t in live.values())
    assert len(seen) == used == sp.pool_size() - sp.free_blocks()


def test_split_pool_exhaustion_is_all_or_nothing():
    sp = P.SplitKvCache(_models([(2, 2, 2)]), 16, 1, 9, max_requests=8, max_blocks_per_request=8)
    assert sp.grow([1], [0], [32]).all()  # 2 native blocks x 2 layers x 2 heads = 8 split blocks
    assert not sp.grow([2], [0], [1]).any()  # needs 4 more
    assert sp.free_blocks() == 1 and sp.table_entries() == 8
    sp.free([1])
    assert sp.free_blocks() == 9


def _fill(split, merged, groups, shapes, ctxs, gen):
    """Write identical K/V of every request's full context into both pools (append)."""
    for (m, ids), (L, H, _), cl in zip(groups, shapes, ctxs):
        for rid, c in zip(ids, cl):
            for layer in range(L):
                k = (torch.randn((1, c, H, D), generator=gen, device="cuda") * 0.5).half()
                v = (torch.randn((1, c, H, D), generator=gen, device="cuda") * 0.5).half()
                split.batch([(m, [rid])]).append([k], [v], layer, n_new=c)
                merged.batch([(m, [rid])]).append([k], [v], layer, n_new=c)


def test_split_decode_matches_merged_and_twin():
    shapes = [(3, 8, 32), (2, 4, 4)]
    ctxs = [[40, 300, 17], [129, 1]]
    models = _models(shapes)
    sp = P.SplitKvCache(models, 16, 1, 4096, max_requests=64, max_blocks_per_request=64)
    mg = P.UnifiedKvCache(models, 16, 1, 64, allocate_storage=True, max_blocks_per_request=64)
    groups, rid = [], 1
    for m, cl in enumerate(ctxs):
        ids = []
        for c in cl:
            assert sp.grow([rid], [m], [c]).all()
            assert mg.try_allocate(rid, m, c)
            ids.append(rid)
            rid += 1
        groups.append((m, ids))
    sp.synth_fill(5)  # unwritten bytes are garbage; every attended token is written below
    gen = torch.Generator(device="cuda").manual_seed(9)
    _fill(sp, mg, groups, shapes, ctxs, gen)
    qs = [torch.randn((len(ids), Hq, D), generator=gen, device="cuda").half() for (_, ids), (_, _, Hq) in
          zip(groups, shapes)]
    for layer in range(3):
        o_sp = [torch.full_like(q, float("nan")) for q in qs]
        o_mg = [torch.full_like(q, float("nan")) for q in qs]
        sp.batch(groups).decode(qs, o_sp, layer)
        mg.batch(groups).decode(qs, o_mg, layer)
        torch.cuda.synchronize()
        for (m, ids), a, b, q, (L, H, Hq) in zip(groups, o_sp, o_mg, qs, shapes):
            if layer >= L:
                continue
            assert torch.equal(a, b)  # same kernel, same K/V, same work split
            G = Hq // H
            for i, rid in enumerate(ids):  # fp32 twin from the split blocks themselves
                c = sp.request_tokens(rid)
                for h in range(H):
                    blocks = sp.read_blocks(sp.block_ids(rid, layer, h)).view(np.float16).reshape(-1, 2, 16, D)
                    kk = blocks[:, 0].reshape(-1, D)[:c].astype(np.float32)
                    vv = blocks[:, 1].reshape(-1, D)[:c].astype(np.float32)
                    for g in range(G):
                        qq = q[i, h * G + g].float().cpu().numpy()
                        s = kk @ qq / np.sqrt(D)
                        p = np.exp(s - s.max())
                        ref = (p / p.sum()) @ vv
                        assert np.abs(a[i, h * G + g].float().cpu().numpy() - ref).max() <= 2e-3


def test_split_fused_append_decode_and_grow():
    shapes = [(2, 4, 16)]
    sp = P.SplitKvCache(_models(shapes), 16, 1, 1024, max_requests=16, max_blocks_per_request=32)
    assert sp.grow([1, 2], [0, 0], [16, 33]).all()
    sp.synth_fill(3)
    b = sp.batch([(0, [1, 2])])
    assert b.grow(1) == 2  # crosses a block boundary for request 1: 2 layers x 4 heads new blocks
    assert sp.table_entries() == (2 + 3) * 2 * 4
    g = torch.Generator(device="cuda").manual_seed(1)
    k = torch.randn((2, 1, 4, D), generator=g, device="cuda").half()
    v = torch.randn((2, 1, 4, D), generator=g, device="cuda").half()
    q = torch.randn((2, 16, D), generator=g, device="cuda").half()
    out = torch.empty_like(q)
    b.decode([q], [out], 1, k=[k], v=[v])
    torch.cuda.synchronize()
    for i, rid in enumerate([1, 2]):
        c = sp.request_tokens(rid)
        for h in range(4):
            ids = sp.block_ids(rid, 1, h)
            blk = sp.read_blocks(ids[-1:]).view(np.float16).reshape(2, 16, D)
            pos = (c - 1) % 16
            assert np.array_equal(blk[0, pos], k[i, 0, h].cpu().numpy())
            assert np.array_equal(blk[1, pos], v[i, 0, h].cpu().numpy())


def test_split_tp2_tables_hold_rank_heads_and_stats_follow_reference():
    """tp=2: each rank's split tables hold L x H/tp rows per native block; the accounting
    (SplitCacheCounter) counts L x num_heads entries as the reference does (it has no tp)."""
    shapes = [(3, 8, 16), (2, 4, 4)]
    sp = P.SplitKvCache(_models(shapes), 16, 2, 4096, max_requests=16, max_blocks_per_request=16)
    ops = [(0, 1, 0, 40), (0, 2, 1, 17), (0, 1, 0, 70), (1, 2, 0, 0), (0, 3, 1, 5)]
    for kind, rid, m, t in ops:
        if kind == 0:
            assert sp.grow([rid], [m], [t]).all()
        else:
            sp.free([rid])
    _, split = O.compare_schemes([(L, H, D, 2) for L, H, _ in shapes], ops, pool=4096)
    assert sp.stats()["block_table_entries"] == split["block_table_entries"]
    assert sp.stats()["native_reads_writes"] == split["native_reads_writes"]
    used = 5 * 3 * (8 // 2) + 1 * 2 * (4 // 2)  # request 1: 5 blocks x 3 layers x 4 heads/rank
    assert sp.pool_size() - sp.free_blocks() == used
    assert len(sp.block_ids(1, 2, 3)) == 5
    with pytest.raises(P.ArgError):
        sp.block_ids(1, 0, 4)  # only H/tp = 4 kv heads on this rank

"""Robustness of the data path and the drop-in boundary on the GPU:

* request-table growth: the reference has no limit on live requests or on a request's
  length below the pool size (kv_cache.hpp:104-123, simulation.hpp:248), so the device table
  grows on demand and the block assignments stay bit-exact with the oracle;
* can_grow_to with a negative token count mirrors the reference's size_t wrap (:93-98);
* argument validation: wrong shape / dtype / device / contiguity raise ArgError before any
  launch (the C-ABI takes raw pointers);
* two pools used concurrently from two threads (kv_cache.hpp:45: single-threaded per
  instance, many instances) give the oracle's answers.
"""
import threading

import numpy as np
import pytest

import oracle_py as O
import paper_2504_15720_b200 as P

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _models(shapes, d=128):
    return [P.ModelSpec(f"s{i}", L, H, d, 2, Hq) for i, (L, H, Hq) in enumerate(shapes)]


def test_request_table_grows_past_initial_capacity():
    shapes = [(4, 4, 4), (2, 2, 2)]
    c = P.UnifiedKvCache(_models(shapes), 16, 1, 512, max_requests=2, max_blocks_per_request=2)
    o = O.OracleCache([(L, H, 128, 2) for L, H, _ in shapes], pool=512)
    rng = np.random.default_rng(5)
    live = []
    for rid in range(1, 41):  # 40 live requests (initial capacity 2), lengths up to 40 blocks
        m = rid % 2
        t = int(rng.integers(1, 640))
        assert c.try_allocate(rid, m, t) == o.try_allocate(rid, m, t)
        live.append(rid)
        if rid % 5 == 0:
            victim = live.pop(int(rng.integers(0, len(live))))
            c.free_request(victim)
            o.free_request(victim)
    for rid in live:
        assert np.array_equal(c.block_table_np(rid), o.block_table_np(rid))
    assert c.stats() == o.stats()
    assert c.free_blocks() == o.free_blocks()


def test_can_grow_to_negative_tokens_matches_reference():
    c = P.UnifiedKvCache(_models([(4, 4, 4)]), 16, 1, 8)
    o = O.OracleCache([(4, 4, 128, 2)], pool=8)
    for t in (-1, -15, -16, -17, -30, -31, -32, -1000):
        assert c.can_grow_to(1, 0, t) == o.can_grow_to(1, 0, t), t


def _small_pool():
    shapes = [(2, 2, 4), (2, 4, 4)]
    c = P.UnifiedKvCache(_models(shapes), 16, 1, 16, allocate_storage=True)
    for rid, (m, t) in {1: (0, 40), 2: (1, 20)}.items():
        assert c.try_allocate(rid, m, t)
    return c, c.batch([(0, [1]), (1, [2])])


def test_argument_validation_raises_argerror():
    c, b = _small_pool()
    q = [torch.zeros((1, 4, 128), device="cuda", dtype=torch.float16) for _ in range(2)]
    o = [torch.empty_like(x) for x in q]
    b.decode(q, o, 0)  # well formed
    with pytest.raises(P.ArgError):  # bf16 tensor on an fp16 pool
        b.decode([q[0].bfloat16(), q[1]], o, 0)
    with pytest.raises(P.ArgError):  # wrong batch size
        b.decode([torch.zeros((2, 4, 128), device="cuda", dtype=torch.float16), q[1]], o, 0)
    with pytest.raises(P.ArgError):  # host tensor
        b.decode([q[0].cpu(), q[1]], o, 0)
    with pytest.raises(P.ArgError):  # non-contiguous
        b.decode([torch.zeros((1, 128, 4), device="cuda", dtype=torch.float16).transpose(1, 2), q[1]], o, 0)
    with pytest.raises(P.ArgError):  # wrong number of groups
        b.decode(q[:1], o[:1], 0)
    with pytest.raises(P.ArgError):  # append: wrong kv-head count
        b.append([torch.zeros((1, 1, 4, 128), device="cuda", dtype=torch.float16)] * 2,
                 [torch.zeros((1, 1, 4, 128), device="cuda", dtype=torch.float16)] * 2, 0)
    with pytest.raises(P.ArgError):  # prefill: q_len mismatch
        b.prefill([torch.zeros((1, 3, 4, 128), device="cuda", dtype=torch.float16)] * 2,
                  [torch.zeros((1, 3, 4, 128), device="cuda", dtype=torch.float16)] * 2, 0, 4)


def test_two_pools_two_threads():
    """Each thread owns one pool (different shapes) and runs allocate + decode in a loop; both
    must match the fp32 oracle."""
    errs, worst = [], []

    def worker(seed, shapes, ctxs):
        try:
            torch.cuda.set_device(0)
            models = _models(shapes)
            cache = P.UnifiedKvCache(models, 16, 1, 256, allocate_storage=True)
            s = torch.cuda.Stream()
            cache.set_stream(s)
            groups, rid = [], 1
            for m, cl in enumerate(ctxs):
                ids = []
                for t in cl:
                    assert cache.try_allocate(rid, m, t)
                    ids.append(rid)
                    rid += 1
                groups.append((m, ids))
            cache.synth_fill(seed, 1.0, s)
            b = cache.batch(groups)
            g = torch.Generator(device="cuda").manual_seed(seed)
            with torch.cuda.stream(s):
                qs = [(torch.rand((len(ids), shapes[m][2], 128), generator=g, device="cuda") * 2 - 1).half()
                      for m, ids in groups]
                outs = [torch.empty_like(x) for x in qs]
                for _ in range(20):
                    b.decode(qs, outs, 1, stream=s)
            s.synchronize()
            img = cache.read_blocks(np.arange(cache.pool_size(), dtype=np.int32))
            for (m, ids), q, out in zip(groups, qs, outs):
                L = cache.layout(m)
                lay = O.layout(L.merged_stride, L.native_stride, L.layer_stride, L.head_stride, L.kv_stride, 16,
                               128, L.kv_heads, L.q_heads, L.phys_layers, 0)
                tabs = [cache.block_table_np(i) for i in ids]
                w = max(len(t) for t in tabs)
                tt = np.zeros((len(ids), w, 2), np.int32)
                for k, t in enumerate(tabs):
                    tt[k, :len(t)] = t
                ref = O.decode_attention(lay, img, 1, tt, np.array(ctxs[m], np.int64),
                                         q.view(torch.int16).cpu().numpy().view(np.uint16), 1 / np.sqrt(128.0))
                worst.append(float(np.abs(out.float().cpu().numpy() - ref).max()))
        except Exception as e:  # noqa: BLE001 - reported by the main thread
            errs.append(repr(e))

    ts = [threading.Thread(target=worker, args=(11, [(4, 8, 32), (2, 4, 4)], [[700, 33, 5], [129, 400]])),
          threading.Thread(target=worker, args=(12, [(3, 2, 16), (2, 8, 8)], [[64, 1000], [17, 250, 3]]))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    assert len(worst) == 4 and max(worst) <= 2e-3, worst

"""Config-3 churn on the GPU: bursty arrivals, chunked prefill, decode, frees and
preemptions through the engine loop; the recorded KvOp stream replayed through the
oracle must give bit-identical block tables and CacheStats."""
import numpy as np
import pytest

import oracle_py as O
import paper_2504_15720_b200 as P
from paper_2504_15720_b200.churn import ChurnEngine, ServiceProfile, generate_trace

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_generate_trace_is_deterministic_and_skewed():
    prof = [ServiceProfile(f"s{i}", i % 2, 50, 10, 20, 5) for i in range(4)]
    a = generate_trace(prof, rate=20.0, duration=5.0, skewness=4, seed=3)
    b = generate_trace(prof, rate=20.0, duration=5.0, skewness=4, seed=3)
    assert [(x.t, x.svc, x.in_len, x.out_len) for x in a] == [(x.t, x.svc, x.in_len, x.out_len) for x in b]
    assert all(a[i].svc == (i // 4) % 4 for i in range(len(a)))  # runs of `skewness` per service
    c = generate_trace(prof, rate=20.0, duration=5.0, skewness=4, seed=3, step_time=2.5, step_factor=3.0)
    early = sum(x.t < 2.5 for x in c)
    assert len(c) - early > early  # bursty: the rate triples after the step


def test_churn_engine_block_tables_bit_exact_vs_oracle():
    shapes = [(2, 4, 16), (3, 8, 8)]  # (layers, kv heads, q heads); GQA 4 and MHA
    models = [P.ModelSpec(f"m{i}", L, H, 128, 2, Hq) for i, (L, H, Hq) in enumerate(shapes)]
    pool = 48
    cache = P.UnifiedKvCache(models, 16, 1, pool, allocate_storage=True, max_blocks_per_request=512)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    cache.set_stream(s)
    cache.synth_fill(5, 1.0, s)
    prof = [ServiceProfile("chat0", 0, 60, 30, 25, 10), ServiceProfile("summ0", 0, 400, 100, 6, 2),
            ServiceProfile("chat1", 1, 50, 20, 30, 10), ServiceProfile("summ1", 1, 300, 80, 5, 2)]
    trace = generate_trace(prof, rate=40.0, duration=3.0, skewness=2, seed=11, step_time=1.5, step_factor=2.0)
    eng = ChurnEngine(cache, shapes, prof, chunk=64, occupancy=0.7, max_decode=64, max_prefill=4, stream=s)
    dt, t, k = 0.05, 0.0, 0
    oracle = O.OracleCache([(L, H, 128, 2) for L, H, _ in shapes], pool=pool)
    n_checked = 0
    for it in range(80):
        t += dt
        new = []
        while k < len(trace) and trace[k].t <= t:
            new.append(trace[k])
            k += 1
        eng.add_arrivals(new)
        start = len(eng.ops)
        eng.step()
        for kind, rid, m, tok in eng.ops[start:]:  # replay this iteration's ops
            if kind == 0:
                oracle.try_allocate(rid, m, tok)
            else:
                oracle.free_request(rid)
        if it % 10 == 9:
            for rid in eng.running:
                assert np.array_equal(cache.block_table_np(rid), oracle.block_table_np(rid))
                n_checked += 1
            assert cache.stats() == oracle.stats()
            assert cache.free_blocks() == oracle.free_blocks()
    summ = eng.summary()
    assert summ["finished"] > 5 and summ["grow_ops"] > 100 and n_checked > 10
    assert cache.fragmentation_bytes() == oracle.fragmentation_bytes()
    for o in eng.o_dec:
        assert torch.isfinite(o[:4]).all()


@pytest.mark.gpu
def test_churn_warm_start_reaches_target_and_replays_bit_exact():
    """warm_start (config-3 steady state): pool brought near the occupancy target with
    prefilled requests, then serving iterations; the whole recorded op stream replays through
    the oracle to identical tables."""
    shapes = [(2, 4, 16), (3, 8, 8)]
    models = [P.ModelSpec(f"m{i}", L, H, 128, 2, Hq) for i, (L, H, Hq) in enumerate(shapes)]
    pool = 64
    cache = P.UnifiedKvCache(models, 16, 1, pool, allocate_storage=True, max_blocks_per_request=512)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    cache.set_stream(s)
    cache.synth_fill(6, 1.0, s)
    prof = [ServiceProfile("chat0", 0, 60, 30, 25, 10), ServiceProfile("summ0", 0, 400, 100, 6, 2),
            ServiceProfile("chat1", 1, 50, 20, 30, 10), ServiceProfile("summ1", 1, 300, 80, 5, 2)]
    trace = generate_trace(prof, rate=40.0, duration=3.0, skewness=2, seed=12, step_time=1.5, step_factor=2.0)
    eng = ChurnEngine(cache, shapes, prof, chunk=64, occupancy=0.7, max_decode=64, max_prefill=4, stream=s)
    k = eng.warm_start(trace)
    assert k > 0 and 0.6 * pool <= cache.allocated_blocks() <= 0.7 * pool + 1
    eng.reset_stats()
    t = 0.0
    for _ in range(30):
        t += 0.05
        new = []
        while k < len(trace) and trace[k].t <= t:
            new.append(trace[k])
            k += 1
        eng.add_arrivals(new)
        eng.step()
    assert eng.summary()["mean_occupancy"] > 0.4
    oracle = O.OracleCache([(L, H, 128, 2) for L, H, _ in shapes], pool=pool)
    for kind, rid, m, tok in eng.ops:
        if kind == 0:
            oracle.try_allocate(rid, m, tok)
        else:
            oracle.free_request(rid)
    for rid in eng.running:
        assert np.array_equal(cache.block_table_np(rid), oracle.block_table_np(rid))
    assert cache.stats() == oracle.stats()


def test_churn_preemption_reprefill_replays_bit_exact():
    """Pool sized so decode growth runs into CacheFull: victims are freed,
    re-queued and re-prefilled from token 0 (simulation.hpp:144-157,333-340); every prefill
    chunk of an iteration runs as one ragged launch per layer.  The whole recorded op stream
    replays through the oracle bit-exact, and a decode over the final running set (including
    re-prefilled requests) matches the fp32 oracle."""
    shapes = [(2, 4, 16), (3, 8, 8)]
    models = [P.ModelSpec(f"m{i}", L, H, 128, 2, Hq) for i, (L, H, Hq) in enumerate(shapes)]
    pool = 40
    cache = P.UnifiedKvCache(models, 16, 1, pool, allocate_storage=True)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    cache.set_stream(s)
    cache.synth_fill(8, 1.0, s)
    prof = [ServiceProfile("chat0", 0, 60, 30, 150, 20), ServiceProfile("summ0", 0, 300, 50, 40, 10),
            ServiceProfile("chat1", 1, 50, 20, 150, 20), ServiceProfile("summ1", 1, 200, 40, 40, 10)]
    trace = generate_trace(prof, rate=20.0, duration=30.0, skewness=2, seed=21)
    eng = ChurnEngine(cache, shapes, prof, chunk=48, occupancy=0.95, max_decode=64, max_prefill=4, stream=s)
    t, k = 0.0, 0
    for _ in range(600):  # until preemptions, re-prefills and completions have all happened
        t += 0.04
        new = []
        while k < len(trace) and trace[k].t <= t:
            new.append(trace[k])
            k += 1
        eng.add_arrivals(new)
        eng.step()
        st = eng.stats
        if st["preemptions"] > 0 and st["reprefilled"] > 0 and st["finished"] > 5:
            break
    summ = eng.summary()
    assert summ["preemptions"] > 0 and summ["reprefilled"] > 0, summ
    assert summ["finished"] > 5
    oracle = O.OracleCache([(L, H, 128, 2) for L, H, _ in shapes], pool=pool)
    for kind, rid, m, tok in eng.ops:
        if kind == 0:
            oracle.try_allocate(rid, m, tok)
        else:
            oracle.free_request(rid)
    for rid in eng.running:
        assert np.array_equal(cache.block_table_np(rid), oracle.block_table_np(rid))
    assert cache.stats() == oracle.stats() and cache.free_blocks() == oracle.free_blocks()
    # decode over every running request (current contexts) against the oracle
    groups = [(m, [r.rid for r in eng.running.values() if r.model == m and cache.request_tokens(r.rid) > 0])
              for m in range(2)]
    groups = [g for g in groups if g[1]]
    b = cache.batch(groups)
    g = torch.Generator(device="cuda").manual_seed(2)
    qs = [torch.rand((len(ids), shapes[m][2], 128), generator=g, device="cuda").half() for m, ids in groups]
    outs = [torch.empty_like(q) for q in qs]
    b.decode(qs, outs, 1)
    torch.cuda.synchronize()
    img = cache.read_blocks(np.arange(pool, dtype=np.int32))
    for (m, ids), q, o in zip(groups, qs, outs):
        lay = cache.layout(m)
        olay = O.layout(lay.merged_stride, lay.native_stride, lay.layer_stride, lay.head_stride, lay.kv_stride, 16,
                        128, lay.kv_heads, lay.q_heads, lay.phys_layers, 0)
        tabs = [cache.block_table_np(i) for i in ids]
        tt = np.zeros((len(ids), max(len(x) for x in tabs), 2), np.int32)
        for j, x in enumerate(tabs):
            tt[j, :len(x)] = x
        ctx = np.array([cache.request_tokens(i) for i in ids], np.int64)
        ref = O.decode_attention(olay, img, 1, tt, ctx, q.view(torch.int16).cpu().numpy().view(np.uint16),
                                 1 / np.sqrt(128.0))
        assert np.abs(o.float().cpu().numpy() - ref).max() <= 2e-3

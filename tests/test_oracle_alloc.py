"""Pins the C allocator oracle (oracle/kv_alloc_oracle.c) before anything trusts it.

1. The reference's own known-answer tests, proj/tests/kv_cache_test.cpp:26-235,
   restated case by case against the oracle (same inputs, same expectations).
2. The reference's seeded 100k-op property test (kv_cache_test.cpp:124-181)
   replayed op for op; the final fragmentation residual must equal the one the
   reference itself leaves (quirk Q1) — 34,839,396,352.
3. Differential replay against the UNMODIFIED reference (oracle/_ref/libref_kv.so,
   compiled from /root/reference) on seeded churn streams: every block table,
   owner_of, counter and CacheStats double must be identical.
4. The reference's test binary built from its own sources + our gtest shim.
"""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle_py as O
from _workloads import FREE, GROW, property_stream, random_stream

ref_only = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")


def model(layers, heads, head_dim=128, dtype=2):
    return (layers, heads, head_dim, dtype)


# --- 1. kv_cache_test.cpp known answers -------------------------------------------------------
def test_single_model_is_identity():  # :26-29
    assert O.plan_merged_shape([model(32, 32)]) == O.native_block_bytes(model(32, 32))


def test_same_architecture_packs_one_sub_slot():  # :31-36
    c = O.OracleCache([model(32, 32), model(32, 32)], pool=8)
    assert (c.sub_slots(0), c.sub_slots(1)) == (1, 1)


def test_seven_b_packs_into_thirteen_b():  # :38-47  (config 1 shapes)
    assert O.plan_merged_shape([model(32, 32), model(40, 40)]) == O.native_block_bytes(model(40, 40))
    assert O.plan_merged_shape([model(32, 32), model(40, 40)]) == 13107200.0
    c = O.OracleCache([model(32, 32), model(40, 40)], pool=8)
    assert (c.sub_slots(0), c.sub_slots(1)) == (1, 1)


def test_small_model_packs_many_sub_slots():  # :49-55
    c = O.OracleCache([model(2, 2), model(8, 8)], pool=8)
    assert (c.sub_slots(0), c.sub_slots(1)) == (16, 1)


def test_empty_model_list_rejected():  # :57-59
    with pytest.raises(ValueError):
        O.plan_merged_shape([])


def test_tp_must_divide_heads():  # kv_cache.hpp:18-19
    with pytest.raises(ValueError):
        O.native_block_bytes(model(32, 30), tp=4)


def test_zero_tokens_is_no_change():  # :61-66
    c = O.OracleCache([model(4, 4)], pool=4)
    assert c.try_allocate(1, 0, 0)
    assert c.free_blocks() == 4
    assert c.block_table(1) == []


def test_cache_full_signal():  # :68-74
    c = O.OracleCache([model(4, 4)], pool=2)
    assert not c.try_allocate(1, 0, 33)
    assert c.free_blocks() == 2
    assert c.registered(1)  # Q3: a failed allocation still registers the request


def test_packing_uses_one_merged_block():  # :76-85
    c = O.OracleCache([model(2, 2), model(4, 4)], pool=8)
    assert c.sub_slots(0) == 4
    assert c.try_allocate(1, 0, 48)
    assert c.allocated_blocks() == 1
    assert c.block_table(1) == [(0, 0), (0, 1), (0, 2)]


def test_grow_reuses_existing_blocks():  # :87-94
    c = O.OracleCache([model(4, 4)], pool=4)
    assert c.try_allocate(1, 0, 10)
    assert c.try_allocate(1, 0, 16)
    assert len(c.block_table(1)) == 1
    assert c.try_allocate(1, 0, 17)
    assert len(c.block_table(1)) == 2


def test_free_restores_free_list():  # :96-102
    c = O.OracleCache([model(4, 4)], pool=4)
    assert c.try_allocate(1, 0, 40)
    assert c.free_blocks() == 1
    c.free_request(1)
    assert c.free_blocks() == 4


def test_shared_merged_block_stays_allocated():  # :104-117
    c = O.OracleCache([model(2, 2), model(4, 4)], pool=2)
    assert c.try_allocate(1, 0, 8)
    assert c.try_allocate(2, 0, 8)
    assert c.allocated_blocks() == 1
    c.free_request(1)
    assert c.allocated_blocks() == 1
    c.free_request(2)
    assert c.allocated_blocks() == 0


def test_unknown_request_is_logic_error():  # :119-122
    c = O.OracleCache([model(4, 4)], pool=4)
    with pytest.raises(RuntimeError):
        c.free_request(77)


def test_model_change_is_logic_error():  # kv_cache.hpp:108
    c = O.OracleCache([model(4, 4), model(2, 2)], pool=4)
    assert c.try_allocate(1, 0, 20)
    with pytest.raises(RuntimeError):
        c.try_allocate(1, 1, 40)


def test_negative_tokens_is_validation_error():  # kv_cache.hpp:105
    c = O.OracleCache([model(4, 4)], pool=4)
    with pytest.raises(ValueError):
        c.try_allocate(1, 0, -1)


def simple_workload(requests, tokens_each):  # :183-190
    ops = [(GROW, i + 1, 0, tokens_each) for i in range(requests)]
    ops += [(FREE, i + 1, 0, 0) for i in range(requests)]
    return ops


def test_split_table_is_1024x_for_llama7b_shape():  # :192-199
    merged, split = O.compare_schemes([model(32, 32)], simple_workload(8, 100), 256)
    assert merged["block_table_entries"] > 0
    assert split["block_table_entries"] == merged["block_table_entries"] * 1024
    assert split["native_reads_writes"] == merged["native_reads_writes"] * 1024


def test_single_layer_head_ratio_is_one():  # :201-206
    merged, split = O.compare_schemes([model(1, 1)], simple_workload(1, 1), 16)
    assert split["block_table_entries"] == merged["block_table_entries"]
    assert split["native_reads_writes"] == merged["native_reads_writes"]


def test_thirteen_b_ratio_is_1600():  # :208-212
    merged, split = O.compare_schemes([model(40, 40)], simple_workload(4, 64), 256)
    assert split["block_table_entries"] == merged["block_table_entries"] * 1600


def test_merged_fragmentation_at_least_split():  # :214-226
    ops = [(GROW, 1, 0, 20), (GROW, 2, 1, 100), (GROW, 1, 0, 50), (FREE, 2, 0, 0)]
    merged, split = O.compare_schemes([model(3, 3), model(8, 8)], ops, 256)
    assert merged["internal_fragmentation_bytes"] >= split["internal_fragmentation_bytes"]
    assert merged["native_reads_writes"] <= split["native_reads_writes"]


def test_compare_schemes_pool_too_small():  # kv_cache.hpp:360-361
    with pytest.raises(ValueError):
        O.compare_schemes([model(4, 4)], simple_workload(4, 64), 2)


def test_peak_utilization_tracks_high_water():  # :228-235
    c = O.OracleCache([model(4, 4)], pool=10)
    assert c.try_allocate(1, 0, 16 * 6)
    c.free_request(1)
    assert c.try_allocate(2, 0, 16 * 2)
    assert c.stats()["peak_utilization"] == 0.6


def test_id_zero_aliases_slots_q2():  # id 0 is the "empty" sentinel
    c = O.OracleCache([model(2, 2), model(8, 8)], pool=4)
    assert c.try_allocate(0, 0, 16)
    assert c.try_allocate(1, 0, 16)
    assert c.block_table(0) == [(0, 0)] and c.block_table(1) == [(0, 0)]


# --- 2. the seeded 100k-op property test ----------------------------------------------------
Q1_RESIDUAL = 34839396352.0  # measured: reference kv_cache_test.cpp:180 residual


def _run_property(cache, check_every=1000):
    gen = property_stream(2024, 100000, 2)
    live = {}
    step = 0
    try:
        op = next(gen)
        while True:
            kind, rid, m, tok = op
            if kind == GROW:
                g = cache.try_allocate(rid, m, tok)
                if g:
                    live[rid] = (m, tok)
                op = gen.send(g)
            else:
                cache.free_request(rid)
                del live[rid]
                op = next(gen)
            if step % check_every == 0:
                assert cache.allocated_blocks() + cache.free_blocks() == 64
                expect, seen = 0, set()
                for i, (mm, t) in live.items():
                    bt = cache.block_table(i)
                    assert len(bt) == cache.native_blocks_for(t)
                    expect += len(bt)
                    for s in bt:
                        assert s not in seen, "aliased slot"
                        seen.add(s)
                        assert cache.owner_of(*s) == i
                assert cache.table_entries() == expect
            step += 1
    except StopIteration:
        pass
    for i in list(live):
        cache.free_request(i)
    return cache


@pytest.mark.slow
def test_property_random_alloc_free_reproduces_reference():
    c = _run_property(O.OracleCache([model(2, 2), model(8, 8)], pool=64))
    assert c.free_blocks() == 64
    assert c.table_entries() == 0
    # kv_cache_test.cpp:180 expects 0.0; the reference itself leaves this residual (Q1).
    assert c.fragmentation_bytes() == Q1_RESIDUAL


# --- 3. differential replay vs the unmodified reference -------------------------------------
def _state(c, ids, P):
    tables = {i: c.block_table(i) for i in ids if c.registered(i)}
    owners = [c.owner_of(b, s) for b in range(P) for s in range(4)]
    return dict(tables=tables, owners=owners, free=c.free_blocks(), alloc=c.allocated_blocks(),
                entries=c.table_entries(), frag=c.fragmentation_bytes(), stats=c.stats())


SHAPE_SETS = [
    [model(2, 2), model(8, 8)],                      # sub 16 / 1
    [model(32, 32), model(40, 40)],                  # config 1 (7B + 13B)
    [model(32, 8), model(32, 8), model(40, 40), model(32, 32)],  # config 2 (sub 6,6,1,1)
    [model(3, 3), model(8, 8), model(4, 2), model(5, 5)],        # ragged sub counts
    [model(1, 1), model(2, 1), model(4, 4), model(8, 8), model(2, 2), model(3, 1), model(6, 2), model(8, 4)],
]


@ref_only
@pytest.mark.parametrize("shapes", range(len(SHAPE_SETS)))
@pytest.mark.parametrize("seed", [1, 7, 2024])
def test_differential_vs_reference(shapes, seed):
    models = SHAPE_SETS[shapes]
    P = 48
    ops = random_stream(seed * 1000 + shapes, 4000, len(models), max_live=40, max_grow=40)
    a, b = O.OracleCache(models, pool=P), O.RefCache(models, pool=P)
    ids = sorted({op[1] for op in ops})
    for k, (kind, rid, m, tok) in enumerate(ops):
        if kind == GROW:
            assert a.try_allocate_rc(rid, m, tok) == b.try_allocate_rc(rid, m, tok)
        else:
            a.free_request(rid)
            b.free_request(rid)
        if k % 97 == 0:
            for mm in range(len(models)):
                assert a.available_slots(mm) == b.available_slots(mm)
    sa, sb = _state(a, ids, P), _state(b, ids, P)
    assert sa == sb


@ref_only
def test_replay_counts_match_reference():
    models = SHAPE_SETS[2]
    ops = random_stream(99, 20000, 4, max_live=200, max_grow=200)
    a, b = O.OracleCache(models, pool=600), O.RefCache(models, pool=600)
    assert a.replay(ops) == b.replay(ops)
    assert a.stats() == b.stats()
    assert a.fragmentation_bytes() == b.fragmentation_bytes()


@ref_only
def test_compare_schemes_matches_reference():
    ops = [(GROW, 1, 0, 20), (GROW, 2, 1, 100), (GROW, 1, 0, 50), (FREE, 2, 0, 0),
           (GROW, 3, 0, 200), (GROW, 4, 1, 33), (FREE, 1, 0, 0)]
    models = [model(3, 3), model(8, 8)]
    assert O.compare_schemes(models, ops, 256) == O.compare_schemes(models, ops, 256, lib="ref")


# --- 4. the reference's own test binary ------------------------------------------------------
@pytest.mark.skipif(not os.path.exists(O.REF_TEST_BIN), reason="reference test binary not built")
def test_reference_binary_fails_only_its_q1_assert():
    r = subprocess.run([O.REF_TEST_BIN], capture_output=True, text=True, timeout=120)
    out = r.stdout
    assert "SUMMARY passed=17 failed=1" in out, out
    fails = re.findall(r"FAILURE (\S+): (.*)", out)
    assert len(fails) == 1 and fails[0][0].endswith("kv_cache_test.cpp:180"), fails
    assert "lhs=34839396352 " in fails[0][1]

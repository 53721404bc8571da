"""Persisted formats of the churn driver (CPU): the reference trace CSV round-trips
(workload.hpp:214-265) and KvOp streams round-trip and replay identically through
the oracle and the reference."""
import os

import pytest

import oracle_py as O
from paper_2504_15720_b200.churn import (ServiceProfile, generate_trace, load_ops, load_trace, paper_services,
                                          save_ops, save_trace)


def test_trace_csv_roundtrip(tmp_path):
    prof = paper_services(2)
    tr = generate_trace(prof, rate=5.0, duration=10.0, skewness=4, seed=9)
    p = tmp_path / "trace.csv"
    save_trace(tr, prof, str(p))
    assert open(p).readline().strip() == "arrival_time,service_id,input_len,output_len"
    back = load_trace(str(p), prof)
    assert [(a.svc, a.in_len, a.out_len) for a in back] == [(a.svc, a.in_len, a.out_len) for a in tr]
    assert all(abs(a.t - b.t) < 1e-6 for a, b in zip(back, tr))


def test_trace_csv_rejects_bad_input(tmp_path):
    prof = paper_services(1)
    p = tmp_path / "bad.csv"
    p.write_text("arrival_time,service_id,input_len,output_len\n1.0,chat0,5,5\n0.5,chat0,5,5\n")
    with pytest.raises(ValueError):
        load_trace(str(p), prof)
    p.write_text("wrong\n")
    with pytest.raises(ValueError):
        load_trace(str(p), prof)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_ops_csv_roundtrip_replays_identically(tmp_path):
    from _workloads import random_stream
    ops = random_stream(5, 3000, 3, max_live=50, max_grow=50)
    p = tmp_path / "ops.csv"
    save_ops(ops, str(p))
    back = load_ops(str(p))
    assert back == [tuple(o) for o in ops]
    models = [(2, 2, 128, 2), (8, 8, 128, 2), (4, 2, 128, 2)]
    a, b = O.OracleCache(models, pool=64), O.RefCache(models, pool=64)
    assert a.replay(back) == b.replay(back)
    assert a.stats() == b.stats()

"""bench.py workloads at small sizes: each prints one JSON line with the contract's keys
(guards the benchmark paths themselves; the numbers are not checked)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "2", "--warmup", "1",
                          "--no-cpu-baseline", *args], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_decode_small():
    d = _run("--workload", "config2", "--requests", "8", "--ctx", "512", "--no-faithful", "--no-prefill")
    for key in ("metric", "value", "unit", "e2e", "roofline", "gpu_launches", "clocks", "config"):
        assert key in d, key
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] == "hbm"


def test_bench_prefill_small():
    d = _run("--workload", "prefill", "--requests", "1", "--ctx", "1024", "--chunk", "256")
    assert d["value"] > 0 and d["roofline"]["bound"] == "tensor" and d["gpu_launches"] == 2


def test_bench_gpus2_dry_run_without_torchrun():
    """`bench.py --gpus 2 --share-gpu` on a 1-GPU box: spawns 2 ranks itself, both on GPU 0
    with gloo; the line reports n_gpus 2 and the head-sharded service's AllReduce."""
    d = _run("--gpus", "2", "--share-gpu", "--workload", "config2", "--requests", "4", "--ctx", "256")
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["allreduce"]["group_size"] == 2 and d["allreduce"]["per_layer_ms_rank0"] > 0
    assert d["parity"]["ok"], d["parity"]


def test_bench_capacity_faithful_sample():
    """The default decode line also times config 2 with every layer stored (SURVEY §8d run (B),
    ~152 GB pool) and config 4 (long contexts, ~150 GB pool) after releasing the layer-sliced pool,
    and reports them under capacity_faithful and config4."""
    d = _run("--workload", "config2", "--requests", "8", "--ctx", "512", "--no-prefill")
    for key in ("config4", "config1", "config3"):
        assert "error" not in d[key] and d[key]["value"] > 0, d[key]
    assert d["config3"]["churn"]["iterations"] > 0
    cf = d["capacity_faithful"]
    assert "error" not in cf, cf
    assert cf["value"] > 0 and cf["requests"] == 152 and cf["pool_gb"] > 100
    assert cf["parity_max_abs"] is not None and cf["parity_max_abs"] <= 2e-3

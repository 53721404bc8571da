"""C-ABI checks that run without a GPU: libseakv.so loads, exports every symbol
include/seakv.h declares, and its pool-less host functions follow the reference
(kv_cache.hpp:17-33) including the ConfigError cases."""
import os
import re
import subprocess

import pytest

import paper_2504_15720_b200 as P
from paper_2504_15720_b200 import kvcache as K

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "seakv.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(skv_[a-z_]+)\s*\(", src))
    return sorted(n for n in names if not n.endswith("_t"))


def test_library_exports_every_declared_symbol():
    K.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", K.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (skv_\w+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    assert len(declared_functions()) >= 40


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", K.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out


def test_sass_uses_bulk_async_copies():
    """The decode kernel stages K/V with cp.async.bulk (SASS UBLKCP)."""
    out = subprocess.run(["cuobjdump", "-sass", K.LIB_PATH], capture_output=True, text=True).stdout
    assert "UBLKCP" in out


def test_sass_prefill_uses_tcgen05_pair_mma_and_tma():
    """The default prefill kernel issues 2-CTA tcgen05 MMAs (SASS UTCHMMA.2CTA) on operands
    staged by TMA tensor loads (UTMALDG), with multicast commits to both CTAs."""
    out = subprocess.run(["cuobjdump", "-sass", K.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA.2CTA" in out
    assert "UTMALDG.2D.2CTA" in out
    assert "UTCBAR.2CTA.MULTICAST" in out


def test_version():
    assert b"sm_100a" in K.lib().skv_version()


def m(layers, heads, q_heads=0, d=128, e=2, name="x"):
    return P.ModelSpec(name, layers, heads, d, e, q_heads)


def test_native_block_bytes_matches_reference_formula():  # kv_cache.hpp:17-22
    assert P.native_block_bytes(m(32, 32)) == 16 * 32 * 2 * 32 * 128 * 2 == 8 * 2 ** 20
    assert P.native_block_bytes(m(40, 40)) == 13107200.0
    assert P.native_block_bytes(m(32, 8, 32)) == 2 * 2 ** 20
    assert P.native_block_bytes(m(80, 64), tp_size=4) == 10 * 2 ** 20


def test_tp_must_divide_heads():  # kv_cache.hpp:18-19
    with pytest.raises(P.ConfigError):
        P.native_block_bytes(m(32, 30), tp_size=4)


def test_plan_merged_shape_is_max_native():  # kv_cache.hpp:26-33
    assert P.plan_merged_shape([m(32, 32), m(40, 40)]) == 13107200.0
    assert P.plan_merged_shape([m(32, 8, 32), m(32, 8, 32), m(40, 40), m(32, 32)]) == 13107200.0


def test_empty_model_list_rejected():  # kv_cache.hpp:28
    with pytest.raises(P.ConfigError):
        P.plan_merged_shape([])


def test_gqa_ratio_must_divide():
    with pytest.raises(P.ConfigError):
        P.native_block_bytes(m(32, 8, 12))


def test_matches_oracle_on_shapes():
    import oracle_py as O
    for shapes in ([(32, 32), (40, 40)], [(2, 2), (8, 8)], [(3, 3), (8, 8), (4, 2), (5, 5)]):
        ours = P.plan_merged_shape([m(a, b) for a, b in shapes])
        assert ours == O.plan_merged_shape([(a, b) for a, b in shapes])

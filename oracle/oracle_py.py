"""ctypes bindings to the oracle libraries — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` leg may
import this module.  It loads:

* ``oracle/_build/libskvo.so`` — the plain-C restatement of the reference
  allocator (kv_alloc_oracle.c, following kv_cache.hpp:17-369) and the fp32
  attention oracle (attn_oracle.c);
* ``oracle/_ref/libref_kv.so`` — the unmodified reference allocator compiled
  from /root/reference (ref_kv.cpp), when it was built.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SKVO_SO = os.path.join(HERE, "_build", "libskvo.so")
REF_SO = os.path.join(HERE, "_ref", "libref_kv.so")
REF_TEST_BIN = os.path.join(HERE, "_ref", "kv_cache_test_ref")

OK, FULL, ECONFIG, EVALIDATION, ELOGIC = 0, 1, -1, -2, -3


def build() -> None:
    """Compile the oracle (and oracle/_ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


class OpRec(C.Structure):
    """skvo_op / ref_op: {kind (0 grow, 1 free), model, id, tokens}."""

    _fields_ = [("kind", C.c_int32), ("model", C.c_int32), ("id", C.c_uint64), ("tokens", C.c_int64)]


def ops_array(ops):
    arr = (OpRec * max(1, len(ops)))()
    for i, (kind, rid, model, tokens) in enumerate(ops):
        arr[i].kind, arr[i].id, arr[i].model, arr[i].tokens = kind, rid, model, tokens
    return arr


class KvLayout(C.Structure):
    _fields_ = [
        ("merged_stride", C.c_int64),
        ("native_stride", C.c_int64),
        ("layer_stride", C.c_int64),
        ("head_stride", C.c_int64),
        ("kv_stride", C.c_int64),
        ("tpb", C.c_int32),
        ("head_dim", C.c_int32),
        ("kv_heads", C.c_int32),
        ("q_heads", C.c_int32),
        ("phys_layers", C.c_int32),
        ("dtype", C.c_int32),
    ]


def _ints(xs):
    return (C.c_int * max(1, len(xs)))(*xs)


def _shape_args(models):
    return (
        _ints([m[0] for m in models]),
        _ints([m[1] for m in models]),
        _ints([m[2] if len(m) > 2 else 128 for m in models]),
        _ints([m[3] if len(m) > 3 else 2 for m in models]),
    )


class _Api:
    """Shared method surface of the C oracle and the reference shim."""

    prefix = ""

    def __init__(self, lib, models, tpb=16, tp=1, pool=0):
        self.lib = lib
        self.models = list(models)
        self.tpb = tpb
        L, H, D, E = _shape_args(self.models)
        st = C.c_int(0)
        create = getattr(lib, self.prefix + "create")
        create.restype = C.c_void_p
        create.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                           C.c_size_t, C.POINTER(C.c_int)]
        self.h = create(len(self.models), L, H, D, E, tpb, tp, pool, C.byref(st))
        if not self.h:
            raise ValueError("ConfigError")
        self._f = {}

    def _fn(self, name, restype, argtypes):
        f = self._f.get(name)
        if f is None:
            f = getattr(self.lib, self.prefix + name)
            f.restype = restype
            f.argtypes = [C.c_void_p] + argtypes
            self._f[name] = f
        return f

    def close(self):
        if self.h:
            f = getattr(self.lib, self.prefix + "destroy")
            f.argtypes = [C.c_void_p]
            f(self.h)
            self.h = None

    __del__ = close

    def sub_slots(self, m):
        return self._fn("sub_slots", C.c_int, [C.c_int])(self.h, m)

    def merged_block_bytes(self):
        return self._fn("merged_block_bytes", C.c_double, [])(self.h)

    def free_blocks(self):
        return self._fn("free_blocks", C.c_size_t, [])(self.h)

    def allocated_blocks(self):
        return self._fn("allocated_blocks", C.c_size_t, [])(self.h)

    def table_entries(self):
        return self._fn("table_entries", C.c_size_t, [])(self.h)

    def available_slots(self, m):
        return self._fn("available_slots", C.c_size_t, [C.c_int])(self.h, m)

    def registered(self, rid):
        return bool(self._fn("registered", C.c_int, [C.c_uint64])(self.h, rid))

    def can_grow_to(self, rid, m, tokens):
        return bool(self._fn("can_grow_to", C.c_int, [C.c_uint64, C.c_int, C.c_long])(self.h, rid, m, tokens))

    def try_allocate_rc(self, rid, m, tokens):
        return self._fn("try_allocate", C.c_int, [C.c_uint64, C.c_int, C.c_long])(self.h, rid, m, tokens)

    def try_allocate(self, rid, m, tokens):
        rc = self.try_allocate_rc(rid, m, tokens)
        if rc == EVALIDATION:
            raise ValueError("ValidationError: negative tokens_needed")
        if rc == ELOGIC:
            raise RuntimeError("logic_error")
        return rc == OK

    def free_request(self, rid):
        rc = self._fn("free_request", C.c_int, [C.c_uint64])(self.h, rid)
        if rc:
            raise RuntimeError("logic_error: free_request: unknown request")

    def record_context_read(self, rid):
        self._fn("record_context_read", None, [C.c_uint64])(self.h, rid)

    def block_table(self, rid):
        f = self._fn("block_table", C.c_long, [C.c_uint64, C.c_void_p, C.c_size_t])
        n = f(self.h, rid, None, 0)
        if n < 0:
            raise RuntimeError("logic_error: block_table: unknown request")
        buf = np.zeros((max(n, 1), 2), dtype=np.int32)
        f(self.h, rid, buf.ctypes.data, n)
        return [tuple(map(int, r)) for r in buf[:n]]

    def block_table_np(self, rid):
        f = self._fn("block_table", C.c_long, [C.c_uint64, C.c_void_p, C.c_size_t])
        n = f(self.h, rid, None, 0)
        if n < 0:
            raise RuntimeError("logic_error: block_table: unknown request")
        buf = np.zeros((n, 2), dtype=np.int32)
        if n:
            f(self.h, rid, buf.ctypes.data, n)
        return buf

    def owner_of(self, b, s):
        return self._fn("owner_of", C.c_uint64, [C.c_int, C.c_int])(self.h, b, s)

    def fragmentation_bytes(self):
        return self._fn("fragmentation_bytes", C.c_double, [])(self.h)

    def native_blocks_for(self, tokens):
        return (tokens + self.tpb - 1) // self.tpb

    def replay(self, ops):
        return self.replay_array(ops_array(ops), len(ops))

    def replay_array(self, arr, n):
        """Replays a prebuilt ops_array (so a timing of this call excludes Python)."""
        return self._fn("replay", C.c_long, [C.c_void_p, C.c_size_t])(self.h, arr, n)


class OracleCache(_Api):
    """C restatement (oracle/kv_alloc_oracle.c) of seasim::UnifiedKvCache."""

    prefix = "skvo_"

    def __init__(self, models, tpb=16, tp=1, pool=0):
        super().__init__(_load(SKVO_SO), models, tpb, tp, pool)

    def stats(self):
        class S(C.Structure):
            _fields_ = [("e", C.c_uint64), ("rw", C.c_uint64), ("frag", C.c_double), ("util", C.c_double)]

        s = S()
        self._fn("get_stats", None, [C.c_void_p])(self.h, C.byref(s))
        return dict(block_table_entries=s.e, native_reads_writes=s.rw,
                    internal_fragmentation_bytes=s.frag, peak_utilization=s.util)

    def open_slots(self, m):
        return self._fn("open_slots", C.c_size_t, [C.c_int])(self.h, m)


class RefCache(_Api):
    """The unmodified reference allocator (oracle/_ref/libref_kv.so)."""

    prefix = "ref_kv_"

    def __init__(self, models, tpb=16, tp=1, pool=0):
        super().__init__(_load(REF_SO), models, tpb, tp, pool)

    def stats(self):
        e, rw = C.c_uint64(), C.c_uint64()
        frag, util = C.c_double(), C.c_double()
        self._fn("stats", None, [C.c_void_p] * 4)(self.h, C.byref(e), C.byref(rw), C.byref(frag), C.byref(util))
        return dict(block_table_entries=e.value, native_reads_writes=rw.value,
                    internal_fragmentation_bytes=frag.value, peak_utilization=util.value)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def plan_merged_shape(models, tpb=16, tp=1, lib="oracle"):
    so = _load(SKVO_SO if lib == "oracle" else REF_SO)
    f = getattr(so, "skvo_plan_merged_shape" if lib == "oracle" else "ref_kv_plan_merged_shape")
    f.restype = C.c_int
    L, H, D, E = _shape_args(models)
    out = C.c_double()
    rc = f(len(models), L, H, D, E, tpb, tp, C.byref(out))
    if rc:
        raise ValueError("ConfigError")
    return out.value


def native_block_bytes(model, tpb=16, tp=1):
    so = _load(SKVO_SO)
    f = so.skvo_native_block_bytes
    f.restype = C.c_int
    m = list(model) + [128, 2][len(model) - 2:]
    out = C.c_double()
    if f(m[0], m[1], m[2], m[3], tpb, tp, C.byref(out)):
        raise ValueError("ConfigError")
    return out.value


def compare_schemes(models, ops, pool, tpb=16, tp=1, lib="oracle"):
    so = _load(SKVO_SO if lib == "oracle" else REF_SO)
    f = getattr(so, "skvo_compare_schemes" if lib == "oracle" else "ref_kv_compare_schemes")
    f.restype = C.c_int
    L, H, D, E = _shape_args(models)
    arr = ops_array(ops)
    out = (C.c_double * 8)()
    rc = f(len(models), L, H, D, E, tpb, tp, arr, C.c_size_t(len(ops)), C.c_size_t(pool), out)
    if rc == EVALIDATION:
        raise ValueError("ValidationError: compare_schemes: pool too small for workload sample")
    if rc:
        raise RuntimeError(f"compare_schemes rc={rc}")
    keys = ["block_table_entries", "native_reads_writes", "internal_fragmentation_bytes", "peak_utilization"]
    merged = {k: out[i] for i, k in enumerate(keys)}
    split = {k: out[4 + i] for i, k in enumerate(keys)}
    for d in (merged, split):
        d["block_table_entries"] = int(d["block_table_entries"])
        d["native_reads_writes"] = int(d["native_reads_writes"])
    return merged, split


# ---------------------------------------------------------------- attention --
def _attn_lib():
    lib = _load(SKVO_SO)
    lib.skvo_decode_attention.restype = None
    lib.skvo_decode_attention.argtypes = [
        C.POINTER(KvLayout), C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p,
        C.c_void_p, C.c_float, C.c_void_p, C.c_void_p, C.c_int]
    lib.skvo_prefill_attention.restype = None
    lib.skvo_prefill_attention.argtypes = [
        C.POINTER(KvLayout), C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p,
        C.c_void_p, C.c_void_p, C.c_void_p, C.c_float, C.c_void_p, C.c_int]
    lib.skvo_append.restype = None
    lib.skvo_append.argtypes = [
        C.POINTER(KvLayout), C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
        C.c_void_p, C.c_void_p]
    lib.skvo_synth_value.restype = C.c_float
    lib.skvo_synth_value.argtypes = [C.c_uint64, C.c_uint64, C.c_float]
    return lib


def layout(merged_stride, native_stride, layer_stride, head_stride, kv_stride, tpb, head_dim,
           kv_heads, q_heads, phys_layers, dtype):
    return KvLayout(merged_stride, native_stride, layer_stride, head_stride, kv_stride, tpb, head_dim,
                    kv_heads, q_heads, phys_layers, dtype)


def decode_attention(lay: KvLayout, pool: np.ndarray, layer: int, tables: np.ndarray, ctx: np.ndarray,
                     q: np.ndarray, scale: float, nthreads: int = 0, want_lse: bool = False):
    """pool: uint8 host image; tables: int32 [nreq, stride, 2]; ctx: int64 [nreq];
    q: uint16 [nreq, Hq, d].  Returns fp32 out [nreq, Hq, d] (and lse)."""
    lib = _attn_lib()
    pool = np.ascontiguousarray(pool)
    tables = np.ascontiguousarray(tables, dtype=np.int32)
    ctx = np.ascontiguousarray(ctx, dtype=np.int64)
    q = np.ascontiguousarray(q, dtype=np.uint16)
    nreq = q.shape[0]
    out = np.zeros(q.shape, dtype=np.float32)
    lse = np.zeros(q.shape[:2], dtype=np.float32) if want_lse else None
    lib.skvo_decode_attention(C.byref(lay), pool.ctypes.data, layer, nreq, tables.ctypes.data,
                              tables.shape[1], ctx.ctypes.data, q.ctypes.data, scale, out.ctypes.data,
                              lse.ctypes.data if want_lse else None, nthreads)
    return (out, lse) if want_lse else out


def prefill_attention(lay: KvLayout, pool, layer, tables, q_start, q_len, q, scale, nthreads=0):
    """q: uint16 [rows, Hq, d] packed by request in order; returns fp32 [rows, Hq, d]."""
    lib = _attn_lib()
    tables = np.ascontiguousarray(tables, dtype=np.int32)
    q_start = np.ascontiguousarray(q_start, dtype=np.int64)
    q_len = np.ascontiguousarray(q_len, dtype=np.int64)
    q_off = np.concatenate([[0], np.cumsum(q_len)[:-1]]).astype(np.int64)
    q = np.ascontiguousarray(q, dtype=np.uint16)
    out = np.zeros(q.shape, dtype=np.float32)
    lib.skvo_prefill_attention(C.byref(lay), np.ascontiguousarray(pool).ctypes.data, layer, len(q_len),
                               tables.ctypes.data, tables.shape[1], q_start.ctypes.data, q_len.ctypes.data,
                               q_off.ctypes.data, q.ctypes.data, scale, out.ctypes.data, nthreads)
    return out


def append(lay: KvLayout, pool: np.ndarray, layer, tables, pos, k, v):
    """In-place scatter of k/v uint16 [nreq, n, Hkv, d] into the host pool image."""
    lib = _attn_lib()
    tables = np.ascontiguousarray(tables, dtype=np.int32)
    pos = np.ascontiguousarray(pos, dtype=np.int64)
    k = np.ascontiguousarray(k, dtype=np.uint16)
    v = np.ascontiguousarray(v, dtype=np.uint16)
    lib.skvo_append(C.byref(lay), pool.ctypes.data, layer, k.shape[0], tables.ctypes.data, tables.shape[1],
                    pos.ctypes.data, k.shape[1], k.ctypes.data, v.ctypes.data)


def synth_value(seed: int, i: int, amp: float = 1.0) -> float:
    return _attn_lib().skvo_synth_value(seed, i, amp)


# ------------------------------------------------------- reference control plane (shims) --
REF_CTL_SO = os.path.join(HERE, "_ref", "libref_ctl.so")


def ref_ctl_available() -> bool:
    return os.path.exists(REF_CTL_SO)


def ref_generate_trace(profiles, rate, duration, skewness, seed, step_time=None, step_factor=1.0):
    """The reference seasim::generate_trace (workload.hpp:181-212) through oracle/ref_ctl.cpp.
    profiles: [(in_mean, in_sd, out_mean, out_sd)]; returns [(t, svc, in_len, out_len)]."""
    lib = _load(REF_CTL_SO)
    f = lib.ref_generate_trace
    f.restype = C.c_long
    d = C.POINTER(C.c_double)
    f.argtypes = [C.c_int, d, d, d, d, C.c_double, C.c_double, C.c_int, C.c_uint64, C.c_int, C.c_double, C.c_double,
                  C.c_long, d, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
    n = len(profiles)
    cols = [np.ascontiguousarray([p[k] for p in profiles], np.float64) for k in range(4)]
    cap = int(rate * duration * max(1.0, step_factor) * 3 + 1000)
    t = np.zeros(cap, np.float64)
    svc, il, ol = (np.zeros(cap, np.int32) for _ in range(3))
    ptr = lambda a, ty: a.ctypes.data_as(C.POINTER(ty))  # noqa: E731
    m = f(n, *[ptr(x, C.c_double) for x in cols], rate, duration, skewness, seed, 0 if step_time is None else 1,
          step_time or 0.0, step_factor, cap, ptr(t, C.c_double), ptr(svc, C.c_int), ptr(il, C.c_int), ptr(ol, C.c_int))
    if m < 0:
        raise ValueError("ConfigError")
    assert m <= cap
    return [(float(t[i]), int(svc[i]), int(il[i]), int(ol[i])) for i in range(m)]


def ref_dedicated_plan(services, gpus_per_node, num_nodes, mem_gib, share_cap, replica_cap, kv_reserve_gib, batch_cap,
                       extra_models=(), min_tp_override=None, extra_entries=None):
    """The reference seasim::dedicated_plan (placement.hpp:284-319) over default_cost_model()
    plus extra models [(id, layers, heads, weight_gib, min_tp, {tp: (act_base_gib, act_per_gib)})]
    (tp in 1, 2, 4, 8 consecutively from 1), min_tp overrides {id: tp} and extra activation
    entries {id: {tp: (base, per)}}.  Returns (groups [(tp, node, gpu0, [services])], unplaced,
    feasible) or None when required_tp throws."""
    lib = _load(REF_CTL_SO)
    f = lib.ref_dedicated_plan
    f.restype = C.c_int
    cs = lambda xs: (C.c_char_p * max(1, len(xs)))(*[x.encode() for x in xs])  # noqa: E731
    ia = lambda xs: (C.c_int * max(1, len(xs)))(*xs)  # noqa: E731
    da = lambda xs: (C.c_double * max(1, len(xs)))(*xs)  # noqa: E731
    ex = list(extra_models)
    act = []
    for _, _, _, _, _, tab in ex:
        for k in range(4):
            act += list(tab.get(1 << k, (0.0, 0.0)))
    ovr = dict(min_tp_override or {})
    ent = [(mid, tp, v) for mid, d in (extra_entries or {}).items() for tp, v in d.items()]
    G = 64
    n_groups, n_unp, feas = C.c_int(), C.c_int(), C.c_int()
    g_tp, g_node, g_gpu0, g_nsvc = (np.zeros(G, np.int32) for _ in range(4))
    g_svcs = np.zeros(G * 32, np.int32)
    unplaced = np.zeros(max(1, len(services)), np.int32)
    ip = lambda a: a.ctypes.data_as(C.POINTER(C.c_int))  # noqa: E731
    rc = f(len(services), cs(services), gpus_per_node, num_nodes, C.c_double(mem_gib), share_cap, replica_cap,
           C.c_double(kv_reserve_gib), batch_cap, len(ex), cs([e[0] for e in ex]), ia([e[1] for e in ex]),
           ia([e[2] for e in ex]), da([e[3] for e in ex]), ia([e[4] for e in ex]),
           ia([max(k for k in range(4) if (1 << k) in e[5]) + 1 for e in ex]), da(act), len(ovr), cs(list(ovr)),
           ia(list(ovr.values())), len(ent), cs([e[0] for e in ent]), ia([e[1] for e in ent]),
           da([x for e in ent for x in e[2]]), C.byref(n_groups), ip(g_tp), ip(g_node), ip(g_gpu0), ip(g_nsvc),
           ip(g_svcs), C.byref(n_unp), ip(unplaced), C.byref(feas))
    if rc < 0:
        return None
    groups = [(int(g_tp[g]), int(g_node[g]), int(g_gpu0[g]), [int(x) for x in g_svcs[g * 32:g * 32 + g_nsvc[g]]])
              for g in range(n_groups.value)]
    return groups, [int(x) for x in unplaced[:n_unp.value]], bool(feas.value)

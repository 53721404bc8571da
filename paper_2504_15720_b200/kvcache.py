"""Python mirror of ``seasim::UnifiedKvCache`` over the C-ABI of libseakv.so.

Same method names, argument meaning and error behaviour as the reference
(/root/reference/proj/include/seasim/kv_cache.hpp:46-267):

* ``ConfigError``     — bad shape / tp / unknown model    (common.hpp:13-16)
* ``ValidationError`` — negative tokens, id 0 (Q2)        (common.hpp:25-28)
* ``LogicError``      — std::logic_error: unknown request, model change
* CacheFull           — ``try_allocate`` returns ``False``  (kv_cache.hpp:110-112)

Beyond the reference surface it exposes the data path: request batches,
KV append, paged decode attention, synthetic fill and pool introspection.
Every call goes to the CUDA library; there is no CPU fallback — importing
this module without a built ``libseakv.so`` raises.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import subprocess
from typing import Iterable, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SKV_LIB_PATH: an alternative build of the same library (A/B measurements, scripts/build_variant.sh)
LIB_PATH = os.environ.get("SKV_LIB_PATH") or os.path.join(_HERE, "libseakv.so")

SKV_OK, SKV_CACHE_FULL = 0, 1
SKV_ERR_CONFIG, SKV_ERR_VALIDATION, SKV_ERR_LOGIC, SKV_ERR_CUDA, SKV_ERR_ARG = -1, -2, -3, -4, -5
FP16, BF16 = 0, 1


class ConfigError(RuntimeError):
    """seasim::ConfigError"""


class ValidationError(RuntimeError):
    """seasim::ValidationError"""


class LogicError(RuntimeError):
    """std::logic_error"""


class CudaError(RuntimeError):
    """CUDA runtime failure or device-side invariant violation."""


class ArgError(ValueError):
    """Bad argument / capacity exceeded."""


_ERRS = {SKV_ERR_CONFIG: ConfigError, SKV_ERR_VALIDATION: ValidationError, SKV_ERR_LOGIC: LogicError,
         SKV_ERR_CUDA: CudaError, SKV_ERR_ARG: ArgError}


@dataclasses.dataclass
class ModelSpec:
    """seasim::ModelSpec (cost_model.hpp:19-40) fields the KV path reads, plus GQA."""

    model_id: str
    num_layers: int
    num_heads: int  # KV heads (the reference's num_heads sizes the native block)
    head_dim: int = 128
    dtype_bytes: int = 2
    num_q_heads: int = 0  # 0 -> num_heads


@dataclasses.dataclass
class CacheStats:
    """seasim::CacheStats (kv_cache.hpp:35-40)."""

    block_table_entries: int = 0
    native_reads_writes: int = 0
    internal_fragmentation_bytes: float = 0.0
    peak_utilization: float = 0.0


class _ModelDesc(C.Structure):
    _fields_ = [("model_id", C.c_char_p), ("num_layers", C.c_int32), ("num_heads", C.c_int32),
                ("num_q_heads", C.c_int32), ("head_dim", C.c_int32), ("dtype_bytes", C.c_int32)]


class _Opts(C.Structure):
    _fields_ = [("device", C.c_int32), ("dtype", C.c_int32), ("phys_layers", C.c_int32),
                ("max_requests", C.c_int32), ("max_blocks_per_request", C.c_int32),
                ("allocate_storage", C.c_int32)]


class _Stats(C.Structure):
    _fields_ = [("block_table_entries", C.c_uint64), ("native_reads_writes", C.c_uint64),
                ("internal_fragmentation_bytes", C.c_double), ("peak_utilization", C.c_double)]


class KvOp(C.Structure):
    """KvOp (kv_cache.hpp:270-275): kind 0 = kGrow, 1 = kFree."""

    _fields_ = [("kind", C.c_int32), ("model_idx", C.c_int32), ("request_id", C.c_uint64),
                ("tokens", C.c_int64)]


# KvOp as a numpy record (same layout as the C struct skv_kv_op)
KVOP_DTYPE = np.dtype([("kind", "<i4"), ("model", "<i4"), ("id", "<u8"), ("tokens", "<i8")])
assert KVOP_DTYPE.itemsize == C.sizeof(KvOp)


class Layout(C.Structure):
    _fields_ = [("merged_stride", C.c_int64), ("native_stride", C.c_int64), ("layer_stride", C.c_int64),
                ("head_stride", C.c_int64), ("kv_stride", C.c_int64), ("tpb", C.c_int32),
                ("head_dim", C.c_int32), ("kv_heads", C.c_int32), ("q_heads", C.c_int32),
                ("phys_layers", C.c_int32), ("dtype", C.c_int32)]


class _DecodeArgs(C.Structure):
    _fields_ = [("q", C.POINTER(C.c_void_p)), ("out", C.POINTER(C.c_void_p)), ("softmax_scale", C.c_float),
                ("layer", C.c_int32), ("split_tokens", C.c_int32), ("k", C.POINTER(C.c_void_p)),
                ("v", C.POINTER(C.c_void_p))]


class _AppendArgs(C.Structure):
    _fields_ = [("k", C.POINTER(C.c_void_p)), ("v", C.POINTER(C.c_void_p)), ("layer", C.c_int32),
                ("n_new", C.c_int32), ("n_news", C.POINTER(C.c_int32))]


class _PrefillArgs(C.Structure):
    _fields_ = [("q", C.POINTER(C.c_void_p)), ("out", C.POINTER(C.c_void_p)), ("softmax_scale", C.c_float),
                ("layer", C.c_int32), ("q_len", C.c_int32), ("q_lens", C.POINTER(C.c_int32))]


_lib = None


def build() -> None:
    """Compile libseakv.so for sm_100a (nvcc cross-compiles without a GPU)."""
    subprocess.run(["make", "-s", "-C", os.path.join(_HERE, "csrc")], check=True)


def lib() -> C.CDLL:
    """The loaded CUDA library.  Raises if it is missing and cannot be built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libseakv.so not built at {LIB_PATH}")
    L = C.CDLL(LIB_PATH)
    P, S, V = C.c_void_p, C.c_int, None
    sig = {
        "skv_version": (C.c_char_p, []),
        "skv_default_opts": (V, [C.POINTER(_Opts)]),
        "skv_native_block_bytes": (S, [C.POINTER(_ModelDesc), C.c_int32, C.c_int32, C.POINTER(C.c_double)]),
        "skv_plan_merged_shape": (S, [C.POINTER(_ModelDesc), C.c_int32, C.c_int32, C.c_int32,
                                      C.POINTER(C.c_double)]),
        "skv_pool_create": (S, [C.POINTER(_ModelDesc), C.c_int32, C.c_int32, C.c_int32, C.c_size_t,
                                C.POINTER(_Opts), C.POINTER(P)]),
        "skv_pool_destroy": (V, [P]),
        "skv_last_error": (C.c_char_p, [P]),
        "skv_model_index": (S, [P, C.c_char_p, C.POINTER(C.c_int32)]),
        "skv_sub_slots_per_merged": (C.c_int32, [P, C.c_int32]),
        "skv_merged_block_bytes": (C.c_double, [P]),
        "skv_pool_size": (C.c_size_t, [P]),
        "skv_free_blocks": (C.c_size_t, [P]),
        "skv_allocated_blocks": (C.c_size_t, [P]),
        "skv_tokens_per_block": (C.c_int32, [P]),
        "skv_native_blocks_for": (C.c_size_t, [P, C.c_int64]),
        "skv_registered": (C.c_int32, [P, C.c_uint64]),
        "skv_request_tokens": (C.c_int64, [P, C.c_uint64]),
        "skv_available_slots": (C.c_size_t, [P, C.c_int32]),
        "skv_can_grow_to": (S, [P, C.c_uint64, C.c_int32, C.c_int64, C.POINTER(C.c_int32)]),
        "skv_try_allocate": (S, [P, C.c_uint64, C.c_int32, C.c_int64]),
        "skv_free_request": (S, [P, C.c_uint64]),
        "skv_record_context_read": (S, [P, C.c_uint64]),
        "skv_block_table": (S, [P, C.c_uint64, P, C.c_size_t, C.POINTER(C.c_size_t)]),
        "skv_owner_of": (S, [P, C.c_int32, C.c_int32, C.POINTER(C.c_uint64)]),
        "skv_table_entries": (C.c_size_t, [P]),
        "skv_fragmentation_bytes": (C.c_double, [P]),
        "skv_stats": (S, [P, C.POINTER(_Stats)]),
        "skv_replay": (S, [P, P, C.c_size_t, P]),
        "skv_flush": (S, [P, P]),
        "skv_synchronize": (S, [P]),
        "skv_set_stream": (S, [P, P]),
        "skv_get_stream": (P, [P]),
        "skv_batch_create": (S, [P, P, P, C.c_int32, P, C.POINTER(P)]),
        "skv_batch_destroy": (V, [P]),
        "skv_batch_reset": (S, [P, P, P, P, C.c_int32, P]),
        "skv_batch_grow": (S, [P, P, C.c_int64, C.POINTER(C.c_int32)]),
        "skv_batch_decode_bytes": (S, [P, P, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "skv_batch_grow_mirror": (S, [P, P, C.c_int64, C.POINTER(C.c_int32)]),
        "skv_batch_grow_launch": (S, [P, P, C.c_int64, P]),
        "skv_decode_attention": (S, [P, P, C.POINTER(_DecodeArgs), P]),
        "skv_batch_plan_info": (S, [P, P, C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "skv_append_kv": (S, [P, P, C.POINTER(_AppendArgs), P]),
        "skv_prefill_attention": (S, [P, P, C.POINTER(_PrefillArgs), P]),
        "skv_model_layout": (S, [P, C.c_int32, C.POINTER(Layout)]),
        "skv_storage": (P, [P, C.POINTER(C.c_size_t)]),
        "skv_synth_fill": (S, [P, C.c_uint64, C.c_float, P]),
        "skv_read_blocks": (S, [P, P, C.c_size_t, P]),
        "skv_kernel_launches": (C.c_uint64, [P]),
        "skv_debug_decode_trace": (S, [P, P, P, C.c_size_t, C.POINTER(C.c_size_t)]),
        "skv_split_create": (S, [C.POINTER(_ModelDesc), C.c_int32, C.c_int32, C.c_int32, C.c_size_t,
                                 C.POINTER(_Opts), C.POINTER(P)]),
        "skv_split_destroy": (V, [P]),
        "skv_split_last_error": (C.c_char_p, [P]),
        "skv_split_registry": (P, [P]),
        "skv_split_free_blocks": (C.c_size_t, [P]),
        "skv_split_pool_size": (C.c_size_t, [P]),
        "skv_split_kernel_launches": (C.c_uint64, [P]),
        "skv_split_grow": (S, [P, P, P, P, C.c_int32, P]),
        "skv_split_free": (S, [P, P, C.c_int32]),
        "skv_split_stats": (S, [P, C.POINTER(_Stats)]),
        "skv_split_table_entries": (C.c_uint64, [P]),
        "skv_split_synth_fill": (S, [P, C.c_uint64, C.c_float, P]),
        "skv_split_decode": (S, [P, P, C.POINTER(_DecodeArgs), P]),
        "skv_split_append": (S, [P, P, C.POINTER(_AppendArgs), P]),
        "skv_split_block_ids": (S, [P, C.c_uint64, C.c_int32, C.c_int32, P, C.c_size_t, C.POINTER(C.c_size_t)]),
        "skv_split_read_blocks": (S, [P, P, C.c_size_t, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _desc(models: Sequence[ModelSpec]):
    arr = (_ModelDesc * max(1, len(models)))()
    keep = []
    for i, m in enumerate(models):
        b = m.model_id.encode()
        keep.append(b)
        arr[i] = _ModelDesc(b, m.num_layers, m.num_heads, m.num_q_heads, m.head_dim, m.dtype_bytes)
    return arr, keep


def _raise(st: int, pool=None):
    if st in (SKV_OK, SKV_CACHE_FULL):
        return
    msg = lib().skv_last_error(pool)
    raise _ERRS.get(st, RuntimeError)(msg.decode() if msg else f"status {st}")


def native_block_bytes(model: ModelSpec, tokens_per_block: int = 16, tp_size: int = 1) -> float:
    """kv_cache.hpp:17-22"""
    arr, _k = _desc([model])
    out = C.c_double()
    _raise(lib().skv_native_block_bytes(arr, tokens_per_block, tp_size, C.byref(out)))
    return out.value


def plan_merged_shape(models: Sequence[ModelSpec], tokens_per_block: int = 16, tp_size: int = 1) -> float:
    """kv_cache.hpp:26-33"""
    arr, _k = _desc(models)
    out = C.c_double()
    _raise(lib().skv_plan_merged_shape(arr, len(models), tokens_per_block, tp_size, C.byref(out)))
    return out.value


def _ptr(x) -> int:
    """Device/host address of a torch tensor, an int, or None."""
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    return int(x.data_ptr())


_CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy: torch's default stream has handle 0, which the C-ABI reads as "pool stream"


def _stream_ptr(stream) -> int | None:
    """Stream handle for the C-ABI.  None -> torch's current stream when torch is in use, so
    kernels are ordered after the torch ops that produced their inputs (and before those
    that consume their outputs); the pool's own stream only when torch is not loaded."""
    if stream is None:
        import sys
        torch = sys.modules.get("torch")
        if torch is None or not torch.cuda.is_available() or not torch.cuda.is_initialized():
            return None
        stream = torch.cuda.current_stream()
    if isinstance(stream, int):
        return stream or _CUDA_STREAM_LEGACY
    return int(stream.cuda_stream) or _CUDA_STREAM_LEGACY


class UnifiedKvCache:
    """The unified merged-block KV pool on one GPU (kv_cache.hpp:46-267)."""

    def __init__(self, models: Sequence[ModelSpec], tokens_per_block: int = 16, tp_size: int = 1,
                 pool_blocks: int = 0, *, device: int = 0, dtype: int = FP16, phys_layers: int = 0,
                 max_requests: int = 4096, max_blocks_per_request: int = 0, allocate_storage: bool = False):
        L = lib()
        self._lib = L
        self.models = list(models)
        arr, self._keep = _desc(self.models)
        opts = _Opts()
        L.skv_default_opts(C.byref(opts))
        opts.device, opts.dtype, opts.phys_layers = device, dtype, phys_layers
        opts.max_requests, opts.max_blocks_per_request = max_requests, max_blocks_per_request
        opts.allocate_storage = 1 if allocate_storage else 0
        h = C.c_void_p()
        st = L.skv_pool_create(arr, len(self.models), tokens_per_block, tp_size, pool_blocks, C.byref(opts),
                               C.byref(h))
        _raise(st, None)
        self._h = h.value
        self.device = device
        self.dtype = dtype

    # -- lifetime ------------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._lib.skv_pool_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _chk(self, st):
        _raise(st, self._h)
        return st

    # -- reference surface (kv_cache.hpp:68-170) -------------------------------------------
    def model_index(self, model_id: str) -> int:
        out = C.c_int32()
        self._chk(self._lib.skv_model_index(self._h, model_id.encode(), C.byref(out)))
        return out.value

    def sub_slots_per_merged(self, m: int) -> int:
        return self._lib.skv_sub_slots_per_merged(self._h, m)

    def merged_block_bytes(self) -> float:
        return self._lib.skv_merged_block_bytes(self._h)

    def pool_size(self) -> int:
        return self._lib.skv_pool_size(self._h)

    def free_blocks(self) -> int:
        return self._lib.skv_free_blocks(self._h)

    def allocated_blocks(self) -> int:
        return self._lib.skv_allocated_blocks(self._h)

    def tokens_per_block(self) -> int:
        return self._lib.skv_tokens_per_block(self._h)

    def native_blocks_for(self, tokens: int) -> int:
        return self._lib.skv_native_blocks_for(self._h, tokens)

    def registered(self, request_id: int) -> bool:
        return bool(self._lib.skv_registered(self._h, request_id))

    def request_tokens(self, request_id: int) -> int:
        return self._lib.skv_request_tokens(self._h, request_id)

    def available_slots(self, m: int) -> int:
        return self._lib.skv_available_slots(self._h, m)

    def can_grow_to(self, request_id: int, m: int, tokens: int) -> bool:
        out = C.c_int32()
        self._chk(self._lib.skv_can_grow_to(self._h, request_id, m, tokens, C.byref(out)))
        return bool(out.value)

    def try_allocate(self, request_id: int, m: int, tokens: int) -> bool:
        return self._chk(self._lib.skv_try_allocate(self._h, request_id, m, tokens)) == SKV_OK

    def try_allocate_rc(self, request_id: int, m: int, tokens: int) -> int:
        """Raw status mapped to the oracle's codes: 0 granted, 1 full, -2 validation, -3 logic."""
        st = self._lib.skv_try_allocate(self._h, request_id, m, tokens)
        return st

    def free_request(self, request_id: int) -> None:
        self._chk(self._lib.skv_free_request(self._h, request_id))

    def record_context_read(self, request_id: int) -> None:
        self._chk(self._lib.skv_record_context_read(self._h, request_id))

    def block_table_np(self, request_id: int) -> np.ndarray:
        n = C.c_size_t()
        self._chk(self._lib.skv_block_table(self._h, request_id, None, 0, C.byref(n)))
        buf = np.zeros((n.value, 2), dtype=np.int32)
        if n.value:
            self._chk(self._lib.skv_block_table(self._h, request_id, buf.ctypes.data, n.value, C.byref(n)))
        return buf

    def block_table(self, request_id: int):
        return [tuple(map(int, r)) for r in self.block_table_np(request_id)]

    def owner_of(self, block: int, slot: int) -> int:
        out = C.c_uint64()
        self._chk(self._lib.skv_owner_of(self._h, block, slot, C.byref(out)))
        return out.value

    def table_entries(self) -> int:
        return self._lib.skv_table_entries(self._h)

    def fragmentation_bytes(self) -> float:
        return self._lib.skv_fragmentation_bytes(self._h)

    def stats(self) -> dict:
        s = _Stats()
        self._chk(self._lib.skv_stats(self._h, C.byref(s)))
        return dict(block_table_entries=s.block_table_entries, native_reads_writes=s.native_reads_writes,
                    internal_fragmentation_bytes=s.internal_fragmentation_bytes,
                    peak_utilization=s.peak_utilization)

    # -- batched / replay -------------------------------------------------------------------
    def replay(self, ops: Iterable[tuple]) -> np.ndarray:
        ops = list(ops)
        arr = (KvOp * max(1, len(ops)))()
        for i, (kind, rid, m, tok) in enumerate(ops):
            arr[i] = KvOp(kind, m, rid, tok)
        granted = np.zeros(max(1, len(ops)), dtype=np.int32)
        self._chk(self._lib.skv_replay(self._h, arr, len(ops), granted.ctypes.data))
        return granted[: len(ops)]

    def replay_array(self, arr: np.ndarray) -> np.ndarray:
        """Batched KvOp stream (numpy structured array of KVOP_DTYPE): one C-ABI call applies every
        op in order with try_allocate / free_request semantics (skv_replay); returns granted
        flags (1 granted / 0 CacheFull for grows, 0 for frees)."""
        arr = np.ascontiguousarray(arr, dtype=KVOP_DTYPE)
        granted = np.zeros(max(1, len(arr)), dtype=np.int32)
        if len(arr):
            self._chk(self._lib.skv_replay(self._h, arr.ctypes.data, len(arr), granted.ctypes.data))
        return granted[: len(arr)]

    def flush(self, stream=None):
        self._chk(self._lib.skv_flush(self._h, _stream_ptr(stream)))

    def synchronize(self):
        self._chk(self._lib.skv_synchronize(self._h))

    def set_stream(self, stream):
        self._chk(self._lib.skv_set_stream(self._h, _stream_ptr(stream)))

    def kernel_launches(self) -> int:
        return self._lib.skv_kernel_launches(self._h)

    # -- storage ----------------------------------------------------------------------------
    def layout(self, m: int) -> Layout:
        out = Layout()
        self._chk(self._lib.skv_model_layout(self._h, m, C.byref(out)))
        return out

    def storage(self):
        n = C.c_size_t()
        p = self._lib.skv_storage(self._h, C.byref(n))
        return p, n.value

    def synth_fill(self, seed: int, amp: float = 1.0, stream=None):
        self._chk(self._lib.skv_synth_fill(self._h, seed, amp, _stream_ptr(stream)))

    def read_blocks(self, ids) -> np.ndarray:
        ids = np.ascontiguousarray(np.asarray(ids, dtype=np.int32))
        stride = self.layout(0).merged_stride
        out = np.zeros(len(ids) * stride, dtype=np.uint8)
        if len(ids):
            self._chk(self._lib.skv_read_blocks(self._h, ids.ctypes.data, len(ids), out.ctypes.data))
        return out

    def batch(self, groups: Sequence[tuple[int, Sequence[int]]]) -> "Batch":
        return Batch(self, groups)


def _check_tensors(ts, shapes, dtype: int, device: int, what: str):
    """Raises ArgError unless every torch tensor in ``ts`` is a contiguous CUDA tensor on
    ``device`` of the pool's dtype with the expected shape (the C-ABI takes raw pointers, so
    a mismatch would otherwise read or write out of bounds).  Raw integer addresses are
    passed through unchecked."""
    if len(ts) != len(shapes):
        raise ArgError(f"{what}: expected {len(shapes)} tensors (one per group), got {len(ts)}")
    for g, (t, shp) in enumerate(zip(ts, shapes)):
        if isinstance(t, int):
            continue
        if not hasattr(t, "data_ptr"):
            raise ArgError(f"{what}[{g}]: expected a torch tensor or a device address")
        if not t.is_cuda or (t.device.index or 0) != device:
            raise ArgError(f"{what}[{g}]: tensor on {t.device}, pool on cuda:{device}")
        want = "float16" if dtype == FP16 else "bfloat16"
        if str(t.dtype).split(".")[-1] != want:
            raise ArgError(f"{what}[{g}]: dtype {t.dtype}, pool stores {want}")
        if tuple(t.shape) != tuple(shp):
            raise ArgError(f"{what}[{g}]: shape {tuple(t.shape)}, expected {tuple(shp)}")
        if not t.is_contiguous():
            raise ArgError(f"{what}[{g}]: tensor must be contiguous")


class Batch:
    """Requests covered by one data-path launch, grouped by service (model index)."""

    def __init__(self, cache: UnifiedKvCache, groups: Sequence[tuple[int, Sequence[int]]]):
        self.cache = cache
        self.groups = [(int(m), [int(i) for i in ids]) for m, ids in groups]
        lay = {m: cache.layout(m) for m in {m for m, _ in self.groups}}
        # per group (B_g, Hq/tp, Hkv/tp, head_dim) for argument validation
        self._shapes = [(len(ids), lay[m].q_heads, lay[m].kv_heads, lay[m].head_dim) for m, ids in self.groups]
        gm = (C.c_int32 * len(self.groups))(*[m for m, _ in self.groups])
        gs = (C.c_int32 * len(self.groups))(*[len(ids) for _, ids in self.groups])
        flat = [i for _, ids in self.groups for i in ids]
        idarr = (C.c_uint64 * max(1, len(flat)))(*flat)
        h = C.c_void_p()
        cache._chk(cache._lib.skv_batch_create(cache._h, gm, gs, len(self.groups), idarr, C.byref(h)))
        self._h = h.value

    def reset(self, groups: Sequence[tuple[int, Sequence[int]]]):
        """Re-point this batch at new requests, reusing its device buffers."""
        self.groups = [(int(m), [int(i) for i in ids]) for m, ids in groups]
        lay = {m: self.cache.layout(m) for m in {m for m, _ in self.groups}}
        self._shapes = [(len(ids), lay[m].q_heads, lay[m].kv_heads, lay[m].head_dim) for m, ids in self.groups]
        gm = (C.c_int32 * len(self.groups))(*[m for m, _ in self.groups])
        gs = (C.c_int32 * len(self.groups))(*[len(ids) for _, ids in self.groups])
        flat = [i for _, ids in self.groups for i in ids]
        idarr = (C.c_uint64 * max(1, len(flat)))(*flat)
        self.cache._chk(self.cache._lib.skv_batch_reset(self.cache._h, self._h, gm, gs, len(self.groups), idarr))

    def close(self):
        if getattr(self, "_h", None) and self.cache._h:
            self.cache._lib.skv_batch_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def grow(self, delta: int = 1) -> int:
        n = C.c_int32()
        self.cache._chk(self.cache._lib.skv_batch_grow(self.cache._h, self._h, delta, C.byref(n)))
        return n.value

    def grow_mirror(self, delta: int = 1) -> bool:
        """Host half of a device-generated decode-step growth (skv_batch_grow_mirror): True when
        every request was granted and the mirror advanced; False = nothing changed."""
        ok = C.c_int32()
        self.cache._chk(self.cache._lib.skv_batch_grow_mirror(self.cache._h, self._h, delta, C.byref(ok)))
        return bool(ok.value)

    def grow_launch(self, delta: int = 1, stream=None):
        """Device half (op generation + placement kernel), once per successful grow_mirror."""
        self.cache._chk(self.cache._lib.skv_batch_grow_launch(self.cache._h, self._h, delta, _stream_ptr(stream)))

    def decode_bytes(self, layer: int) -> tuple[float, float]:
        kv, tot = C.c_double(), C.c_double()
        self.cache._chk(self.cache._lib.skv_batch_decode_bytes(self.cache._h, self._h, layer, C.byref(kv),
                                                               C.byref(tot)))
        return kv.value, tot.value

    def decode(self, q: Sequence, out: Sequence, layer: int, softmax_scale: float = 0.0, split_tokens: int = 0,
               stream=None, k: Sequence | None = None, v: Sequence | None = None):
        """Paged decode attention of every group for ``layer``.  With ``k``/``v`` (each
        [B_g, 1, Hkv, d]) the step's new token is appended at position tokens-1 inside the
        same launch (fused ``append(k, v, layer, 1)``)."""
        self.cache._chk(self.cache._lib.skv_decode_attention(self.cache._h, self._h,
                                                             C.byref(self._decode_args(q, out, layer, softmax_scale,
                                                                                       split_tokens, k, v)),
                                                             _stream_ptr(stream)))

    def _decode_args(self, q, out, layer, softmax_scale, split_tokens, k, v):
        dt, dev = self.cache.dtype, self.cache.device
        _check_tensors(q, [(B, Hq, d) for B, Hq, _, d in self._shapes], dt, dev, "decode q")
        _check_tensors(out, [(B, Hq, d) for B, Hq, _, d in self._shapes], dt, dev, "decode out")
        if k is not None and v is not None:
            _check_tensors(k, [(B, 1, Hkv, d) for B, _, Hkv, d in self._shapes], dt, dev, "decode k")
            _check_tensors(v, [(B, 1, Hkv, d) for B, _, Hkv, d in self._shapes], dt, dev, "decode v")
        n = len(self.groups)
        qa = (C.c_void_p * n)(*[_ptr(t) for t in q])
        oa = (C.c_void_p * n)(*[_ptr(t) for t in out])
        a = _DecodeArgs(C.cast(qa, C.POINTER(C.c_void_p)), C.cast(oa, C.POINTER(C.c_void_p)), softmax_scale,
                        layer, split_tokens)
        if (k is None) != (v is None):
            raise ValueError("decode: pass both k and v for the fused append, or neither")
        if k is not None:
            ka = (C.c_void_p * n)(*[_ptr(t) for t in k])
            va = (C.c_void_p * n)(*[_ptr(t) for t in v])
            a.k = C.cast(ka, C.POINTER(C.c_void_p))
            a.v = C.cast(va, C.POINTER(C.c_void_p))
        a._keep = (qa, oa) + ((ka, va) if k is not None else ())
        return a

    def plan_info(self) -> dict:
        """Schedule of the last decode launch: split_tokens, n_cut (the last n_cut (request,
        kv head)s of the batch, in batch order, were cut into pieces merged in-kernel), sum_hkv."""
        s, n, h = C.c_int32(), C.c_int64(), C.c_int64()
        self.cache._chk(self.cache._lib.skv_batch_plan_info(self.cache._h, self._h, C.byref(s), C.byref(n),
                                                            C.byref(h)))
        return {"split_tokens": s.value, "n_cut": n.value, "sum_hkv": h.value}

    def decode_trace(self, max_records: int = 4096) -> np.ndarray:
        """Debug (SKV_TRACE=1): per-warp [start_ns, after_wait_ns, end_ns, tiles<<32|items]
        of the last decode launch (or, for a prefill built with -DSKV_PF_TRACE, 16 u64 of
        per-role wait cycles per CTA); empty when tracing is off."""
        buf = np.zeros((max_records, 4), dtype=np.uint64)
        n = C.c_size_t()
        self.cache._chk(self.cache._lib.skv_debug_decode_trace(self.cache._h, self._h, buf.ctypes.data,
                                                               buf.size, C.byref(n)))
        return buf[: n.value]

    def append(self, k: Sequence, v: Sequence, layer: int, n_new=1, stream=None):
        """Writes each request's last ``n_new`` tokens' K/V of ``layer``.  ``n_new``: one int
        (k/v of group g: [B_g, n_new, Hkv, d]) or one count per request in batch order (k/v of
        group g packed by request: [sum of its counts, Hkv, d])."""
        self.cache._chk(self.cache._lib.skv_append_kv(self.cache._h, self._h, C.byref(self._append_args(k, v, layer,
                                                                                                       n_new)),
                                                      _stream_ptr(stream)))

    def _ragged_shapes(self, lens, what, heads):
        lens = [int(x) for x in lens]
        total = sum(B for B, _, _, _ in self._shapes)
        if len(lens) != total:
            raise ArgError(f"{what}: {len(lens)} lengths for {total} requests")
        shp, k = [], 0
        for B, Hq, Hkv, d in self._shapes:
            shp.append((sum(lens[k:k + B]), Hq if heads == "q" else Hkv, d))
            k += B
        return lens, shp

    def _append_args(self, k, v, layer, n_new):
        dt, dev = self.cache.dtype, self.cache.device
        ragged = not isinstance(n_new, (int, np.integer))
        if ragged:
            lens, shp = self._ragged_shapes(n_new, "append", "kv")
        else:
            shp = [(B, int(n_new), Hkv, d) for B, _, Hkv, d in self._shapes]
        _check_tensors(k, shp, dt, dev, "append k")
        _check_tensors(v, shp, dt, dev, "append v")
        n = len(self.groups)
        ka = (C.c_void_p * n)(*[_ptr(t) for t in k])
        va = (C.c_void_p * n)(*[_ptr(t) for t in v])
        a = _AppendArgs(C.cast(ka, C.POINTER(C.c_void_p)), C.cast(va, C.POINTER(C.c_void_p)), layer,
                        0 if ragged else int(n_new))
        a._keep = (ka, va)
        if ragged:
            arr = (C.c_int32 * max(1, len(lens)))(*lens)
            a.n_news = C.cast(arr, C.POINTER(C.c_int32))
            a._keep = (ka, va, arr)
        return a

    def prefill(self, q: Sequence, out: Sequence, layer: int, q_len, softmax_scale: float = 0.0,
                stream=None):
        """Causal chunked prefill of every request's last ``q_len`` tokens (already appended).
        ``q_len``: one int for the whole batch (q/out of group g: [B_g, q_len, Hq, d]) or one
        length per request in batch order (q/out of group g packed by request:
        [sum of its lengths, Hq, d])."""
        dt, dev = self.cache.dtype, self.cache.device
        n = len(self.groups)
        ragged = not isinstance(q_len, (int, np.integer))
        if ragged:
            lens, shp = self._ragged_shapes(q_len, "prefill", "q")
            ql = (C.c_int32 * max(1, len(lens)))(*lens)
        else:
            shp = [(B, int(q_len), Hq, d) for B, Hq, _, d in self._shapes]
        _check_tensors(q, shp, dt, dev, "prefill q")
        _check_tensors(out, shp, dt, dev, "prefill out")
        qa = (C.c_void_p * n)(*[_ptr(t) for t in q])
        oa = (C.c_void_p * n)(*[_ptr(t) for t in out])
        a = _PrefillArgs(C.cast(qa, C.POINTER(C.c_void_p)), C.cast(oa, C.POINTER(C.c_void_p)), softmax_scale,
                         layer, 0 if ragged else int(q_len))
        if ragged:
            a.q_lens = C.cast(ql, C.POINTER(C.c_int32))
        self.cache._chk(self.cache._lib.skv_prefill_attention(self.cache._h, self._h, C.byref(a),
                                                              _stream_ptr(stream)))


class SplitKvCache:
    """The split scheme on the GPU (reference SplitCacheCounter,
    kv_cache.hpp:277-348): per-(layer, kv head) 8 KiB blocks with one table entry each,
    same decode kernel as the merged pool.  ``grow``/``free`` are batched
    SplitCacheCounter calls; ``stats()`` is SplitCacheCounter::stats."""

    def __init__(self, models: Sequence[ModelSpec], tokens_per_block: int = 16, tp_size: int = 1,
                 split_blocks: int = 0, *, device: int = 0, dtype: int = FP16, max_requests: int = 4096,
                 max_blocks_per_request: int = 0):
        L = lib()
        self._lib = L
        self.models = list(models)
        arr, self._keep = _desc(self.models)
        opts = _Opts()
        L.skv_default_opts(C.byref(opts))
        opts.device, opts.dtype = device, dtype
        opts.max_requests, opts.max_blocks_per_request = max_requests, max_blocks_per_request
        h = C.c_void_p()
        _raise(L.skv_split_create(arr, len(self.models), tokens_per_block, tp_size, split_blocks, C.byref(opts),
                                  C.byref(h)), None)
        self._s = h.value
        reg = UnifiedKvCache.__new__(UnifiedKvCache)  # the registry pool is owned by the split pool
        reg._lib, reg._h, reg.models, reg.device, reg.dtype = L, L.skv_split_registry(self._s), self.models, device, dtype
        reg.close = lambda: None
        self.registry = reg
        self.device, self.dtype = device, dtype

    def close(self):
        if getattr(self, "_s", None):
            self.registry._h = None
            self._lib.skv_split_destroy(self._s)
            self._s = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, st):
        if st not in (SKV_OK, SKV_CACHE_FULL):
            msg = self._lib.skv_split_last_error(self._s)
            raise _ERRS.get(st, RuntimeError)(msg.decode() if msg else f"status {st}")
        return st

    def grow(self, ids: Sequence[int], models: Sequence[int], tokens: Sequence[int]) -> np.ndarray:
        n = len(ids)
        ia = np.asarray(ids, dtype=np.uint64)
        ma = np.asarray(models, dtype=np.int32)
        ta = np.asarray(tokens, dtype=np.int64)
        g = np.zeros(n, dtype=np.int32)
        self._chk(self._lib.skv_split_grow(self._s, ia.ctypes.data, ma.ctypes.data, ta.ctypes.data, n, g.ctypes.data))
        return g.astype(bool)

    def free(self, ids: Sequence[int]):
        ia = np.asarray(ids, dtype=np.uint64)
        self._chk(self._lib.skv_split_free(self._s, ia.ctypes.data, len(ia)))

    def stats(self) -> dict:
        st = _Stats()
        self._chk(self._lib.skv_split_stats(self._s, C.byref(st)))
        return {"block_table_entries": st.block_table_entries, "native_reads_writes": st.native_reads_writes,
                "internal_fragmentation_bytes": st.internal_fragmentation_bytes,
                "peak_utilization": st.peak_utilization}

    def table_entries(self) -> int:
        return self._lib.skv_split_table_entries(self._s)

    def free_blocks(self) -> int:
        return self._lib.skv_split_free_blocks(self._s)

    def pool_size(self) -> int:
        return self._lib.skv_split_pool_size(self._s)

    def kernel_launches(self) -> int:
        return self._lib.skv_split_kernel_launches(self._s) + self.registry.kernel_launches()

    def request_tokens(self, request_id: int) -> int:
        return self.registry.request_tokens(request_id)

    def synth_fill(self, seed: int, amp: float = 1.0, stream=None):
        self._chk(self._lib.skv_split_synth_fill(self._s, seed, amp, _stream_ptr(stream)))

    def set_stream(self, stream):
        self.registry.set_stream(stream)

    def block_ids(self, request_id: int, layer: int, head: int) -> np.ndarray:
        out = np.zeros(1 << 16, dtype=np.int32)
        n = C.c_size_t()
        self._chk(self._lib.skv_split_block_ids(self._s, request_id, layer, head, out.ctypes.data, out.size,
                                                C.byref(n)))
        return out[: n.value].copy()

    def read_blocks(self, ids) -> np.ndarray:
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        out = np.empty(len(ids) * 8192, dtype=np.uint8)
        self._chk(self._lib.skv_split_read_blocks(self._s, ids.ctypes.data, len(ids), out.ctypes.data))
        return out

    def batch(self, groups: Sequence[tuple[int, Sequence[int]]]) -> "SplitBatch":
        return SplitBatch(self, groups)


class SplitBatch(Batch):
    """A batch of a SplitKvCache: decode / append address the split tables."""

    def __init__(self, split: SplitKvCache, groups):
        self.split = split
        super().__init__(split.registry, groups)

    def grow(self, delta: int = 1) -> int:
        ids = [i for _, g in self.groups for i in g]
        models = [m for m, g in self.groups for _ in g]
        toks = [self.split.request_tokens(i) + delta for i in ids]
        return int(self.split.grow(ids, models, toks).sum())

    def decode(self, q, out, layer, softmax_scale=0.0, split_tokens=0, stream=None, k=None, v=None):
        if (k is None) != (v is None):
            raise ValueError("decode: pass both k and v for the fused append, or neither")
        a = self._decode_args(q, out, layer, softmax_scale, split_tokens, k, v)
        self.split._chk(self.split._lib.skv_split_decode(self.split._s, self._h, C.byref(a), _stream_ptr(stream)))

    def append(self, k, v, layer, n_new=1, stream=None):
        a = self._append_args(k, v, layer, n_new)
        self.split._chk(self.split._lib.skv_split_append(self.split._s, self._h, C.byref(a), _stream_ptr(stream)))

    def prefill(self, *a, **k):
        raise NotImplementedError("the split-scheme pool implements the decode path (SURVEY §8(f) row 2)")

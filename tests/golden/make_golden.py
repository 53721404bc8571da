#!/usr/bin/env python
"""Generates the committed golden fixtures (run in the dev container, where
/root/reference exists):

* alloc_golden.npz — seeded KvOp streams replayed through the UNMODIFIED reference
  allocator (oracle/_ref/libref_kv.so, built from /root/reference/proj/include):
  per-op grant results, the final block table of every registered request,
  CacheStats, fragmentation_bytes, free blocks.
* attn_golden.npz — a small two-service pool: block tables from the reference
  allocator, K/V contents from the SplitMix64 synthetic generator (the formula of
  skv_synth_fill, recomputed here in numpy), fp16 queries, and decode outputs from
  an independent float64 numpy implementation of softmax(q·Kᵀ/√d)·V.
* prefill_golden.npz — causal chunked prefill (the last 32 tokens of every request
  with at least 32) on the same pool and tables, float64 numpy.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import oracle_py as O  # noqa: E402
from _workloads import random_stream  # noqa: E402

ALLOC_CASES = [  # (shapes (layers, heads), pool, seed, n_ops, max_live, max_grow)
    ([(2, 2), (8, 8)], 64, 11, 6000, 60, 40),
    ([(32, 8), (32, 8), (40, 40), (32, 32)], 400, 22, 8000, 150, 200),
    ([(3, 3), (8, 8), (4, 2), (5, 5)], 80, 33, 6000, 80, 60),
]


def synth_fp16(seed, n):
    """skv_synth_fill: element i = (2u-1), u = top 24 bits of SplitMix64(seed + (i+1)*golden)."""
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (i + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)
    return (np.float32(2.0) * u - np.float32(1.0)).astype(np.float16)


def make_alloc():
    out = {}
    for ci, (shapes, pool, seed, n_ops, max_live, max_grow) in enumerate(ALLOC_CASES):
        models = [(L, H, 128, 2) for L, H in shapes]
        ops = random_stream(seed, n_ops, len(shapes), max_live=max_live, max_grow=max_grow)
        ref = O.RefCache(models, pool=pool)
        granted = []
        for kind, rid, m, tok in ops:
            if kind == 0:
                granted.append(1 if ref.try_allocate(rid, m, tok) else 0)
            else:
                ref.free_request(rid)
                granted.append(0)
        ids = sorted({op[1] for op in ops if ref.registered(op[1])})
        tabs = [np.array(ref.block_table(i), dtype=np.int32).reshape(-1, 2) for i in ids]
        offs = np.cumsum([0] + [len(t) for t in tabs]).astype(np.int64)
        s = ref.stats()
        out[f"c{ci}_shapes"] = np.array(shapes, dtype=np.int32)
        out[f"c{ci}_pool"] = np.int64(pool)
        out[f"c{ci}_ops"] = np.array(ops, dtype=np.int64)
        out[f"c{ci}_granted"] = np.array(granted, dtype=np.int8)
        out[f"c{ci}_ids"] = np.array(ids, dtype=np.uint64)
        out[f"c{ci}_table_offsets"] = offs
        out[f"c{ci}_tables"] = np.concatenate(tabs) if tabs else np.zeros((0, 2), np.int32)
        out[f"c{ci}_stats"] = np.array([s["block_table_entries"], s["native_reads_writes"],
                                        s["internal_fragmentation_bytes"], s["peak_utilization"]], dtype=np.float64)
        out[f"c{ci}_frag"] = np.float64(ref.fragmentation_bytes())
        out[f"c{ci}_free"] = np.int64(ref.free_blocks())
    out["n_cases"] = np.int64(len(ALLOC_CASES))
    np.savez_compressed(os.path.join(HERE, "alloc_golden.npz"), **out)


def make_attn():
    # two services: GQA (L=3, 4 KV / 16 Q heads) and MHA (L=2, 4 / 4); d=128 fp16; tpb 16
    shapes = [(3, 4, 16), (2, 4, 4)]
    seed = 77
    models = [(L, H, 128, 2) for L, H, _ in shapes]
    pool = 24
    ref = O.RefCache(models, pool=pool)
    ctx = {1: (0, 70), 2: (1, 33), 3: (0, 1), 4: (1, 100), 5: (0, 48)}
    ops = []
    for rid, (m, t) in ctx.items():
        assert ref.try_allocate(rid, m, t)
        ops.append((0, rid, m, t))
    merged = int(O.plan_merged_shape(models))
    stride = (merged + 255) // 256 * 256
    elems = synth_fp16(seed, pool * stride // 2)
    img = elems.view(np.uint8)
    rng = np.random.default_rng(5)
    layer = 1
    res = {"ops": np.array(ops, np.int64), "seed": np.int64(seed), "pool": np.int64(pool), "layer": np.int64(layer),
           "shapes": np.array(shapes, np.int32)}
    for m, (L, H, Hq) in enumerate(shapes):
        ids = [r for r, (mm, _) in ctx.items() if mm == m]
        layer_stride = H * 2 * 16 * 128 * 2
        native = L * layer_stride
        q = (rng.standard_normal((len(ids), Hq, 128)) * 0.7).astype(np.float16)
        out = np.zeros((len(ids), Hq, 128), np.float64)
        G = Hq // H
        for k, rid in enumerate(ids):
            n = ctx[rid][1]
            bt = ref.block_table(rid)
            K = np.zeros((H, n, 128))
            V = np.zeros((H, n, 128))
            for t in range(n):
                b, s = bt[t // 16]
                base = b * stride + s * native + layer * layer_stride + (t % 16) * 256
                for h in range(H):
                    ko = base + h * 2 * 16 * 256
                    K[h, t] = img[ko:ko + 256].view(np.float16).astype(np.float64)
                    V[h, t] = img[ko + 16 * 256:ko + 16 * 256 + 256].view(np.float16).astype(np.float64)
            for hq in range(Hq):
                s_ = K[hq // G] @ q[k, hq].astype(np.float64) / np.sqrt(128.0)
                p = np.exp(s_ - s_.max())
                out[k, hq] = (p / p.sum()) @ V[hq // G]
        res[f"m{m}_ids"] = np.array(ids, np.uint64)
        res[f"m{m}_q"] = q.view(np.uint16)
        res[f"m{m}_out"] = out.astype(np.float32)
        res[f"m{m}_ctx"] = np.array([ctx[r][1] for r in ids], np.int64)
        res[f"m{m}_tables"] = np.array([ref.block_table(r) + [(0, 0)] * (8 - len(ref.block_table(r))) for r in ids],
                                       np.int32)
    np.savez_compressed(os.path.join(HERE, "attn_golden.npz"), **res)


def make_prefill():
    """prefill_golden.npz: causal chunked-prefill attention (the last Q_LEN tokens of each
    request attend to every key at or before their position) on the attn_golden pool and
    tables, float64 numpy."""
    a = np.load(os.path.join(HERE, "attn_golden.npz"))
    shapes = [tuple(int(x) for x in r) for r in a["shapes"]]
    seed, pool, layer = int(a["seed"]), int(a["pool"]), int(a["layer"])
    models = [(L, H, 128, 2) for L, H, _ in shapes]
    merged = int(O.plan_merged_shape(models))
    stride = (merged + 255) // 256 * 256
    img = synth_fp16(seed, pool * stride // 2).view(np.uint8)
    q_len = 32
    rng = np.random.default_rng(9)
    res = {"q_len": np.int64(q_len)}
    for m, (L, H, Hq) in enumerate(shapes):
        layer_stride = H * 2 * 16 * 128 * 2
        native = L * layer_stride
        G = Hq // H
        ids = [int(i) for i in a[f"m{m}_ids"]]
        ctxs = [int(c) for c in a[f"m{m}_ctx"]]
        keep = [k for k, c in enumerate(ctxs) if c >= q_len]
        tabs = a[f"m{m}_tables"][keep]
        q = (rng.standard_normal((len(keep), q_len, Hq, 128)) * 0.7).astype(np.float16)
        out = np.zeros((len(keep), q_len, Hq, 128), np.float64)
        for kk, k in enumerate(keep):
            n = ctxs[k]
            K = np.zeros((H, n, 128))
            V = np.zeros((H, n, 128))
            for t in range(n):
                b, sl = tabs[kk][t // 16]
                base = int(b) * stride + int(sl) * native + layer * layer_stride + (t % 16) * 256
                for h in range(H):
                    ko = base + h * 2 * 16 * 256
                    K[h, t] = img[ko:ko + 256].view(np.float16).astype(np.float64)
                    V[h, t] = img[ko + 16 * 256:ko + 16 * 256 + 256].view(np.float16).astype(np.float64)
            for i in range(q_len):
                pos = n - q_len + i
                for hq in range(Hq):
                    s_ = K[hq // G, :pos + 1] @ q[kk, i, hq].astype(np.float64) / np.sqrt(128.0)
                    pr = np.exp(s_ - s_.max())
                    out[kk, i, hq] = (pr / pr.sum()) @ V[hq // G, :pos + 1]
        res[f"m{m}_ids"] = np.array([ids[k] for k in keep], np.uint64)
        res[f"m{m}_ctx"] = np.array([ctxs[k] for k in keep], np.int64)
        res[f"m{m}_tables"] = tabs
        res[f"m{m}_q"] = q.view(np.uint16)
        res[f"m{m}_out"] = out.astype(np.float32)
    np.savez_compressed(os.path.join(HERE, "prefill_golden.npz"), **res)


if __name__ == "__main__":
    if not O.ref_available():
        O.build()
    make_alloc()
    make_attn()
    make_prefill()
    for f in ("alloc_golden.npz", "attn_golden.npz", "prefill_golden.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")

"""Multi-GPU host logic on CPU (gloo, world size 2): placement -> per-rank roles, the
head-sharded (tp>1) service path whose only collective is the output AllReduce,
and the determinism that lets every TP rank replay the allocator without
communication.  Attention is computed by the fp32 oracle here (no GPU); on a
GPU the same HeadShardedDecode drives Batch.decode and NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_py as O
from paper_2504_15720_b200 import placement as PL
from paper_2504_15720_b200.tp import HeadShardedDecode, head_slice


def test_placement_reproduces_reference_default_outcomes():
    """SURVEY §8e (measured with the reference dedicated_plan): 16 services, share_cap 2,
    80 GiB GPUs: 4 GPUs -> 1 group + 14 unplaced; 8 GPUs -> 5 groups + 6 unplaced."""
    svcs = PL.config5_services()
    p4 = PL.dedicated_plan(svcs, PL.PlacementConfig(share_cap=2, gpus_per_node=4, gpu_mem_gib=80.0))
    assert (len(p4.groups), len(p4.unplaced)) == (1, 14) and p4.groups[0].tp_size == 4
    p8 = PL.dedicated_plan(svcs, PL.PlacementConfig(share_cap=2, gpus_per_node=8, gpu_mem_gib=80.0))
    assert (len(p8.groups), len(p8.unplaced)) == (5, 6)


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_config5_overrides_place_everything(n):
    plan = PL.dedicated_plan(PL.config5_services(), PL.config5_overrides(n))
    assert plan.feasible and not plan.unplaced
    seen = [gpu for g in plan.groups for gpu in g.gpu_ids]
    assert sorted(seen) == list(range(len(seen))) and len(seen) <= n
    big = [g for g in plan.groups if 0 in g.services][0]
    assert big.tp_size == min(n, 4)  # the 70B-shape service is head-sharded
    for r in range(len(seen)):
        role = PL.rank_role(plan, r)
        assert role is not None and role.group.gpu_ids[role.tp_rank] == r


def test_required_tp_follows_reference_rules():
    cfg = PL.PlacementConfig()
    assert PL.required_tp(PL.MODELS["llama2-70b"], cfg) == 4
    assert PL.required_tp(PL.MODELS["llama3-8b"], cfg) == 1
    with pytest.raises(RuntimeError):
        PL.required_tp(PL.MODELS["llama2-70b"], PL.PlacementConfig(gpus_per_node=2))


# --------------------------------------------------------------------------- TP decode ---
L, H, HQ, D, HID = 2, 8, 16, 128, 256
SMALL = (2, 4, 4)  # a second service sharing the head-sharded group's pool
CTX = [37, 100, 16, 250]


def _kv(rid, layer):
    rng = np.random.default_rng(1000 * rid + layer)
    return (rng.standard_normal((max(CTX) + 1, H, 2, D)) * 0.5).astype(np.float16)


def _pool(tp, tp_rank):
    """Oracle allocator + host pool image holding this rank's KV heads."""
    models = [(L, H, D, 2), (SMALL[0], SMALL[1], D, 2)]
    cache = O.OracleCache(models, pool=128, tp=tp)
    for i, c in enumerate(CTX):
        assert cache.try_allocate(i + 1, 0, c)
        assert cache.try_allocate(100 + i, 1, 3 * c + 5)
    merged = int(cache.merged_block_bytes())
    stride = (merged + 255) // 256 * 256
    hl = H // tp
    lay = O.layout(stride, L * hl * 2 * 16 * D * 2, hl * 2 * 16 * D * 2, 2 * 16 * D * 2, 16 * D * 2, 16, D, hl,
                   HQ // tp, L, 0)
    img = np.zeros(128 * stride, np.uint8)
    hs = head_slice(H, tp, tp_rank)
    for i, c in enumerate(CTX):
        tab = cache.block_table_np(i + 1)[None]
        for layer in range(L):
            kv = _kv(i + 1, layer)[:c, hs]
            O.append(lay, img, layer, tab, np.zeros(1, np.int64), kv[None, :, :, 0].view(np.uint16),
                     kv[None, :, :, 1].view(np.uint16))
    return cache, lay, img


def _attend_fn(cache, lay, img):
    def attend(q_local, out_local, layer):
        tabs = np.stack([np.pad(cache.block_table_np(i + 1), ((0, 32 - len(cache.block_table_np(i + 1))), (0, 0)))
                         for i in range(len(CTX))])
        out = O.decode_attention(lay, img, layer, tabs, np.array(CTX, np.int64),
                                 q_local.contiguous().view(torch.int16).numpy().view(np.uint16), 1 / np.sqrt(D))
        out_local.copy_(torch.from_numpy(out).to(out_local.dtype))
    return attend


def _inputs():
    g = torch.Generator().manual_seed(7)
    q = torch.randn((len(CTX), HQ, D), generator=g).half()
    w_o = torch.randn((HQ * D, HID), generator=g) / 32
    return q, w_o


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _work(rank, world, out_q)
    except Exception as e:  # surface worker failures to the parent immediately
        import traceback
        out_q.put((rank, "error", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _work(rank, world, out_q):
    if True:
        cache, lay, img = _pool(world, rank)
        # allocator determinism: every TP rank derives the same tables without communicating
        tabs = [cache.block_table(i + 1) for i in range(len(CTX))] + [cache.block_table(100 + i) for i in range(len(CTX))]
        allt = [None] * world
        dist.all_gather_object(allt, tabs)
        assert all(t == allt[0] for t in allt)
        q, w_o = _inputs()
        step = HeadShardedDecode(w_o, HQ, D, world, rank, attend=_attend_fn(cache, lay, img))
        q_local = q[:, step.q_heads].contiguous()
        ys = [step(q_local, layer).numpy() for layer in range(L)]
        out_q.put((rank, tabs, ys))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_head_sharded_decode_allreduce_matches_unsharded_gloo():
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out_q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(2):
        rank, tabs, ys = out_q.get(timeout=180)
        assert tabs != "error", ys
        res[rank] = (tabs, ys)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # unsharded reference (tp=1, all heads in one pool)
    cache, lay, img = _pool(1, 0)
    full_tabs = [cache.block_table(i + 1) for i in range(len(CTX))] + [cache.block_table(100 + i) for i in range(len(CTX))]
    assert res[0][0] == full_tabs  # tables are tp-invariant (kv_cache.hpp:20-21)
    q, w_o = _inputs()
    full = HeadShardedDecode(w_o, HQ, D, 1, 0, attend=_attend_fn(cache, lay, img))
    for layer in range(L):
        y_full = full(q, layer).numpy()
        for r in range(2):
            np.testing.assert_allclose(res[r][1][layer], y_full, rtol=1e-4, atol=1e-4)

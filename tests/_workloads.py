"""Seeded KvOp streams shared by the oracle differ and the GPU parity tests.

Op tuple: (kind, request_id, model, tokens) with kind 0 = kGrow (grow the
request to cover `tokens` in total), 1 = kFree — the KvOp record of
kv_cache.hpp:270-275."""
from _rng import Rng

GROW, FREE = 0, 1


def property_stream(seed=2024, steps=100000, n_models=2):
    """The op sequence of kv_cache_test.cpp:124-158 (seed 2024) with the
    reference's own control flow; `live` tracks what the reference test
    tracks.  Needs the allocator's answers, so it is a generator that is
    sent the grant result of each grow."""
    rng = Rng(seed)
    live = {}  # id -> (model, tokens)
    next_id = 1
    for _ in range(steps):
        do_alloc = (not live) or rng.next_double() < 0.6
        if do_alloc:
            grow_existing = bool(live) and rng.next_double() < 0.5
            if grow_existing:
                ids = sorted(live)
                rid = ids[rng.next_below(len(ids))]
                mi, tok = live[rid]
                tokens = tok + 1 + rng.next_below(40)
            else:
                rid = next_id
                next_id += 1
                mi = rng.next_below(n_models)
                tokens = 1 + rng.next_below(64)
            granted = yield (GROW, rid, mi, tokens)
            if granted:
                live[rid] = (mi, tokens)
        else:
            ids = sorted(live)
            rid = ids[rng.next_below(len(ids))]
            yield (FREE, rid, 0, 0)
            del live[rid]
    return live


def random_stream(seed, n_ops, n_models, max_live=64, max_grow=48, p_free=0.35, first_id=1):
    """Grant-independent churn stream (frees only target ids known to be live
    in the reference semantics is NOT required: a failed grow still registers
    the id (Q3), so freeing any id that was ever grown is legal)."""
    rng = Rng(seed)
    known = {}  # id -> (model, tokens requested so far)
    order = []
    next_id = first_id
    ops = []
    for _ in range(n_ops):
        if known and (rng.next_double() < p_free or len(known) >= max_live):
            rid = order[rng.next_below(len(order))]
            ops.append((FREE, rid, 0, 0))
            del known[rid]
            order.remove(rid)
        elif known and rng.next_double() < 0.5:
            rid = order[rng.next_below(len(order))]
            m, tok = known[rid]
            tok += 1 + rng.next_below(max_grow)
            known[rid] = (m, tok)
            ops.append((GROW, rid, m, tok))
        else:
            rid = next_id
            next_id += 1
            m = rng.next_below(n_models)
            tok = rng.next_below(4 * max_grow)
            known[rid] = (m, tok)
            order.append(rid)
            ops.append((GROW, rid, m, tok))
    return ops

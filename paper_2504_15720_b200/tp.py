"""Head-sharded (tensor-parallel) services on the unified pool — row N4 of SURVEY §8.

A tp>1 sharing group (e.g. the 70B-shape service at tp=4) keeps ONE pool per rank
with ``tp_size=tp``: native and merged block bytes scale by 1/tp
(kv_cache.hpp:20-21), so sub-slot counts — and therefore every block table — are
identical on all ranks of the group when they replay the same op stream; the
allocator needs no communication.  Each rank attends its Hq/tp query heads over
its Hkv/tp KV heads, multiplies by its row slice of the output projection, and
the only collective of the data path is the AllReduce(sum) of that partial
output (NCCL over NVLink on the GPU; gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist


def head_slice(n_heads: int, tp: int, tp_rank: int) -> slice:
    if n_heads % tp:
        raise ValueError(f"tp={tp} does not divide {n_heads} heads")
    per = n_heads // tp
    return slice(tp_rank * per, (tp_rank + 1) * per)


class HeadShardedDecode:
    """One decode layer of a head-sharded service: local paged attention over this
    rank's heads, row-parallel output projection, AllReduce of the partial output.

    ``attend(q_local, out_local, layer)`` runs the attention for this rank's heads —
    ``Batch.decode`` on the GPU (the product path); the CPU tests inject the oracle.
    """

    def __init__(self, w_o: torch.Tensor, num_q_heads: int, head_dim: int, tp: int, tp_rank: int,
                 group: Optional[dist.ProcessGroup] = None,
                 attend: Optional[Callable[[torch.Tensor, torch.Tensor, int], None]] = None):
        hs = head_slice(num_q_heads, tp, tp_rank)
        self.q_heads = slice(hs.start, hs.stop)
        rows = slice(hs.start * head_dim, hs.stop * head_dim)
        self.w_o = w_o[rows].contiguous()  # [Hq/tp * d, hidden] row slice of W_o
        self.tp, self.tp_rank, self.group = tp, tp_rank, group
        self.head_dim = head_dim
        self.attend = attend

    def partial(self, q_local: torch.Tensor, layer: int, out_local: Optional[torch.Tensor] = None) -> torch.Tensor:
        if out_local is None:
            out_local = torch.empty_like(q_local)
        self.attend(q_local, out_local, layer)
        b = q_local.shape[0]
        return out_local.reshape(b, -1).to(self.w_o.dtype) @ self.w_o

    def __call__(self, q_local: torch.Tensor, layer: int, out_local: Optional[torch.Tensor] = None) -> torch.Tensor:
        y = self.partial(q_local, layer, out_local)
        if self.tp > 1:
            dist.all_reduce(y, op=dist.ReduceOp.SUM, group=self.group)
        return y


def gpu_attend(batch, group_index: int, n_groups: int):
    """Adapter: attention of one service (batch group ``group_index``) through the
    unified-pool decode kernel."""
    def attend(q_local, out_local, layer):
        qs = [None] * n_groups
        os_ = [None] * n_groups
        qs[group_index], os_[group_index] = q_local, out_local
        for i in range(n_groups):
            if qs[i] is None:
                raise ValueError("gpu_attend drives single-group batches")
        batch.decode(qs, os_, layer)
    return attend

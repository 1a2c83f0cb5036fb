"""Data parallelism over prompt groups.

Prompt groups are independent units of DualKV attention: a GPU owns whole
groups (co-location contract, packing.py:191-198 / pipeline.py:130-145 of the
reference), so no collective ever runs inside attention.  The only exchange
is the sum of parameter gradients across ranks after the backward -- the
step gradient is the sum over cells (pipeline.py:147-158), exact by the
pipeline theorem (verify.py:522-533).

* `lpt_assign` deals whole groups to ranks longest-processing-time first,
  with the exact visible-pair count as the cost (ragged C4 responses).
* `GradSync` flattens parameter gradients into buckets and all-reduces them
  (NCCL over NVLink/NVSwitch on the GPU box; gloo in the CPU tests).
"""

from __future__ import annotations

import heapq
from typing import Dict, List, Sequence, Tuple

import torch
import torch.distributed as dist

from .costmodel import visible_pairs

__all__ = ["group_cost", "lpt_assign", "GradSync"]


def group_cost(p_len: int, r_list: Sequence[int]) -> int:
    """Work of one group's Call 1 + Call 2 (visible pairs; FLOPs are proportional)."""
    return visible_pairs(p_len, r_list, "dualkv")


def lpt_assign(costs: Sequence[int], world: int) -> List[List[int]]:
    """Whole groups -> ranks, largest first onto the least-loaded rank (ties: lowest rank)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    heap = [(0, r) for r in range(world)]
    heapq.heapify(heap)
    out: List[List[int]] = [[] for _ in range(world)]
    for gi in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        load, r = heapq.heappop(heap)
        out[r].append(gi)
        heapq.heappush(heap, (load + int(costs[gi]), r))
    for lst in out:
        lst.sort()
    return out


class GradSync:
    """Bucketed sum all-reduce of parameter gradients (the step's only collective)."""

    def __init__(self, params: Sequence[torch.Tensor], bucket_bytes: int = 64 << 20, group=None):
        self.params = [p for p in params if p.requires_grad]
        self.group = group
        self.buckets: List[List[torch.Tensor]] = []
        cur, size = [], 0
        for p in self.params:
            nbytes = p.numel() * p.element_size()
            if cur and size + nbytes > bucket_bytes:
                self.buckets.append(cur)
                cur, size = [], 0
            cur.append(p)
            size += nbytes
        if cur:
            self.buckets.append(cur)

    def sync(self, average: bool = False) -> None:
        if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(self.group) == 1:
            return
        world = dist.get_world_size(self.group)
        for bucket in self.buckets:
            grads = [p.grad if p.grad is not None else torch.zeros_like(p) for p in bucket]
            flat = torch.cat([g.reshape(-1) for g in grads])
            dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=self.group)
            if average:
                flat /= world
            off = 0
            for p, g in zip(bucket, grads):
                n = g.numel()
                chunk = flat[off:off + n].view_as(g)
                if p.grad is None:
                    p.grad = chunk.clone()
                else:
                    p.grad.copy_(chunk)
                off += n

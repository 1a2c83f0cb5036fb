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
    """Bucketed sum all-reduce of parameter gradients (the step's only collective).

    * Buckets are reduced in fp32 (or the parameter dtype when wider) and cast back ONCE into
      `p.grad` -- a bf16 reduction would round the cross-rank sum at every hop; the reference sums
      per-cell gradients in float64 (pipeline.py:147-158).
    * `overlap=True` launches a bucket's all-reduce from the autograd engine as soon as the last
      gradient of that bucket is accumulated (post-accumulate-grad hooks), so NCCL runs on its
      own stream under the rest of the backward; `sync()` then only waits.  Inside `no_sync()`
      (gradient accumulation over micro-batches) the hooks stay idle.
    """

    def __init__(self, params: Sequence[torch.Tensor], bucket_bytes: int = 64 << 20, group=None,
                 overlap: bool = False):
        self.params = [p for p in params if p.requires_grad]
        self.group = group
        self.buckets: List[List[torch.Tensor]] = []
        cur, size = [], 0
        for p in self.params:
            nbytes = p.numel() * max(4, p.element_size())
            if cur and size + nbytes > bucket_bytes:
                self.buckets.append(cur)
                cur, size = [], 0
            cur.append(p)
            size += nbytes
        if cur:
            self.buckets.append(cur)
        self._bucket_of = {id(p): b for b, bucket in enumerate(self.buckets) for p in bucket}
        self._ready = [0] * len(self.buckets)
        self._pending: Dict[int, Tuple[object, torch.Tensor]] = {}
        self._hooks_on = True
        self._handles = []
        if overlap:
            for p in self.params:
                self._handles.append(p.register_post_accumulate_grad_hook(self._on_grad))

    def _distributed(self) -> bool:
        return dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1

    def _on_grad(self, p: torch.Tensor) -> None:
        if not self._hooks_on or not self._distributed():
            return
        b = self._bucket_of[id(p)]
        self._ready[b] += 1
        if self._ready[b] == len(self.buckets[b]) and b not in self._pending:
            self._launch(b)

    def _launch(self, b: int) -> None:
        bucket = self.buckets[b]
        acc = torch.float64 if any(p.dtype == torch.float64 for p in bucket) else torch.float32
        flat = torch.cat([(p.grad if p.grad is not None else torch.zeros_like(p)).reshape(-1).to(acc)
                          for p in bucket])
        work = dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
        self._pending[b] = (work, flat)

    class _NoSync:
        def __init__(self, owner):
            self.owner = owner

        def __enter__(self):
            self.owner._hooks_on = False

        def __exit__(self, *exc):
            self.owner._hooks_on = True

    def no_sync(self):
        """Accumulate gradients locally (earlier micro-batches); the last backward syncs."""
        return GradSync._NoSync(self)

    def sync(self, average: bool = False) -> None:
        if not self._distributed():
            self._ready = [0] * len(self.buckets)
            return
        world = dist.get_world_size(self.group)
        for b in range(len(self.buckets)):
            if b not in self._pending:
                self._launch(b)
        for b in sorted(self._pending):
            work, flat = self._pending[b]
            work.wait()
            if average:
                flat /= world
            off = 0
            for p in self.buckets[b]:
                n = p.numel()
                chunk = flat[off:off + n].view(p.shape).to(p.dtype)  # the single cast back
                if p.grad is None:
                    p.grad = chunk
                else:
                    p.grad.copy_(chunk)
                off += n
        self._pending.clear()
        self._ready = [0] * len(self.buckets)

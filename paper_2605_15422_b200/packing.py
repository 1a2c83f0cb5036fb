"""Device-side repack between the replicated layout N(P+R) and the shared
DualKV layout P+NR (packing.py:159-220 of the reference, as a data-movement
op on activations instead of host token lists).

The layout metadata (prompt length and response lengths per group) is tiny
host data; the O(tokens) row-index maps are built once per layout with
numpy and uploaded, and the bytes move on the GPU through the C ABI
(`dkv_gather_rows`, `dkv_segment_sum_rows`), HBM-bound and vectorised.

Row conventions (all row-major, any trailing shape):
  replicated : per group g, per response i: [prompt_g ; response_{g,i}]
  shared     : per group g: [prompt_g ; response_{g,1} ; ... ; response_{g,N_g}]
Logical positions: prompt token j -> j, response token r -> P_g + r
(`PackedBatch.position_ids`, packing.py:105-120).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np
import torch

from ._lib import DKV_BF16, DKV_F32, check, lib

__all__ = ["GroupLayout", "PackPlan", "make_plan", "repack_to_dualkv", "broadcast_to_standard",
           "reduce_to_dualkv", "position_ids"]


@dataclass
class GroupLayout:
    """One group's rows in both layouts (packing.py:69-86)."""

    prompt_len: int
    resp_lens: List[int]
    seq_cu: np.ndarray        # replicated layout: global offsets of the N sequences (N+1)
    context_start: int        # shared layout
    resp_start: int
    resp_cu: np.ndarray       # shared layout, group-local response offsets (N+1)


@dataclass
class PackPlan:
    groups: List[GroupLayout]
    total_standard: int
    total_dualkv: int
    dk_from_std: np.ndarray    # [T_dk]  source row in the replicated layout (prompt from copy 0)
    std_from_dk: np.ndarray    # [T_std] source row in the shared layout
    seg: np.ndarray            # [T_dk+1] CSR offsets of the adjoint (sum over prompt copies)
    seg_src: np.ndarray        # [T_std] replicated rows summed into each shared row
    _dev: dict = field(default_factory=dict, repr=False)

    def device(self, name: str, dev) -> torch.Tensor:
        key = (name, str(dev))
        if key not in self._dev:
            self._dev[key] = torch.as_tensor(getattr(self, name), dtype=torch.int64, device=dev)
        return self._dev[key]

    def cu_seqlens_standard(self) -> np.ndarray:
        cu = [0]
        for g in self.groups:
            cu.extend(int(x) for x in g.seq_cu[1:])
        return np.asarray(cu, dtype=np.int64)


def make_plan(groups: Sequence[Tuple[int, Sequence[int]]]) -> PackPlan:
    """Layouts + index maps for [(P_g, [R_g1, ..., R_gN]), ...]."""
    if not groups:
        raise ValueError("cannot pack an empty group list")
    layouts, dk_from_std, std_from_dk = [], [], []
    seg_lens, seg_src = [], []
    std_cur = dk_cur = 0
    for p_len, rs in groups:
        p_len = int(p_len)
        rs = [int(r) for r in rs]
        if p_len < 0 or any(r < 0 for r in rs):
            raise ValueError("negative length")
        if not rs:
            # the reference rejects a rollout group with no responses (RolloutGroup.__post_init__);
            # its prompt rows would otherwise have no copy to come from
            raise ValueError("a prompt group needs at least one response")
        seq_cu = np.concatenate([[0], np.cumsum([p_len + r for r in rs])]).astype(np.int64) + std_cur
        resp_cu = np.concatenate([[0], np.cumsum(rs)]).astype(np.int64)
        ctx0, rs0 = dk_cur, dk_cur + p_len
        starts = seq_cu[:-1]
        # shared <- replicated (prompt from copy 0)
        if rs:
            dk_from_std.append(starts[0] + np.arange(p_len))
        for st, r in zip(starts, rs):
            dk_from_std.append(st + p_len + np.arange(r))
        # replicated <- shared (broadcast the single prompt copy)
        for i, (st, r) in enumerate(zip(starts, rs)):
            std_from_dk.append(ctx0 + np.arange(p_len))
            std_from_dk.append(rs0 + resp_cu[i] + np.arange(r))
        # adjoint: prompt row j sums the N copies, response rows copy through
        if rs:
            seg_lens.extend([len(rs)] * p_len)
            seg_src.append((starts[:, None] + np.arange(p_len)[None, :]).T.reshape(-1))
        for st, r in zip(starts, rs):
            seg_lens.extend([1] * r)
            seg_src.append(st + p_len + np.arange(r))
        layouts.append(GroupLayout(p_len, rs, seq_cu, ctx0, rs0, resp_cu))
        std_cur = int(seq_cu[-1])
        dk_cur = rs0 + int(resp_cu[-1]) if rs else dk_cur
    cat = lambda xs: np.concatenate(xs).astype(np.int64) if xs else np.zeros(0, np.int64)
    return PackPlan(layouts, std_cur, dk_cur, cat(dk_from_std), cat(std_from_dk),
                    np.concatenate([[0], np.cumsum(seg_lens)]).astype(np.int64), cat(seg_src))


def _stream(device):
    return torch.cuda.current_stream(device).cuda_stream


def _gather(x: torch.Tensor, idx: torch.Tensor, n_out: int) -> torch.Tensor:
    x = x.contiguous()
    out = torch.empty((n_out,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    row_bytes = x[0].numel() * x.element_size() if x.shape[0] else 0
    if n_out and row_bytes:
        with torch.cuda.device(x.device):
            check(lib.dkv_gather_rows(x.data_ptr(), out.data_ptr(), row_bytes, idx.data_ptr(), n_out,
                                      _stream(x.device)), "gather_rows")
    return out


def repack_to_dualkv(x_std: torch.Tensor, plan: PackPlan) -> torch.Tensor:
    """[T_std, ...] replicated activations -> [T_dk, ...] shared layout (prompt from copy 0)."""
    if x_std.shape[0] != plan.total_standard:
        raise ValueError(f"expected {plan.total_standard} rows, got {x_std.shape[0]}")
    return _gather(x_std, plan.device("dk_from_std", x_std.device), plan.total_dualkv)


def broadcast_to_standard(x_dk: torch.Tensor, plan: PackPlan) -> torch.Tensor:
    """[T_dk, ...] -> [T_std, ...]: the prompt copy is broadcast to every response."""
    if x_dk.shape[0] != plan.total_dualkv:
        raise ValueError(f"expected {plan.total_dualkv} rows, got {x_dk.shape[0]}")
    return _gather(x_dk, plan.device("std_from_dk", x_dk.device), plan.total_standard)


def reduce_to_dualkv(g_std: torch.Tensor, plan: PackPlan) -> torch.Tensor:
    """Adjoint of `broadcast_to_standard`: prompt rows sum their N copies (fp32 accumulate)."""
    if g_std.shape[0] != plan.total_standard:
        raise ValueError(f"expected {plan.total_standard} rows, got {g_std.shape[0]}")
    if g_std.dtype not in (torch.bfloat16, torch.float32):
        raise ValueError("reduce_to_dualkv supports bf16 / fp32")
    g_std = g_std.contiguous()
    out = torch.empty((plan.total_dualkv,) + tuple(g_std.shape[1:]), dtype=g_std.dtype, device=g_std.device)
    row = g_std[0].numel() if g_std.shape[0] else 0
    if plan.total_dualkv and row:
        with torch.cuda.device(g_std.device):
            check(lib.dkv_segment_sum_rows(
                g_std.data_ptr(), out.data_ptr(), DKV_F32 if g_std.dtype == torch.float32 else DKV_BF16, row,
                plan.device("seg", g_std.device).data_ptr(), plan.device("seg_src", g_std.device).data_ptr(),
                plan.total_dualkv, _stream(g_std.device)), "segment_sum_rows")
    return out


def position_ids(plan: PackPlan, mode: str = "dualkv") -> np.ndarray:
    """Logical positions of every packed row (packing.py:105-120)."""
    pos = []
    for g in plan.groups:
        if mode == "dualkv":
            pos.append(np.arange(g.prompt_len))
            for r in g.resp_lens:
                pos.append(g.prompt_len + np.arange(r))
        else:
            for r in g.resp_lens:
                pos.append(np.arange(g.prompt_len + r))
    return np.concatenate(pos).astype(np.int64) if pos else np.zeros(0, np.int64)

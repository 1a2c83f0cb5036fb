"""The attention block around the DualKV op, in the P+NR layout (the reference's
`_attn_dualkv_fwd/_bwd`, layer.py:236-290, inside `model_fwd`'s per-layer block, layer.py:318-325).

`DualKVSelfAttention` is what a trainer swaps in (the paper's veRL monkey-patch installs the same
call on supported model classes): QKV projections run once per prompt token (plain
library GEMMs on the P+NR rows -- the rho saving), Qwen3's per-head RMSNorm of q and k (optional,
`qk_norm=True`; the reference toy model has none), RoPE rotates rows at their LOGICAL
positions (prompt j -> j, response r -> P + r), and ALL prompt groups of the micro-batch run in ONE
fused two-call launch (Call 1 over every prompt, Call 2 over every response, each group's prompt
K/V gradient accumulated in fp32 and cast once) -- the reference loops over groups
(layer.py:239).  Every device op is a registered torch.library op, so the block compiles with
`torch.compile(fullgraph=True)`; parameter gradients are what `dp.GradSync` all-reduces.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Union

import numpy as np
import torch

from . import library  # noqa: F401  (registers the dualkv:: ops)
from ._lib import DKV_MAX_GROUPS
from .packing import PackPlan, position_ids

__all__ = ["DualKVSelfAttention", "DualKVBatch"]


@dataclass
class DualKVBatch:
    """Device metadata of one P+NR micro-batch, built once per layout (outside any compiled region).

    The packed rows keep the reference layout (per group [prompt; responses], packing.py:182-220);
    the single launch takes every prompt and every response as two contiguous row sets, picked
    with `ctx_rows` / `resp_rows` and put back with `inv_perm`."""

    total: int
    positions: torch.Tensor   # [T_dk] int64 logical positions (packing.py:105-120)
    ctx_rows: torch.Tensor    # [sum P_g] int64 packed rows of the prompts, group order
    resp_rows: torch.Tensor   # [sum R] int64 packed rows of the responses
    inv_perm: torch.Tensor    # [T_dk] int64: row of cat(prompts, responses) holding packed row i
    perm: torch.Tensor        # [T_dk] int64: its inverse, packed row held at cat(...) row j
    cu_seqlens: torch.Tensor  # [N+1] int32 response offsets over all groups
    max_seqlen: int
    group_seq_cu: List[int]
    group_ctx_cu: List[int]

    @staticmethod
    def from_plan(plan: PackPlan, device) -> "DualKVBatch":
        key = ("dualkv_batch", str(device))
        if key in plan._dev:
            return plan._dev[key]
        if len(plan.groups) > DKV_MAX_GROUPS:
            raise ValueError(f"at most {DKV_MAX_GROUPS} prompt groups per launch")
        ctx_rows, resp_rows, lens, gs, gc = [], [], [], [0], [0]
        for g in plan.groups:
            ctx_rows.append(g.context_start + np.arange(g.prompt_len))
            resp_rows.append(g.resp_start + np.arange(int(g.resp_cu[-1])))
            lens.extend(int(r) for r in g.resp_lens)
            gs.append(gs[-1] + len(g.resp_lens))
            gc.append(gc[-1] + g.prompt_len)
        ctx_rows = np.concatenate(ctx_rows).astype(np.int64)
        resp_rows = np.concatenate(resp_rows).astype(np.int64)
        order = np.concatenate([ctx_rows, resp_rows])
        inv = np.empty_like(order)
        inv[order] = np.arange(order.size)
        cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        t = lambda a, dt=torch.int64: torch.as_tensor(a, dtype=dt, device=device)
        b = DualKVBatch(plan.total_dualkv, t(position_ids(plan, "dualkv")), t(ctx_rows), t(resp_rows), t(inv),
                        t(order), t(cu, torch.int32), int(max(lens)) if lens else 0, gs, gc)
        plan._dev[key] = b
        return b


def _rms_norm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    """Per-head RMSNorm over head_dim (Qwen3 q_norm / k_norm), fp32 statistics -- the unfused torch
    composition the fused `dualkv::qkv_prep` kernel is tested against."""
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps) * w.float()).to(x.dtype)


class DualKVSelfAttention(torch.nn.Module):
    def __init__(self, d_model: int, heads: int, kv_heads: int, head_dim: int, rope_base: float = 10000.0,
                 dtype=torch.bfloat16, device="cuda", qk_norm: bool = False, eps: float = 1e-6):
        super().__init__()
        if heads % kv_heads:
            raise ValueError("heads must be a multiple of kv_heads")
        self.h, self.hk, self.d, self.base, self.eps = heads, kv_heads, head_dim, float(rope_base), eps
        self.scale = 1.0 / math.sqrt(head_dim)
        mk = lambda i, o: torch.nn.Parameter(
            (torch.randn(i, o, device=device) / math.sqrt(i)).to(dtype))
        # one [d_model, (H + 2 H_k) d] projection: a single GEMM whose output rows feed the fused
        # norm + RoPE + split epilogue
        self.w_qkv = mk(d_model, (heads + 2 * kv_heads) * head_dim)
        self.w_o = mk(heads * head_dim, d_model)
        self.qk_norm = qk_norm
        if qk_norm:
            self.q_norm = torch.nn.Parameter(torch.ones(head_dim, device=device, dtype=dtype))
            self.k_norm = torch.nn.Parameter(torch.ones(head_dim, device=device, dtype=dtype))

    # column views of the fused projection (W_Q, W_K, W_V of the reference block)
    @property
    def w_q(self):
        return self.w_qkv[:, :self.h * self.d]

    @property
    def w_k(self):
        return self.w_qkv[:, self.h * self.d:(self.h + self.hk) * self.d]

    @property
    def w_v(self):
        return self.w_qkv[:, (self.h + self.hk) * self.d:]

    def forward(self, x: torch.Tensor, batch: Union[DualKVBatch, PackPlan]) -> torch.Tensor:
        """x: [T_dk, d_model] hidden states of the P+NR rows; returns the block's output projection
        [T_dk, d_model] (no residual)."""
        if isinstance(batch, PackPlan):
            batch = DualKVBatch.from_plan(batch, x.device)
        if x.shape[0] != batch.total:
            raise ValueError(f"expected {batch.total} rows, got {x.shape[0]}")
        t = x.shape[0]
        qkv = x @ self.w_qkv
        # fused epilogue: q/k RMSNorm, RoPE at logical positions, scatter to [all prompts; all responses]
        q, k, v = torch.ops.dualkv.qkv_prep(qkv, self.q_norm if self.qk_norm else None,
                                            self.k_norm if self.qk_norm else None, batch.positions,
                                            batch.inv_perm, self.h, self.hk, self.eps, self.base)
        # every group's Call 1 + Call 2, one forward and one backward launch, on the split layout
        o, _, _ = torch.ops.dualkv.two_call_split(q, k, v, batch.ctx_rows.shape[0], batch.cu_seqlens,
                                                  batch.max_seqlen, self.scale, batch.group_seq_cu,
                                                  batch.group_ctx_cu)
        # back to the packed row order (a permutation: gather forward, gather by the inverse backward)
        return library.permute_rows(o, batch.inv_perm, batch.perm).reshape(t, self.h * self.d) @ self.w_o

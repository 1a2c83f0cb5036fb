"""The attention block around the DualKV op, in the P+NR layout (the reference's
`_attn_dualkv_fwd/_bwd`, layer.py:236-290, inside `model_fwd`'s per-layer block, layer.py:318-325).

`DualKVSelfAttention` is what a trainer swaps in (the paper's veRL monkey-patch installs the same
call on supported model classes): QKV projections run once per prompt token (plain
library GEMMs on the P+NR rows -- the rho saving), RoPE rotates rows at their LOGICAL positions
(prompt j -> j, response r -> P + r), and each prompt group runs the fused two-call op (Call 1
over the prompt, Call 2 over the responses, one fp32 prompt-KV gradient cast once).  Autograd
covers the whole block; parameter gradients are what `dp.GradSync` all-reduces.
"""

from __future__ import annotations

import math

import torch

from .api import dualkv_two_call_attention
from .packing import PackPlan
from .rope import RoPE, dualkv_positions

__all__ = ["DualKVSelfAttention"]


class DualKVSelfAttention(torch.nn.Module):
    def __init__(self, d_model: int, heads: int, kv_heads: int, head_dim: int, rope_base: float = 10000.0,
                 dtype=torch.bfloat16, device="cuda"):
        super().__init__()
        if heads % kv_heads:
            raise ValueError("heads must be a multiple of kv_heads")
        self.h, self.hk, self.d, self.base = heads, kv_heads, head_dim, rope_base
        mk = lambda i, o: torch.nn.Parameter(
            (torch.randn(i, o, device=device) / math.sqrt(i)).to(dtype))
        self.w_q, self.w_k, self.w_v = mk(d_model, heads * head_dim), mk(d_model, kv_heads * head_dim), \
            mk(d_model, kv_heads * head_dim)
        self.w_o = mk(heads * head_dim, d_model)

    def forward(self, x: torch.Tensor, plan: PackPlan) -> torch.Tensor:
        """x: [T_dk, d_model] hidden states of the P+NR rows of `plan`; returns the block's output
        projection [T_dk, d_model] (no residual)."""
        if x.shape[0] != plan.total_dualkv:
            raise ValueError(f"expected {plan.total_dualkv} rows, got {x.shape[0]}")
        t = x.shape[0]
        pos = dualkv_positions(plan, x.device)
        q = RoPE.apply((x @ self.w_q).view(t, self.h, self.d), pos, self.base)
        k = RoPE.apply((x @ self.w_k).view(t, self.hk, self.d), pos, self.base)
        v = (x @ self.w_v).view(t, self.hk, self.d)
        outs = []
        for g in plan.groups:
            c0, c1 = g.context_start, g.context_start + g.prompt_len
            r0, r1 = g.resp_start, g.resp_start + int(g.resp_cu[-1])
            if g.prompt_len == 0 or r1 == r0:
                raise ValueError("DualKVSelfAttention needs P > 0 and at least one response token per group")
            oc, od = dualkv_two_call_attention(q[c0:c1], k[c0:c1], v[c0:c1], q[r0:r1], k[r0:r1], v[r0:r1],
                                               g.resp_cu)
            outs += [oc, od]
        o = torch.cat(outs, dim=0).reshape(t, self.h * self.d)
        return o @ self.w_o

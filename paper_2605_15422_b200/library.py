"""The DualKV ops registered with `torch.library` (namespace ``dualkv``).

The paper ships its kernel as a `torch.autograd.Function` (the
reference's five-tensor surface kernel.py:308-348); here every entry point is a
registered custom op with a fake (meta) implementation and a registered autograd
formula, so `torch.compile(fullgraph=True)` traces through models that use it
(the op stays one opaque node, launched through the C ABI at run time):

  dualkv::fwd / dualkv::bwd                 five-tensor two-region op (Call 2)
  dualkv::two_call_fwd / dualkv::two_call_bwd   Call 1 + Call 2 in one launch
  dualkv::rope                              RoPE at logical positions (layer.py:182-205)

Offsets travel as a CUDA int32 tensor plus the max sequence length (no host
sync inside the op); the optional group table (several prompt groups in one
launch) as two int lists.  The backward uses the atomic prompt-gradient fold
unless `torch.use_deterministic_algorithms(True)` is set, which selects the
reference's fixed-order fold (kernel.py:250, `deterministic=True`).
"""

from __future__ import annotations

from typing import List, Optional, Tuple

import torch
from torch import Tensor

from . import api
from .api import DualKVInput

__all__ = ["attention", "two_call_attention", "rope"]


def _input(q, kc, vc, kd, vd, cu, max_seqlen, scale, gs, gc) -> DualKVInput:
    return DualKVInput(q, kc, vc, kd, vd, cu, max_seqlen_q=max_seqlen, softmax_scale=scale,
                       group_seq_cu=list(gs) if gs else None, group_ctx_cu=list(gc) if gc else None)


def _lse_like(q: Tensor) -> Tensor:
    return q.new_empty((q.shape[1], q.shape[0]), dtype=torch.float32)


def _deterministic() -> bool:
    return torch.are_deterministic_algorithms_enabled()


# ---------------------------------------------------------------- five-tensor op (Call 2)
@torch.library.custom_op("dualkv::fwd", mutates_args=(), device_types="cuda")
def _fwd(q: Tensor, k_context: Tensor, v_context: Tensor, k_decoded: Tensor, v_decoded: Tensor,
         cu_seqlens: Tensor, max_seqlen: int, softmax_scale: float, group_seq_cu: List[int],
         group_ctx_cu: List[int]) -> Tuple[Tensor, Tensor]:
    return api.dualkv_fwd(_input(q, k_context, v_context, k_decoded, v_decoded, cu_seqlens, max_seqlen,
                                 softmax_scale, group_seq_cu, group_ctx_cu))


@_fwd.register_fake
def _fwd_fake(q, k_context, v_context, k_decoded, v_decoded, cu_seqlens, max_seqlen, softmax_scale,
              group_seq_cu, group_ctx_cu):
    return torch.empty_like(q), _lse_like(q)


@torch.library.custom_op("dualkv::bwd", mutates_args=(), device_types="cuda")
def _bwd(q: Tensor, k_context: Tensor, v_context: Tensor, k_decoded: Tensor, v_decoded: Tensor,
         cu_seqlens: Tensor, max_seqlen: int, softmax_scale: float, group_seq_cu: List[int],
         group_ctx_cu: List[int], out: Tensor, lse: Tensor, d_out: Tensor,
         deterministic: bool) -> Tuple[Tensor, Tensor, Tensor, Tensor, Tensor]:
    inp = _input(q, k_context, v_context, k_decoded, v_decoded, cu_seqlens, max_seqlen, softmax_scale,
                 group_seq_cu, group_ctx_cu)
    return tuple(api.dualkv_bwd(inp, out, lse, d_out, deterministic=deterministic))


@_bwd.register_fake
def _bwd_fake(q, k_context, v_context, k_decoded, v_decoded, cu_seqlens, max_seqlen, softmax_scale,
              group_seq_cu, group_ctx_cu, out, lse, d_out, deterministic):
    return tuple(torch.empty_like(x) for x in (q, k_context, v_context, k_decoded, v_decoded))


def _fwd_setup(ctx, inputs, output):
    q, kc, vc, kd, vd, cu, max_seqlen, scale, gs, gc = inputs
    out, lse = output
    ctx.save_for_backward(q, kc, vc, kd, vd, cu, out, lse)
    ctx.meta = (max_seqlen, scale, gs, gc)
    ctx.mark_non_differentiable(lse)


def _fwd_backward(ctx, d_out, d_lse):
    q, kc, vc, kd, vd, cu, out, lse = ctx.saved_tensors
    max_seqlen, scale, gs, gc = ctx.meta
    d_out = torch.zeros_like(out) if d_out is None else d_out.contiguous()
    grads = torch.ops.dualkv.bwd(q, kc, vc, kd, vd, cu, max_seqlen, scale, gs, gc, out, lse, d_out,
                                 _deterministic())
    return tuple(grads) + (None,) * 5


torch.library.register_autograd("dualkv::fwd", _fwd_backward, setup_context=_fwd_setup)


def _table(inp: DualKVInput) -> Tuple[List[int], List[int]]:
    if inp._groups is None:
        return [], []
    return [int(x) for x in inp._groups[0]], [int(x) for x in inp._groups[1]]


def attention(inp: DualKVInput) -> Tensor:
    """O of the five-tensor op through `dualkv::fwd` (autograd-enabled)."""
    gs, gc = _table(inp)
    out, _ = torch.ops.dualkv.fwd(inp.q, inp.k_context, inp.v_context, inp.k_decoded, inp.v_decoded,
                                  inp.cu_dev, int(inp._grid_max), float(inp.softmax_scale), gs, gc)
    return out


# ---------------------------------------------------------------- two-call op (Call 1 + Call 2)
@torch.library.custom_op("dualkv::two_call_fwd", mutates_args=(), device_types="cuda")
def _two_fwd(q_context: Tensor, k_context: Tensor, v_context: Tensor, q: Tensor, k_decoded: Tensor,
             v_decoded: Tensor, cu_seqlens: Tensor, max_seqlen: int, softmax_scale: float,
             group_seq_cu: List[int], group_ctx_cu: List[int]) -> Tuple[Tensor, Tensor, Tensor, Tensor]:
    inp = _input(q, k_context, v_context, k_decoded, v_decoded, cu_seqlens, max_seqlen, softmax_scale,
                 group_seq_cu, group_ctx_cu)
    return api.dualkv_two_call_fwd(q_context, inp)


@_two_fwd.register_fake
def _two_fwd_fake(q_context, k_context, v_context, q, k_decoded, v_decoded, cu_seqlens, max_seqlen,
                  softmax_scale, group_seq_cu, group_ctx_cu):
    return torch.empty_like(q_context), _lse_like(q_context), torch.empty_like(q), _lse_like(q)


@torch.library.custom_op("dualkv::two_call_bwd", mutates_args=(), device_types="cuda")
def _two_bwd(q_context: Tensor, k_context: Tensor, v_context: Tensor, q: Tensor, k_decoded: Tensor,
             v_decoded: Tensor, cu_seqlens: Tensor, max_seqlen: int, softmax_scale: float,
             group_seq_cu: List[int], group_ctx_cu: List[int], out_context: Tensor, lse_context: Tensor,
             d_out_context: Tensor, out: Tensor, lse: Tensor, d_out: Tensor,
             deterministic: bool) -> Tuple[Tensor, Tensor, Tensor, Tensor, Tensor, Tensor]:
    inp = _input(q, k_context, v_context, k_decoded, v_decoded, cu_seqlens, max_seqlen, softmax_scale,
                 group_seq_cu, group_ctx_cu)
    return tuple(api.dualkv_two_call_bwd(q_context, inp, out_context, lse_context, d_out_context, out, lse,
                                         d_out, deterministic=deterministic))


@_two_bwd.register_fake
def _two_bwd_fake(q_context, k_context, v_context, q, k_decoded, v_decoded, cu_seqlens, max_seqlen,
                  softmax_scale, group_seq_cu, group_ctx_cu, out_context, lse_context, d_out_context, out,
                  lse, d_out, deterministic):
    return tuple(torch.empty_like(x) for x in (q_context, k_context, v_context, q, k_decoded, v_decoded))


def _two_setup(ctx, inputs, output):
    q_c, kc, vc, q, kd, vd, cu, max_seqlen, scale, gs, gc = inputs
    o_c, l_c, o, l = output
    ctx.save_for_backward(q_c, kc, vc, q, kd, vd, cu, o_c, l_c, o, l)
    ctx.meta = (max_seqlen, scale, gs, gc)
    ctx.mark_non_differentiable(l_c, l)


def _two_backward(ctx, d_oc, d_lc, d_o, d_l):
    q_c, kc, vc, q, kd, vd, cu, o_c, l_c, o, l = ctx.saved_tensors
    max_seqlen, scale, gs, gc = ctx.meta
    d_oc = torch.zeros_like(o_c) if d_oc is None else d_oc.contiguous()
    d_o = torch.zeros_like(o) if d_o is None else d_o.contiguous()
    grads = torch.ops.dualkv.two_call_bwd(q_c, kc, vc, q, kd, vd, cu, max_seqlen, scale, gs, gc, o_c, l_c,
                                          d_oc, o, l, d_o, _deterministic())
    return tuple(grads) + (None,) * 5


torch.library.register_autograd("dualkv::two_call_fwd", _two_backward, setup_context=_two_setup)


def two_call_attention(q_context: Tensor, inp: DualKVInput) -> Tuple[Tensor, Tensor]:
    """(O_context, O_decoded) of the fused two-call op through `dualkv::two_call_fwd`."""
    gs, gc = _table(inp)
    o_c, _, o, _ = torch.ops.dualkv.two_call_fwd(q_context, inp.k_context, inp.v_context, inp.q,
                                                 inp.k_decoded, inp.v_decoded, inp.cu_dev, int(inp._grid_max),
                                                 float(inp.softmax_scale), gs, gc)
    return o_c, o


# ---------------------------------------------------------------- RoPE at logical positions
@torch.library.custom_op("dualkv::rope", mutates_args=(), device_types="cuda")
def _rope(x: Tensor, positions: Tensor, base: float, inverse: bool) -> Tensor:
    from .rope import _rope_rows
    return _rope_rows(x, positions, base, inverse)


@_rope.register_fake
def _rope_fake(x, positions, base, inverse):
    return torch.empty_like(x)


def _rope_setup(ctx, inputs, output):
    _, positions, base, inverse = inputs
    ctx.save_for_backward(positions)
    ctx.meta = (base, inverse)


def _rope_backward(ctx, dy):
    (positions,) = ctx.saved_tensors
    base, inverse = ctx.meta
    # the rotation is orthogonal: its adjoint is the inverse rotation (rope_bwd, layer.py:198-205)
    return torch.ops.dualkv.rope(dy.contiguous(), positions, base, not inverse), None, None, None


torch.library.register_autograd("dualkv::rope", _rope_backward, setup_context=_rope_setup)


def rope(x: Tensor, positions: Tensor, base: float = 10000.0) -> Tensor:
    """[T, heads, d] rotated at device int64 `positions` [T] (autograd-enabled)."""
    return torch.ops.dualkv.rope(x, positions, float(base), False)

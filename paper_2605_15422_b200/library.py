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

__all__ = ["attention", "two_call_attention", "rope"]  # + dualkv::qkv_prep (the fused QKV epilogue)


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


# ---------------------------------------------------------------- row permutation
@torch.library.custom_op("dualkv::permute_rows", mutates_args=(), device_types="cuda")
def _permute_rows(x: Tensor, idx: Tensor, inv_idx: Tensor) -> Tensor:
    from .packing import _gather
    return _gather(x, idx, idx.shape[0])


@_permute_rows.register_fake
def _permute_rows_fake(x, idx, inv_idx):
    return x.new_empty((idx.shape[0],) + tuple(x.shape[1:]))


def _permute_setup(ctx, inputs, output):
    _, idx, inv_idx = inputs
    ctx.save_for_backward(idx, inv_idx)


def _permute_backward(ctx, dy):
    idx, inv_idx = ctx.saved_tensors
    # a permutation's adjoint is the inverse permutation: a gather, not index_select's
    # index_add_ backward (30 ms per C4 micro-batch pair in tools/profile_layer.py)
    return torch.ops.dualkv.permute_rows(dy.contiguous(), inv_idx, idx), None, None


torch.library.register_autograd("dualkv::permute_rows", _permute_backward, setup_context=_permute_setup)


def permute_rows(x: Tensor, idx: Tensor, inv_idx: Tensor) -> Tensor:
    """out[i] = x[idx[i]] for a permutation `idx` (device int64) with inverse `inv_idx`."""
    return torch.ops.dualkv.permute_rows(x, idx, inv_idx)


# ---------------------------------------------------------------- fused QKV epilogue
@torch.library.custom_op("dualkv::qkv_prep", mutates_args=(), device_types="cuda")
def _qkv_prep(qkv: Tensor, q_norm: Optional[Tensor], k_norm: Optional[Tensor], positions: Tensor, dst_rows: Tensor,
              heads: int, kv_heads: int, eps: float, base: float) -> Tuple[Tensor, Tensor, Tensor]:
    from .rope import qkv_prep
    return qkv_prep(qkv, q_norm, k_norm, positions, dst_rows, heads, kv_heads, eps, base)


@_qkv_prep.register_fake
def _qkv_prep_fake(qkv, q_norm, k_norm, positions, dst_rows, heads, kv_heads, eps, base):
    t = qkv.shape[0]
    d = qkv.numel() // (t * (heads + 2 * kv_heads)) if t else 0
    return (qkv.new_empty((t, heads, d)), qkv.new_empty((t, kv_heads, d)), qkv.new_empty((t, kv_heads, d)))


@torch.library.custom_op("dualkv::qkv_prep_bwd", mutates_args=(), device_types="cuda")
def _qkv_prep_bwd(dq: Tensor, dk: Tensor, dv: Tensor, qkv: Tensor, q_norm: Optional[Tensor],
                  k_norm: Optional[Tensor], positions: Tensor, dst_rows: Tensor, heads: int, kv_heads: int,
                  eps: float, base: float) -> Tuple[Tensor, Tensor, Tensor]:
    from .rope import qkv_prep_backward
    dqkv, dwq, dwk = qkv_prep_backward(dq, dk, dv, qkv, q_norm, k_norm, positions, dst_rows, heads, kv_heads, eps,
                                       base)
    if dwq is None:  # custom ops return tensors: empty placeholders for "no norm"
        dwq, dwk = qkv.new_empty((0,), dtype=torch.float32), qkv.new_empty((0,), dtype=torch.float32)
    return dqkv, dwq, dwk


@_qkv_prep_bwd.register_fake
def _qkv_prep_bwd_fake(dq, dk, dv, qkv, q_norm, k_norm, positions, dst_rows, heads, kv_heads, eps, base):
    n = dq.shape[-1] if q_norm is not None else 0
    return torch.empty_like(qkv), qkv.new_empty((n,), dtype=torch.float32), qkv.new_empty((n,), dtype=torch.float32)


def _qkv_setup(ctx, inputs, output):
    qkv, q_norm, k_norm, positions, dst_rows, heads, kv_heads, eps, base = inputs
    ctx.save_for_backward(qkv, q_norm, k_norm, positions, dst_rows)
    ctx.meta = (heads, kv_heads, eps, base)


def _qkv_backward(ctx, dq, dk, dv):
    qkv, q_norm, k_norm, positions, dst_rows = ctx.saved_tensors
    heads, kv_heads, eps, base = ctx.meta
    zeros = lambda like, n: like.new_zeros((like.shape[0], n, like.shape[-1]))
    dq = zeros(qkv, heads) if dq is None else dq
    dk = zeros(qkv, kv_heads) if dk is None else dk
    dv = zeros(qkv, kv_heads) if dv is None else dv
    dqkv, dwq, dwk = torch.ops.dualkv.qkv_prep_bwd(dq, dk, dv, qkv, q_norm, k_norm, positions, dst_rows, heads,
                                                  kv_heads, eps, base)
    dqn = dwq.to(q_norm.dtype) if q_norm is not None else None
    dkn = dwk.to(k_norm.dtype) if k_norm is not None else None
    return dqkv, dqn, dkn, None, None, None, None, None, None


torch.library.register_autograd("dualkv::qkv_prep", _qkv_backward, setup_context=_qkv_setup)


# ---------------------------------------------------------------- two-call op on the split layout
@torch.library.custom_op("dualkv::two_call_split", mutates_args=(), device_types="cuda")
def _split_fwd(q: Tensor, k: Tensor, v: Tensor, p_rows: int, cu_seqlens: Tensor, max_seqlen: int,
               softmax_scale: float, group_seq_cu: List[int], group_ctx_cu: List[int]) -> Tuple[Tensor, Tensor, Tensor]:
    return api.two_call_split_fwd(q, k, v, p_rows, cu_seqlens, max_seqlen, softmax_scale, group_seq_cu,
                                  group_ctx_cu)


@_split_fwd.register_fake
def _split_fwd_fake(q, k, v, p_rows, cu_seqlens, max_seqlen, softmax_scale, group_seq_cu, group_ctx_cu):
    h = q.shape[1]
    return (torch.empty_like(q), q.new_empty((h, p_rows), dtype=torch.float32),
            q.new_empty((h, q.shape[0] - p_rows), dtype=torch.float32))


@torch.library.custom_op("dualkv::two_call_split_bwd", mutates_args=(), device_types="cuda")
def _split_bwd(q: Tensor, k: Tensor, v: Tensor, p_rows: int, cu_seqlens: Tensor, max_seqlen: int,
               softmax_scale: float, group_seq_cu: List[int], group_ctx_cu: List[int], out: Tensor, lse_ctx: Tensor,
               lse: Tensor, d_out: Tensor, deterministic: bool) -> Tuple[Tensor, Tensor, Tensor]:
    return api.two_call_split_bwd(q, k, v, p_rows, cu_seqlens, max_seqlen, softmax_scale, group_seq_cu,
                                  group_ctx_cu, out, lse_ctx, lse, d_out, deterministic)


@_split_bwd.register_fake
def _split_bwd_fake(q, k, v, p_rows, cu_seqlens, max_seqlen, softmax_scale, group_seq_cu, group_ctx_cu, out,
                    lse_ctx, lse, d_out, deterministic):
    return torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)


def _split_setup(ctx, inputs, output):
    q, k, v, p_rows, cu, max_seqlen, scale, gs, gc = inputs
    out, lse_c, lse = output
    ctx.save_for_backward(q, k, v, cu, out, lse_c, lse)
    ctx.meta = (p_rows, max_seqlen, scale, gs, gc)
    ctx.mark_non_differentiable(lse_c, lse)


def _split_backward(ctx, d_out, d_lc, d_l):
    q, k, v, cu, out, lse_c, lse = ctx.saved_tensors
    p_rows, max_seqlen, scale, gs, gc = ctx.meta
    d_out = torch.zeros_like(out) if d_out is None else d_out.contiguous()
    dq, dk, dv = torch.ops.dualkv.two_call_split_bwd(q, k, v, p_rows, cu, max_seqlen, scale, gs, gc, out, lse_c,
                                                     lse, d_out, _deterministic())
    return dq, dk, dv, None, None, None, None, None, None


torch.library.register_autograd("dualkv::two_call_split", _split_backward, setup_context=_split_setup)

"""Rotary embedding at DualKV logical positions, fused with the N(P+R) -> P+NR repack
(reference layer.py:182-205 for `rope` / `rope_bwd`, packing.py:105-120 for
positions: prompt token j -> j, response token r -> P + r).

With DualKV the QKV projection runs once per prompt (on the P+NR rows, the rho token saving);
RoPE must then rotate every response row by its LOGICAL position P + r, not its packed row
index.  `repack_rope_to_dualkv` does the gather from the replicated layout and the rotation of
q and k in one HBM pass per tensor (`dkv_rope_rows` with a row index), `rope_logical` rotates
rows already in the DualKV layout, and `RoPE` is the autograd wrapper (backward = the inverse
rotation, the reference's rope_bwd).  No CPU path: the CUDA library is required.
"""

from __future__ import annotations

from typing import Optional, Sequence, Tuple

import numpy as np
import torch

from ._lib import DKV_BF16, DKV_F32, check, lib
from .packing import PackPlan, position_ids

__all__ = ["rope_logical", "RoPE", "repack_rope_to_dualkv", "dualkv_positions"]

_DT = {torch.bfloat16: DKV_BF16, torch.float32: DKV_F32}


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def dualkv_positions(plan: PackPlan, device) -> torch.Tensor:
    """Device int64 logical positions of the P+NR rows of `plan` (cached on the plan)."""
    key = ("pos_dualkv", str(device))
    if key not in plan._dev:
        plan._dev[key] = torch.as_tensor(position_ids(plan, "dualkv"), dtype=torch.int64, device=device)
    return plan._dev[key]


def _as_positions(positions, n: int, device) -> torch.Tensor:
    if isinstance(positions, torch.Tensor):
        pos = positions.to(device=device, dtype=torch.int64)
    else:
        pos = torch.as_tensor(np.asarray(positions, dtype=np.int64), device=device)
    if pos.dim() != 1 or pos.shape[0] != n:
        raise ValueError(f"positions must be [{n}], got {tuple(pos.shape)}")
    return pos.contiguous()


def _rope_rows(x: torch.Tensor, pos: torch.Tensor, base: float, inverse: bool,
               idx: Optional[torch.Tensor] = None, n_out: Optional[int] = None) -> torch.Tensor:
    if not x.is_cuda:
        raise ValueError("rope: CUDA tensor required (the op has no CPU path)")
    if x.dtype not in _DT:
        raise ValueError(f"rope: dtype {x.dtype} unsupported (bf16 or fp32)")
    if x.dim() != 3 or x.shape[-1] % 2:
        raise ValueError(f"rope: expected [T, heads, even head_dim], got {tuple(x.shape)}")
    x = x.contiguous()
    n = x.shape[0] if n_out is None else n_out
    if pos.device != x.device or pos.dtype != torch.int64 or pos.dim() != 1 or pos.shape[0] != n:
        raise ValueError(f"rope: positions must be int64 [{n}] on {x.device}")
    with torch.cuda.device(x.device):
        out = torch.empty((n,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        check(lib.dkv_rope_rows(x.data_ptr(), out.data_ptr(), _DT[x.dtype], n, x.shape[1], x.shape[2],
                                pos.data_ptr() if n else None, None if idx is None else idx.data_ptr(),
                                float(base), int(inverse), _stream(x.device)), "rope_rows")
    return out


def rope_logical(x: torch.Tensor, positions, base: float = 10000.0, inverse: bool = False) -> torch.Tensor:
    """[T, heads, d] rows rotated by their logical positions (layer.py:188-196); `inverse` =
    the adjoint rope_bwd (layer.py:198-205)."""
    return _rope_rows(x, _as_positions(positions, x.shape[0], x.device), base, inverse)


class RoPE:
    """y = rope(x, positions); dx = rope_bwd(dy, positions) (an orthogonal rotation) -- the
    registered op `dualkv::rope` (library.py), autograd-enabled and torch.compile-traceable."""

    @staticmethod
    def apply(x, positions, base=10000.0):
        from .library import rope
        return rope(x, _as_positions(positions, x.shape[0], x.device), base)


def repack_rope_to_dualkv(q_std: torch.Tensor, k_std: torch.Tensor, v_std: torch.Tensor, plan: PackPlan,
                          base: float = 10000.0) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Replicated-layout projections [T_std, H(_k), d] -> the DualKV layout [T_dk, ...] with q and k
    rotated at logical positions, one fused gather+rotate pass each (v is only gathered).  Prompt
    rows come from the first copy (packing.py:182-220); positions from position_ids."""
    for name, x in (("q", q_std), ("k", k_std), ("v", v_std)):
        if x.shape[0] != plan.total_standard:
            raise ValueError(f"{name}: expected {plan.total_standard} rows, got {x.shape[0]}")
    for x in (q_std, k_std, v_std):
        if not x.is_cuda or x.dtype not in _DT or x.dim() != 3 or x.dtype != q_std.dtype \
                or x.device != q_std.device:
            raise ValueError("repack_rope_to_dualkv: CUDA [T, heads, d] bf16/fp32 tensors of one dtype")
    if k_std.shape != v_std.shape or k_std.shape[2] != q_std.shape[2]:
        raise ValueError("repack_rope_to_dualkv: k / v shapes inconsistent with q")
    q_std, k_std, v_std = q_std.contiguous(), k_std.contiguous(), v_std.contiguous()
    idx = plan.device("dk_from_std", q_std.device)
    pos = dualkv_positions(plan, q_std.device)
    n = plan.total_dualkv
    if pos.shape[0] != n or idx.shape[0] != n:
        raise ValueError(f"repack plan inconsistent: {pos.shape[0]} positions / {idx.shape[0]} rows for "
                         f"{n} packed rows")
    q = torch.empty((n,) + tuple(q_std.shape[1:]), dtype=q_std.dtype, device=q_std.device)
    k = torch.empty((n,) + tuple(k_std.shape[1:]), dtype=k_std.dtype, device=k_std.device)
    v = torch.empty_like(k)
    if n:
        with torch.cuda.device(q_std.device):
            check(lib.dkv_rope_qkv_rows(q_std.data_ptr(), k_std.data_ptr(), v_std.data_ptr(), q.data_ptr(),
                                        k.data_ptr(), v.data_ptr(), _DT[q_std.dtype], n, q_std.shape[1],
                                        k_std.shape[1], q_std.shape[2], pos.data_ptr(), idx.data_ptr(),
                                        float(base), 0, _stream(q_std.device)), "rope_qkv_rows")
    return q, k, v


def qkv_prep(qkv: torch.Tensor, q_norm: Optional[torch.Tensor], k_norm: Optional[torch.Tensor],
             positions: torch.Tensor, dst_rows: torch.Tensor, heads: int, kv_heads: int, eps: float = 1e-6,
             base: float = 10000.0) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Fused epilogue of the QKV projection (`dkv_qkv_prep_fwd`): per-head q/k RMSNorm (Qwen3;
    skipped when the weights are None), RoPE at logical positions, and the scatter of every packed
    row r to row dst_rows[r] of q [T, H, d], k / v [T, H_k, d] -- one HBM pass."""
    if not qkv.is_cuda or qkv.dtype != torch.bfloat16:
        raise ValueError("qkv_prep: bf16 CUDA tensor required")
    t = qkv.shape[0]
    ht = heads + 2 * kv_heads
    if qkv.numel() % max(1, t * ht) or (t and qkv.numel() // (t * ht) % 8):
        raise ValueError(f"qkv_prep: qkv {tuple(qkv.shape)} is not [T, (H + 2 H_k) d]")
    d = qkv.numel() // (t * ht) if t else 0
    qkv = qkv.contiguous()
    for name, x in (("positions", positions), ("dst_rows", dst_rows)):
        if x.device != qkv.device or x.dtype != torch.int64 or tuple(x.shape) != (t,):
            raise ValueError(f"qkv_prep: {name} must be int64 [{t}] on {qkv.device}")
    w = [x.contiguous() if x is not None else None for x in (q_norm, k_norm)]
    if (w[0] is None) != (w[1] is None):
        raise ValueError("qkv_prep: q_norm and k_norm go together")
    with torch.cuda.device(qkv.device):
        q = torch.empty((t, heads, d), dtype=qkv.dtype, device=qkv.device)
        k = torch.empty((t, kv_heads, d), dtype=qkv.dtype, device=qkv.device)
        v = torch.empty_like(k)
        check(lib.dkv_qkv_prep_fwd(qkv.data_ptr(), _p(w[0]), _p(w[1]), float(eps), positions.data_ptr(),
                                   dst_rows.data_ptr(), q.data_ptr(), k.data_ptr(), v.data_ptr(), t, heads, kv_heads,
                                   d, float(base), _stream(qkv.device)), "qkv_prep")
    return q, k, v


def qkv_prep_backward(dq, dk, dv, qkv, q_norm, k_norm, positions, dst_rows, heads: int, kv_heads: int,
                      eps: float = 1e-6, base: float = 10000.0):
    """Adjoint of `qkv_prep` -> (dqkv [T, (H + 2 H_k) d] in qkv's shape, dq_norm, dk_norm fp32 or None)."""
    t, h, d = dq.shape
    dq, dk, dv, qkv = dq.contiguous(), dk.contiguous(), dv.contiguous(), qkv.contiguous()
    with torch.cuda.device(qkv.device):
        dqkv = torch.empty_like(qkv)
        dwq = dwk = None
        if q_norm is not None:
            dwq = torch.empty(d, dtype=torch.float32, device=qkv.device)
            dwk = torch.empty(d, dtype=torch.float32, device=qkv.device)
        check(lib.dkv_qkv_prep_bwd(dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), qkv.data_ptr(), _p(q_norm),
                                   _p(k_norm), float(eps), positions.data_ptr(), dst_rows.data_ptr(),
                                   dqkv.data_ptr(), _p(dwq), _p(dwk), t, heads, kv_heads, d, float(base),
                                   _stream(qkv.device)), "qkv_prep_backward")
    return dqkv, dwq, dwk


def _p(x):
    return None if x is None else x.data_ptr()

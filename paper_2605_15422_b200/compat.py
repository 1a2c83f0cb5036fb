"""Adapter for the reference's own objects (duck-typed, no import of `dualkv`).

Lets the reference's check suites (`verify.py:112-384`, bound by name at
`verify.py:17-26`) and its toy-model backend (`layer.py:35-36`) run against
the GPU op unchanged: patch `dualkv.verify.dualkv_fwd = compat.dualkv_fwd`
etc..  Inputs are the reference's `Tensor`
(`tensor.py:95-124`: `.data` NumPy array + `.precision` with `.value` in
{"f64","f32","bf16"}), `DualKVInput` and `VarlenBatch`; outputs are built
with the caller's own `Tensor` class.

Precision mapping: BF16EMU -> torch.bfloat16 (lossless, the values already
lie on the bf16 grid), F32 -> torch.float32; F64 has no GPU path and raises
ValueError (it stays CPU-oracle-only).
"""

from __future__ import annotations

import numpy as np
import torch

from . import api

_TORCH = {"bf16": torch.bfloat16, "f32": torch.float32}


def _prec(t) -> str:
    p = getattr(t, "precision", None)
    return getattr(p, "value", str(p))


def _dev(t, dtype):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(t.data, dtype=np.float32))).to("cuda", dtype)


def _wrap(like, arr: torch.Tensor, precision=None):
    cls = type(like)
    prec = like.precision if precision is None else precision
    return cls(arr.detach().float().cpu().numpy(), prec)


def _dtype_of(t):
    pv = _prec(t)
    if pv not in _TORCH:
        raise ValueError(f"precision {pv!r} has no GPU path (F64 stays CPU-only)")
    return _TORCH[pv]


def _gpu_input(inp):
    dt = _dtype_of(inp.q)
    return api.DualKVInput(_dev(inp.q, dt), _dev(inp.k_context, dt), _dev(inp.v_context, dt),
                           _dev(inp.k_decoded, dt), _dev(inp.v_decoded, dt), np.asarray(inp.cu_seqlens_q),
                           context_seqlen=inp.context_seqlen, softmax_scale=inp.softmax_scale,
                           causal=inp.causal, tile_size=inp.tile_size)


def _saved_prec(like):
    # the reference returns saved O / lse in compute precision (kernel.py:207-210)
    return type(like.precision)("f32") if _prec(like) != "f64" else like.precision


def dualkv_fwd(inp):
    g = _gpu_input(inp)
    o, lse = api.dualkv_fwd(g)
    sp = _saved_prec(inp.q)
    return _wrap(inp.q, o, sp), _wrap(inp.q, lse, sp)


def dualkv_bwd(inp, out, lse, d_out, deterministic=True, fold_seed=None):
    g = _gpu_input(inp)
    dt = _dtype_of(inp.q)
    grads = api.dualkv_bwd(g, _dev(out, dt), _dev(lse, torch.float32), _dev(d_out, dt),
                           deterministic=deterministic, fold_seed=fold_seed)
    likes = (inp.q, inp.k_context, inp.v_context, inp.k_decoded, inp.v_decoded)
    return tuple(_wrap(l, x) for l, x in zip(likes, grads))


def context_grad_contributions(inp, out, lse, d_out):
    g = _gpu_input(inp)
    dt = _dtype_of(inp.q)
    parts = api.context_grad_contributions(g, _dev(out, dt), _dev(lse, torch.float32), _dev(d_out, dt))
    return [(k.cpu().numpy(), v.cpu().numpy()) for k, v in parts]


def fa2_varlen_fwd(batch):
    dt = _dtype_of(batch.q)
    b = api.VarlenBatch(_dev(batch.q, dt), _dev(batch.k, dt), _dev(batch.v, dt),
                        np.asarray(batch.cu_seqlens), softmax_scale=batch.softmax_scale,
                        tile_size=batch.tile_size)
    o, lse = api.fa2_varlen_fwd(b)
    sp = _saved_prec(batch.q)
    return _wrap(batch.q, o, sp), _wrap(batch.q, lse, sp)


def fa2_varlen_bwd(batch, out, lse, d_out):
    dt = _dtype_of(batch.q)
    b = api.VarlenBatch(_dev(batch.q, dt), _dev(batch.k, dt), _dev(batch.v, dt),
                        np.asarray(batch.cu_seqlens), softmax_scale=batch.softmax_scale,
                        tile_size=batch.tile_size)
    dq, dk, dv = api.fa2_varlen_bwd(b, _dev(out, dt), _dev(lse, torch.float32), _dev(d_out, dt))
    return _wrap(batch.q, dq), _wrap(batch.k, dk), _wrap(batch.v, dv)

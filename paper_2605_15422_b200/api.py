"""Reference-compatible Python surface of the B200 DualKV op.

Mirrors `/root/reference/pkg/src/dualkv/{kernel,fa2}.py` -- same names,
argument order and meaning, and the same ValueError conditions -- but takes
CUDA `torch.Tensor`s (bf16 or fp32) and runs every computation through the
C ABI of libdkv.so on the caller's current CUDA stream.  PyTorch provides
device memory, streams and autograd plumbing only.

Differences from the CPU reference, by design:
  * the saved forward output O is returned in the storage dtype (bf16 for
    bf16 inputs) -- the reference keeps it in f32 (kernel.py:207-210);
  * `tile_size` is accepted and ignored (results are tile-independent,
    verify.py:297-322); the GPU tiles are 128 x 128;
  * `fold_seed` is accepted; with ``deterministic=False`` the shared-prompt
    fold order is whatever order the hardware atomics complete in.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import BwdParams, FwdParams, TwoCallBwdParams, TwoCallFwdParams, check, lib

__all__ = [
    "DualKVInput", "VarlenBatch", "ContextGradScratch",
    "dualkv_fwd", "dualkv_bwd", "context_grad_contributions", "convert_dkv_context",
    "bf16_naive_accumulate", "fa2_varlen_fwd", "fa2_varlen_bwd", "dualkv_attention_varlen",
    "uses_tensor_cores", "dualkv_two_call_fwd", "dualkv_two_call_bwd", "dualkv_two_call_attention",
]

_DTYPES = {torch.bfloat16: _lib.DKV_BF16, torch.float32: _lib.DKV_F32}


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None or t.numel() == 0 else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _check_tensor(t, name, ndim=3):
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (the op has no CPU path)")
    if t.dim() != ndim:
        raise ValueError(f"{name} must be {ndim}-D, got shape {tuple(t.shape)}")
    if t.dtype not in _DTYPES:
        raise ValueError(f"{name} dtype {t.dtype} unsupported (bf16 or fp32)")
    return t.contiguous()


def _offsets(cu, total: int, what: str) -> Tuple[np.ndarray, torch.Tensor]:
    """Host copy (validated as kernel.py:79-82 / fa2.py:72-75) + device int32 copy."""
    if isinstance(cu, torch.Tensor):
        dev = cu if cu.is_cuda else None
        host = cu.detach().to("cpu", torch.int64).numpy()
    else:
        dev = None
        host = np.asarray(cu, dtype=np.int64)
    if host.ndim != 1 or host.size < 2 or host[0] != 0 or host[-1] != total:
        raise ValueError(f"malformed {what} {host!r} for T={total}")
    if np.any(np.diff(host) < 0):
        raise ValueError(f"{what} must be non-decreasing")
    if dev is None or dev.dtype != torch.int32:
        dev = _device_offsets(host)
    return host, dev.contiguous()


_CU_CACHE: dict = {}


def _device_offsets(host: np.ndarray) -> torch.Tensor:
    """int32 device copy of host offsets, cached by content: the first use pays one synchronous
    copy, every later call with the same offsets (every training step of a fixed layout) enqueues
    nothing -- a per-call pageable copy would block the host on the current stream."""
    key = (torch.cuda.current_device(), host.tobytes())
    dev = _CU_CACHE.get(key)
    if dev is None:
        if len(_CU_CACHE) >= 256:  # rare: drop the cache once no kernel can still read it
            for d in {k[0] for k in _CU_CACHE}:
                torch.cuda.synchronize(d)
            _CU_CACHE.clear()
        dev = torch.as_tensor(host.astype(np.int32), device="cuda")
        _CU_CACHE[key] = dev
    return dev


def uses_tensor_cores(dtype: torch.dtype, head_dim: int, heads: int, kv_heads: int) -> bool:
    return bool(lib.dkv_uses_tensor_cores(_DTYPES[dtype], head_dim, heads, kv_heads))


# ---------------------------------------------------------------------------
# input contracts (kernel.py:52-114, fa2.py:57-91)
# ---------------------------------------------------------------------------

@dataclass
class DualKVInput:
    """Five-tensor contract of the two-region kernel (kernel.py:52-114)."""

    q: torch.Tensor          # [sum R_i, H, d]
    k_context: torch.Tensor  # [P, H_k, d]
    v_context: torch.Tensor  # [P, H_k, d]
    k_decoded: torch.Tensor  # [sum R_i, H_k, d]
    v_decoded: torch.Tensor  # [sum R_i, H_k, d]
    cu_seqlens_q: object     # [N+1] host array / tensor
    context_seqlen: Optional[int] = None
    max_seqlen_q: Optional[int] = None
    softmax_scale: Optional[float] = None
    causal: bool = True
    tile_size: int = 64

    def __post_init__(self):
        self.q = _check_tensor(self.q, "q")
        t_dec, h, d = self.q.shape
        self.cu_host, self.cu_dev = _offsets(self.cu_seqlens_q, t_dec, "cu_seqlens_q")
        self.k_context = _check_tensor(self.k_context, "k_context")
        self.v_context = _check_tensor(self.v_context, "v_context")
        self.k_decoded = _check_tensor(self.k_decoded, "k_decoded")
        self.v_decoded = _check_tensor(self.v_decoded, "v_decoded")
        if self.k_context.shape != self.v_context.shape:
            raise ValueError("k_context / v_context shape mismatch")
        if self.k_decoded.shape != self.v_decoded.shape:
            raise ValueError("k_decoded / v_decoded shape mismatch")
        if self.context_seqlen is None:
            self.context_seqlen = self.k_context.shape[0]
        if self.context_seqlen < 0:
            raise ValueError("context_seqlen must be non-negative")
        if self.context_seqlen != self.k_context.shape[0]:
            raise ValueError(f"context_seqlen={self.context_seqlen} != k_context length "
                             f"{self.k_context.shape[0]}")
        if self.k_decoded.shape[0] != t_dec:
            raise ValueError("k_decoded must share q's packed token count")
        h_k = self.k_context.shape[1]
        if self.k_decoded.shape[1] != h_k or self.k_context.shape[2] != d or self.k_decoded.shape[2] != d:
            raise ValueError("context/decoded KV head layout mismatch")
        if h_k == 0 or h % h_k != 0:
            raise ValueError(f"H={h} must be a positive multiple of H_k={h_k}")
        if not self.causal:
            raise ValueError("only causal=True is supported")
        if self.tile_size < 1:
            raise ValueError("tile_size must be >= 1")
        dts = {x.dtype for x in (self.q, self.k_context, self.v_context, self.k_decoded, self.v_decoded)}
        if len(dts) != 1:
            raise ValueError(f"all five tensors must share one dtype, got {dts}")
        if self.softmax_scale is None:
            self.softmax_scale = 1.0 / math.sqrt(d)
        lens = np.diff(self.cu_host)
        true_max = int(lens.max()) if lens.size else 0
        if self.max_seqlen_q is None:
            self.max_seqlen_q = true_max
        self._grid_max = max(int(self.max_seqlen_q), true_max)

    @property
    def num_sequences(self) -> int:
        return self.cu_host.size - 1


@dataclass
class VarlenBatch:
    """Packed varlen batch for per-sequence causal attention (fa2.py:57-91)."""

    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    cu_seqlens: object
    max_seqlen: Optional[int] = None
    softmax_scale: Optional[float] = None
    tile_size: int = 64

    def __post_init__(self):
        self.q = _check_tensor(self.q, "q")
        t_total, h, d = self.q.shape
        self.cu_host, self.cu_dev = _offsets(self.cu_seqlens, t_total, "cu_seqlens")
        self.k = _check_tensor(self.k, "k")
        self.v = _check_tensor(self.v, "v")
        if self.k.shape != self.v.shape or self.k.shape[0] != t_total or self.k.shape[2] != d:
            raise ValueError(f"K/V shape {tuple(self.k.shape)} inconsistent with Q {tuple(self.q.shape)}")
        h_k = self.k.shape[1]
        if h_k == 0 or h % h_k != 0:
            raise ValueError(f"H={h} must be a positive multiple of H_k={h_k}")
        if self.tile_size < 1:
            raise ValueError("tile_size must be >= 1")
        if len({self.q.dtype, self.k.dtype, self.v.dtype}) != 1:
            raise ValueError("q/k/v must share one dtype")
        if self.softmax_scale is None:
            self.softmax_scale = 1.0 / math.sqrt(d)
        lens = np.diff(self.cu_host)
        true_max = int(lens.max()) if lens.size else 0
        if self.max_seqlen is None:
            self.max_seqlen = true_max
        self._grid_max = max(int(self.max_seqlen), true_max)

    @property
    def num_sequences(self) -> int:
        return self.cu_host.size - 1


# ---------------------------------------------------------------------------
# forward (kernel.py:177-210, fa2.py:237-265)
# ---------------------------------------------------------------------------

def _fwd_params(q, kc, vc, k, v, cu_dev, n, p_len, grid_max, scale, out, lse):
    t, h, d = q.shape
    prm = FwdParams()
    prm.q, prm.k_ctx, prm.v_ctx, prm.k, prm.v = _ptr(q), _ptr(kc), _ptr(vc), _ptr(k), _ptr(v)
    prm.cu_seqlens, prm.out, prm.lse = cu_dev.data_ptr(), _ptr(out), _ptr(lse)
    prm.num_seqs, prm.total_q, prm.ctx_len = n, t, p_len
    prm.heads, prm.kv_heads, prm.head_dim = h, k.shape[1], d
    prm.max_seqlen = grid_max
    prm.softmax_scale = float(scale)
    prm.dtype = _DTYPES[q.dtype]
    return prm


def dualkv_fwd(inp: DualKVInput) -> Tuple[torch.Tensor, torch.Tensor]:
    """Two-region forward -> (O [sum R_i, H, d], lse [H, sum R_i] f32)."""
    q = inp.q
    out = torch.empty_like(q)
    lse = torch.empty((q.shape[1], q.shape[0]), dtype=torch.float32, device=q.device)
    prm = _fwd_params(q, inp.k_context, inp.v_context, inp.k_decoded, inp.v_decoded, inp.cu_dev,
                      inp.num_sequences, inp.context_seqlen, inp._grid_max, inp.softmax_scale, out, lse)
    check(lib.dkv_dualkv_fwd(ctypes_ref(prm), _stream()), "dualkv_fwd")
    return out, lse


def fa2_varlen_fwd(batch: VarlenBatch) -> Tuple[torch.Tensor, torch.Tensor]:
    """Per-sequence causal attention -> (O [T, H, d], lse [H, T] f32)."""
    q = batch.q
    out = torch.empty_like(q)
    lse = torch.empty((q.shape[1], q.shape[0]), dtype=torch.float32, device=q.device)
    prm = _fwd_params(q, None, None, batch.k, batch.v, batch.cu_dev, batch.num_sequences, 0,
                      batch._grid_max, batch.softmax_scale, out, lse)
    check(lib.dkv_varlen_fwd(ctypes_ref(prm), _stream()), "fa2_varlen_fwd")
    return out, lse


def ctypes_ref(s):
    import ctypes
    return ctypes.byref(s)


# ---------------------------------------------------------------------------
# backward (kernel.py:213-305, fa2.py:268-306)
# ---------------------------------------------------------------------------

def _bwd_params(q, kc, vc, k, v, cu_dev, n, p_len, grid_max, scale, out, lse, d_out, deterministic,
                ctx_chunk=0):
    """Shape checks, output allocation and the C parameter block of one backward."""
    t, h, d = q.shape
    if tuple(d_out.shape) != tuple(q.shape) or tuple(out.shape) != tuple(q.shape):
        raise ValueError(f"O/dO shape {tuple(out.shape)}/{tuple(d_out.shape)} inconsistent with q "
                         f"{tuple(q.shape)}")
    if tuple(lse.shape) != (h, t):
        raise ValueError(f"lse shape {tuple(lse.shape)} != {(h, t)}")
    keep = dict(out=out.to(q.dtype).contiguous(), d_out=d_out.to(q.dtype).contiguous(),
                lse=lse.to(torch.float32).contiguous())
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    dkc = torch.empty_like(kc) if kc is not None else None
    dvc = torch.empty_like(vc) if vc is not None else None
    prm = BwdParams()
    prm.q, prm.k_ctx, prm.v_ctx, prm.k, prm.v = _ptr(q), _ptr(kc), _ptr(vc), _ptr(k), _ptr(v)
    prm.cu_seqlens, prm.out = cu_dev.data_ptr(), _ptr(keep["out"])
    prm.lse, prm.dout = _ptr(keep["lse"]), _ptr(keep["d_out"])
    prm.dq, prm.dk_ctx, prm.dv_ctx, prm.dk, prm.dv = _ptr(dq), _ptr(dkc), _ptr(dvc), _ptr(dk), _ptr(dv)
    prm.num_seqs, prm.total_q, prm.ctx_len = n, t, p_len
    prm.heads, prm.kv_heads, prm.head_dim = h, k.shape[1], d
    prm.max_seqlen = grid_max
    prm.softmax_scale = float(scale)
    prm.dtype = _DTYPES[q.dtype]
    prm.deterministic = 1 if deterministic else 0
    prm.ctx_chunk = int(ctx_chunk)
    return prm, (dq, dkc, dvc, dk, dv), keep


def _bwd_run(q, kc, vc, k, v, cu_dev, n, p_len, grid_max, scale, out, lse, d_out, deterministic,
             ctx_chunk=0, partials_for_chunks=False, varlen=False):
    prm, grads, keep = _bwd_params(q, kc, vc, k, v, cu_dev, n, p_len, grid_max, scale, out, lse, d_out,
                                   deterministic, ctx_chunk)
    partials = None
    if partials_for_chunks:
        nch = int(lib.dkv_bwd_num_ctx_chunks(ctypes_ref(prm)))
        kk = kc if kc is not None else k
        partials = torch.empty((nch, 2, p_len, kk.shape[1], q.shape[2]), dtype=torch.float32, device=q.device)
        prm.ctx_partials = _ptr(partials)
    ws_bytes = int(lib.dkv_bwd_workspace_size(ctypes_ref(prm)))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=q.device)
    fn = lib.dkv_varlen_bwd if varlen else lib.dkv_dualkv_bwd
    check(fn(ctypes_ref(prm), ws.data_ptr(), ws_bytes, _stream()),
          "fa2_varlen_bwd" if varlen else "dualkv_bwd")
    del keep
    return grads + (partials,)


def dualkv_bwd(inp: DualKVInput, out, lse, d_out, deterministic: bool = True,
               fold_seed: Optional[int] = None):
    """Two-region backward -> (dQ_d, dK_c, dV_c, dK_d, dV_d) in storage dtype.

    dK_c/dV_c are the fp32 sum over all sequences cast once
    (kernel.py:279-285).  ``fold_seed`` is accepted for interface parity.
    """
    del fold_seed
    dq, dkc, dvc, dkd, dvd, _ = _bwd_run(
        inp.q, inp.k_context, inp.v_context, inp.k_decoded, inp.v_decoded, inp.cu_dev,
        inp.num_sequences, inp.context_seqlen, inp._grid_max, inp.softmax_scale, out, lse, d_out,
        deterministic)
    return dq, dkc, dvc, dkd, dvd


def context_grad_contributions(inp: DualKVInput, out, lse, d_out) -> List[Tuple[torch.Tensor, torch.Tensor]]:
    """Per-sequence fp32 (dK_c^i, dV_c^i) before any fold (kernel.py:296-305).

    Zero-length sequences contribute nothing and are skipped, as in the
    reference generator (kernel.py:231-234)."""
    res = _bwd_run(inp.q, inp.k_context, inp.v_context, inp.k_decoded, inp.v_decoded, inp.cu_dev,
                   inp.num_sequences, inp.context_seqlen, inp._grid_max, inp.softmax_scale, out, lse,
                   d_out, True, ctx_chunk=1, partials_for_chunks=True)
    parts = res[5]
    lens = np.diff(inp.cu_host)
    return [(parts[i, 0], parts[i, 1]) for i in range(inp.num_sequences) if lens[i] > 0]


def fa2_varlen_bwd(batch: VarlenBatch, out, lse, d_out):
    """Backward of `fa2_varlen_fwd` -> (dQ, dK, dV) in storage dtype (fa2.py:268-306)."""
    dq, _, _, dk, dv, _ = _bwd_run(batch.q, None, None, batch.k, batch.v, batch.cu_dev,
                                   batch.num_sequences, 0, batch._grid_max, batch.softmax_scale, out,
                                   lse, d_out, True, varlen=True)
    return dq, dk, dv


# ---------------------------------------------------------------------------
# shared-prompt gradient scratch and cast (kernel.py:117-165)
# ---------------------------------------------------------------------------

@dataclass
class ContextGradScratch:
    """fp32 accumulators for the shared-context gradients (kernel.py:117-137)."""

    dk_acc: torch.Tensor
    dv_acc: torch.Tensor

    @staticmethod
    def zeros(p: int, h_k: int, d: int, dtype=torch.float32, device="cuda") -> "ContextGradScratch":
        return ContextGradScratch(torch.zeros((p, h_k, d), dtype=dtype, device=device),
                                  torch.zeros((p, h_k, d), dtype=dtype, device=device))

    def add(self, dk_contrib, dv_contrib) -> None:
        self.dk_acc += torch.as_tensor(dk_contrib, device=self.dk_acc.device)
        self.dv_acc += torch.as_tensor(dv_contrib, device=self.dv_acc.device)


def convert_dkv_context(scratch: ContextGradScratch, out_dtype=torch.bfloat16):
    """Exactly one RNE cast per element (kernel.py:140-148) through the C ABI."""
    if out_dtype in (torch.float32, "f32"):
        return scratch.dk_acc.clone(), scratch.dv_acc.clone()
    outs = []
    for acc in (scratch.dk_acc, scratch.dv_acc):
        acc = acc.to(torch.float32).contiguous()
        dst = torch.empty(acc.shape, dtype=torch.bfloat16, device=acc.device)
        check(lib.dkv_convert_f32_to_bf16(_ptr(acc), _ptr(dst), acc.numel(), _stream()),
              "convert_dkv_context")
        outs.append(dst)
    return outs[0], outs[1]


def bf16_naive_accumulate(contributions) -> torch.Tensor:
    """The rejected fold acc = bf16(acc + bf16(c)) (kernel.py:151-165), a precision foil."""
    acc = None
    for c in contributions:
        c = torch.as_tensor(c).to(torch.bfloat16)
        acc = c if acc is None else (acc.float() + c.float()).to(torch.bfloat16)
    if acc is None:
        raise ValueError("need at least one contribution")
    return acc


# ---------------------------------------------------------------------------
# five-tensor autograd surface (kernel.py:308-348)
# ---------------------------------------------------------------------------

class _DualKVFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k_context, v_context, k_decoded, v_decoded, inp):
        out, lse = dualkv_fwd(inp)
        ctx.save_for_backward(out, lse)
        ctx.inp = inp
        return out

    @staticmethod
    def backward(ctx, d_out):
        out, lse = ctx.saved_tensors
        dq, dkc, dvc, dkd, dvd = dualkv_bwd(ctx.inp, out, lse, d_out.contiguous(), deterministic=False)
        return dq, dkc, dvc, dkd, dvd, None


def dualkv_attention_varlen(q, k_context, v_context, k_decoded, v_decoded, cu_seqlens_q,
                            cu_seqlens_k_decoded=None, max_seqlen_q: Optional[int] = None,
                            context_seqlen: Optional[int] = None,
                            max_seqlen_k_decoded: Optional[int] = None,
                            softmax_scale: Optional[float] = None, causal: bool = True,
                            tile_size: int = 64) -> torch.Tensor:
    """Five-tensor call surface; lse is saved on the autograd ctx, not returned."""
    if cu_seqlens_k_decoded is not None:
        a = np.asarray(cu_seqlens_k_decoded.cpu() if isinstance(cu_seqlens_k_decoded, torch.Tensor)
                       else cu_seqlens_k_decoded)
        b = np.asarray(cu_seqlens_q.cpu() if isinstance(cu_seqlens_q, torch.Tensor) else cu_seqlens_q)
        if not np.array_equal(a, b):
            raise ValueError("cu_seqlens_k_decoded must equal cu_seqlens_q")
    del max_seqlen_k_decoded  # decoded KV shares q's offsets (kernel.py:333)
    inp = DualKVInput(q, k_context, v_context, k_decoded, v_decoded, cu_seqlens_q,
                      context_seqlen=context_seqlen, max_seqlen_q=max_seqlen_q,
                      softmax_scale=softmax_scale, causal=causal, tile_size=tile_size)
    return _DualKVFunction.apply(inp.q, inp.k_context, inp.v_context, inp.k_decoded,
                                 inp.v_decoded, inp)


# ---------------------------------------------------------------------------
# fused two-call op (layer.py:236-290 composed in one launch)
# ---------------------------------------------------------------------------

def _check_prompt_q(q_ctx, inp: DualKVInput):
    q_ctx = _check_tensor(q_ctx, "q_context")
    p_len = inp.context_seqlen
    if tuple(q_ctx.shape) != (p_len, inp.q.shape[1], inp.q.shape[2]) or q_ctx.dtype != inp.q.dtype:
        raise ValueError(f"q_context shape/dtype {tuple(q_ctx.shape)}/{q_ctx.dtype} inconsistent with "
                         f"P={p_len}, q {tuple(inp.q.shape)}/{inp.q.dtype}")
    return q_ctx


def dualkv_two_call_fwd(q_context, inp: DualKVInput):
    """Call 1 (causal self-attention of the prompt's own queries) + Call 2 (DualKV) in ONE launch.

    Returns (O_ctx [P,H,d], lse_ctx [H,P], O_dec [sum R_i,H,d], lse_dec [H,sum R_i]) -- equal to
    `fa2_varlen_fwd` over the prompt and `dualkv_fwd(inp)` (layer.py:243-255)."""
    q_ctx = _check_prompt_q(q_context, inp)
    q = inp.q
    p_len, h, d = q_ctx.shape
    out = torch.empty_like(q)
    lse = torch.empty((h, q.shape[0]), dtype=torch.float32, device=q.device)
    out_c = torch.empty_like(q_ctx)
    lse_c = torch.empty((h, p_len), dtype=torch.float32, device=q.device)
    prm = TwoCallFwdParams()
    prm.call2 = _fwd_params(q, inp.k_context, inp.v_context, inp.k_decoded, inp.v_decoded, inp.cu_dev,
                            inp.num_sequences, p_len, inp._grid_max, inp.softmax_scale, out, lse)
    prm.q_ctx, prm.out_ctx, prm.lse_ctx = _ptr(q_ctx), _ptr(out_c), _ptr(lse_c)
    check(lib.dkv_twocall_fwd(ctypes_ref(prm), _stream()), "dualkv_two_call_fwd")
    return out_c, lse_c, out, lse


def dualkv_two_call_bwd(q_context, inp: DualKVInput, out_ctx, lse_ctx, d_out_ctx, out, lse, d_out,
                        deterministic: bool = True):
    """Backward of both calls in ONE launch.  Returns (dQ_ctx, dK_c, dV_c, dQ_dec, dK_dec, dV_dec),
    dK_c / dV_c being the TOTAL prompt-key gradient (Call 1 + Call 2, layer.py:278-279) accumulated
    in one fp32 scratch and cast once."""
    q_ctx = _check_prompt_q(q_context, inp)
    p_len, h, d = q_ctx.shape
    if tuple(out_ctx.shape) != tuple(q_ctx.shape) or tuple(d_out_ctx.shape) != tuple(q_ctx.shape):
        raise ValueError("O_ctx/dO_ctx shape inconsistent with q_context")
    if tuple(lse_ctx.shape) != (h, p_len):
        raise ValueError(f"lse_ctx shape {tuple(lse_ctx.shape)} != {(h, p_len)}")
    prm2, grads, keep = _bwd_params(inp.q, inp.k_context, inp.v_context, inp.k_decoded, inp.v_decoded,
                                    inp.cu_dev, inp.num_sequences, p_len, inp._grid_max, inp.softmax_scale,
                                    out, lse, d_out, deterministic)
    dq, dkc, dvc, dkd, dvd = grads
    o_c = out_ctx.to(q_ctx.dtype).contiguous()
    l_c = lse_ctx.to(torch.float32).contiguous()
    do_c = d_out_ctx.to(q_ctx.dtype).contiguous()
    dq_c = torch.empty_like(q_ctx)
    prm = TwoCallBwdParams()
    prm.call2 = prm2
    prm.q_ctx, prm.out_ctx, prm.lse_ctx = _ptr(q_ctx), _ptr(o_c), _ptr(l_c)
    prm.dout_ctx, prm.dq_ctx = _ptr(do_c), _ptr(dq_c)
    ws_bytes = int(lib.dkv_twocall_bwd_workspace_size(ctypes_ref(prm)))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=q_ctx.device)
    check(lib.dkv_twocall_bwd(ctypes_ref(prm), ws.data_ptr(), ws_bytes, _stream()), "dualkv_two_call_bwd")
    del keep
    return dq_c, dkc, dvc, dq, dkd, dvd


class _TwoCallFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q_context, k_context, v_context, q, k_decoded, v_decoded, inp):
        o_c, l_c, o, l = dualkv_two_call_fwd(q_context, inp)
        ctx.save_for_backward(q_context, o_c, l_c, o, l)
        ctx.inp = inp
        return o_c, o

    @staticmethod
    def backward(ctx, d_oc, d_o):
        q_c, o_c, l_c, o, l = ctx.saved_tensors
        d_oc = torch.zeros_like(o_c) if d_oc is None else d_oc.contiguous()
        d_o = torch.zeros_like(o) if d_o is None else d_o.contiguous()
        dq_c, dkc, dvc, dq, dkd, dvd = dualkv_two_call_bwd(q_c, ctx.inp, o_c, l_c, d_oc, o, l, d_o,
                                                           deterministic=False)
        return dq_c, dkc, dvc, dq, dkd, dvd, None


def dualkv_two_call_attention(q_context, k_context, v_context, q_decoded, k_decoded, v_decoded,
                              cu_seqlens_q, max_seqlen_q: Optional[int] = None,
                              softmax_scale: Optional[float] = None):
    """The whole attention of one prompt group in the P+NR layout (layer.py:236-290): returns
    (O_context [P,H,d], O_decoded [sum R_i,H,d]); autograd gives all six input gradients, the
    prompt K/V gradient summed over both calls and all N sequences in fp32 and cast once."""
    inp = DualKVInput(q_decoded, k_context, v_context, k_decoded, v_decoded, cu_seqlens_q,
                      max_seqlen_q=max_seqlen_q, softmax_scale=softmax_scale)
    q_ctx = _check_prompt_q(q_context, inp)
    return _TwoCallFunction.apply(q_ctx, inp.k_context, inp.v_context, inp.q, inp.k_decoded,
                                  inp.v_decoded, inp)

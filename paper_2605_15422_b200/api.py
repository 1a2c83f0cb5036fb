"""Reference-compatible Python surface of the B200 DualKV op.

Mirrors `/root/reference/pkg/src/dualkv/{kernel,fa2}.py` -- same names,
argument order and meaning, and the same ValueError conditions -- but takes
CUDA `torch.Tensor`s (bf16 or fp32) and runs every computation through the
C ABI of libdkv.so on the current CUDA stream of the tensors' device.
PyTorch provides device memory, streams and autograd plumbing only.

Differences from the CPU reference, by design:
  * the saved forward output O is returned in the storage dtype (bf16 for
    bf16 inputs) -- the reference keeps it in f32 (kernel.py:207-210);
  * `tile_size` is accepted and ignored (results are tile-independent,
    verify.py:297-322); the GPU tiles are 128 x 128;
  * `fold_seed` is accepted; with ``deterministic=False`` the shared-prompt
    fold order is whatever order the hardware atomics complete in;
  * `cu_seqlens` may be a CUDA int32/int64 tensor: given together with the
    max sequence length it is used as is, with no host synchronisation (the
    values are the caller's contract, as in flash-attn's varlen API);
    otherwise it is copied to the host once and validated like the reference;
  * several prompt groups can run in ONE launch (`group_seq_cu` /
    `group_ctx_cu`, the C ABI's group table): the reference loops over groups
    in its caller (layer.py:239).
"""

from __future__ import annotations

import copy
import ctypes
import math
import threading
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


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _check_tensor(t, name, ndim=3, device=None):
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (the op has no CPU path)")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, the other inputs on {device}")
    if t.dim() != ndim:
        raise ValueError(f"{name} must be {ndim}-D, got shape {tuple(t.shape)}")
    if t.dtype not in _DTYPES:
        raise ValueError(f"{name} dtype {t.dtype} unsupported (bf16 or fp32)")
    return t.contiguous()


def _validate_offsets(host: np.ndarray, total: int, what: str) -> None:
    """kernel.py:79-82 / fa2.py:72-75."""
    if host.ndim != 1 or host.size < 2 or host[0] != 0 or host[-1] != total:
        raise ValueError(f"malformed {what} {host!r} for T={total}")
    if np.any(np.diff(host) < 0):
        raise ValueError(f"{what} must be non-decreasing")


def _offsets(cu, total: int, what: str, device: torch.device, max_len: Optional[int]):
    """-> (host int64 copy or None, device int32 tensor, number of sequences, true max or None).

    A CUDA tensor with `max_len` given is trusted and never read on the host (no device sync);
    everything else is validated on the host first."""
    if isinstance(cu, torch.Tensor) and cu.is_cuda:
        if cu.device != device:
            raise ValueError(f"{what} is on {cu.device}, the tensors on {device}")
        if cu.dim() != 1 or cu.numel() < 2:
            raise ValueError(f"malformed {what}: shape {tuple(cu.shape)}")
        dev = (cu if cu.dtype == torch.int32 else cu.to(torch.int32)).contiguous()
        if max_len is not None:
            return None, dev, cu.numel() - 1, None
        host = cu.detach().to("cpu", torch.int64).numpy()
    else:
        host = np.asarray(cu.detach().cpu().numpy() if isinstance(cu, torch.Tensor) else cu, dtype=np.int64)
        dev = None
    _validate_offsets(host, total, what)
    if dev is None:
        dev = _device_offsets(host, device)
    lens = np.diff(host)
    return host, dev, host.size - 1, int(lens.max()) if lens.size else 0


_CU_CACHE: dict = {}
_CU_LOCK = threading.Lock()


def _device_offsets(host: np.ndarray, device: torch.device) -> torch.Tensor:
    """int32 device copy of host offsets, cached by (device, content): the first use pays one
    synchronous copy, every later call with the same offsets (every training step of a fixed
    layout) enqueues nothing -- a per-call pageable copy would block the host."""
    key = (device.index, host.tobytes())
    with _CU_LOCK:
        dev = _CU_CACHE.get(key)
        if dev is None:
            if len(_CU_CACHE) >= 256:  # rare: drop the cache once no kernel can still read it
                for d in {k[0] for k in _CU_CACHE}:
                    torch.cuda.synchronize(d)
                _CU_CACHE.clear()
            dev = torch.as_tensor(host.astype(np.int32), device=device)
            _CU_CACHE[key] = dev
    return dev


def _group_table(seq_cu, ctx_cu, n_seqs: int, p_total: int):
    """Validated host int32 copies of a multi-group table (include/dkv.h dkv_group_table), or None."""
    if seq_cu is None and ctx_cu is None:
        return None
    if seq_cu is None or ctx_cu is None:
        raise ValueError("group_seq_cu and group_ctx_cu go together")
    s = np.asarray(seq_cu, dtype=np.int64)
    c = np.asarray(ctx_cu, dtype=np.int64)
    if s.ndim != 1 or c.shape != s.shape or s.size < 2:
        raise ValueError("group tables must be 1-D of equal length >= 2")
    if s.size - 1 > _lib.DKV_MAX_GROUPS:
        raise ValueError(f"at most {_lib.DKV_MAX_GROUPS} groups per launch")
    if s[0] != 0 or s[-1] != n_seqs or np.any(np.diff(s) <= 0):
        raise ValueError(f"group_seq_cu {s!r} must rise strictly from 0 to N={n_seqs} "
                         "(every group has at least one sequence)")
    if c[0] != 0 or c[-1] != p_total or np.any(np.diff(c) < 0):
        raise ValueError(f"group_ctx_cu {c!r} must rise from 0 to the prompt rows {p_total}")
    return np.ascontiguousarray(s, dtype=np.int32), np.ascontiguousarray(c, dtype=np.int32)


def _set_groups(dst, table) -> None:
    if table is None:
        dst.num_groups, dst.seq_cu, dst.ctx_cu = 0, None, None
    else:
        dst.num_groups = table[0].size - 1
        dst.seq_cu, dst.ctx_cu = table[0].ctypes.data, table[1].ctypes.data


def uses_tensor_cores(dtype: torch.dtype, head_dim: int, heads: int, kv_heads: int) -> bool:
    return bool(lib.dkv_uses_tensor_cores(_DTYPES[dtype], head_dim, heads, kv_heads))


# ---------------------------------------------------------------------------
# input contracts (kernel.py:52-114, fa2.py:57-91)
# ---------------------------------------------------------------------------

@dataclass
class DualKVInput:
    """Five-tensor contract of the two-region kernel (kernel.py:52-114).

    Extension: `group_seq_cu` / `group_ctx_cu` (host, N_groups + 1) put several prompt groups in
    one launch -- k_context / v_context then hold every group's prompt rows back to back and
    `context_seqlen` is their total."""

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
    group_seq_cu: Optional[Sequence[int]] = None
    group_ctx_cu: Optional[Sequence[int]] = None

    def __post_init__(self):
        self.q = _check_tensor(self.q, "q")
        dev = self.q.device
        t_dec, h, d = self.q.shape
        self.cu_host, self.cu_dev, self._n, true_max = _offsets(self.cu_seqlens_q, t_dec, "cu_seqlens_q", dev,
                                                               self.max_seqlen_q)
        self.k_context = _check_tensor(self.k_context, "k_context", device=dev)
        self.v_context = _check_tensor(self.v_context, "v_context", device=dev)
        self.k_decoded = _check_tensor(self.k_decoded, "k_decoded", device=dev)
        self.v_decoded = _check_tensor(self.v_decoded, "v_decoded", device=dev)
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
        if self.max_seqlen_q is None:
            self.max_seqlen_q = true_max
        if self.max_seqlen_q < 0:
            raise ValueError("max_seqlen_q must be non-negative")
        self._grid_max = max(int(self.max_seqlen_q), true_max or 0)
        self._groups = _group_table(self.group_seq_cu, self.group_ctx_cu, self._n, self.context_seqlen)

    @property
    def num_sequences(self) -> int:
        return self._n

    @property
    def num_groups(self) -> int:
        return 1 if self._groups is None else self._groups[0].size - 1

    def _rebind(self, q, k_context, v_context, k_decoded, v_decoded) -> "DualKVInput":
        """The same (validated) metadata over other tensors of identical shapes (autograd saves
        the tensors through save_for_backward and rebuilds the input in backward)."""
        new = copy.copy(self)
        new.q, new.k_context, new.v_context, new.k_decoded, new.v_decoded = (
            q, k_context, v_context, k_decoded, v_decoded)
        return new


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
        dev = self.q.device
        t_total, h, d = self.q.shape
        self.cu_host, self.cu_dev, self._n, true_max = _offsets(self.cu_seqlens, t_total, "cu_seqlens", dev,
                                                               self.max_seqlen)
        self.k = _check_tensor(self.k, "k", device=dev)
        self.v = _check_tensor(self.v, "v", device=dev)
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
        if self.max_seqlen is None:
            self.max_seqlen = true_max
        self._grid_max = max(int(self.max_seqlen), true_max or 0)

    @property
    def num_sequences(self) -> int:
        return self._n


# ---------------------------------------------------------------------------
# forward (kernel.py:177-210, fa2.py:237-265)
# ---------------------------------------------------------------------------

def _fwd_params(q, kc, vc, k, v, cu_dev, n, p_len, grid_max, scale, out, lse, groups=None):
    t, h, d = q.shape
    prm = FwdParams()
    prm.q, prm.k_ctx, prm.v_ctx, prm.k, prm.v = _ptr(q), _ptr(kc), _ptr(vc), _ptr(k), _ptr(v)
    prm.cu_seqlens, prm.out, prm.lse = cu_dev.data_ptr(), _ptr(out), _ptr(lse)
    prm.num_seqs, prm.total_q, prm.ctx_len = n, t, p_len
    prm.heads, prm.kv_heads, prm.head_dim = h, k.shape[1], d
    prm.max_seqlen = grid_max
    prm.softmax_scale = float(scale)
    prm.dtype = _DTYPES[q.dtype]
    _set_groups(prm.groups, groups)
    return prm


def dualkv_fwd(inp: DualKVInput) -> Tuple[torch.Tensor, torch.Tensor]:
    """Two-region forward -> (O [sum R_i, H, d], lse [H, sum R_i] f32)."""
    q = inp.q
    with torch.cuda.device(q.device):
        out = torch.empty_like(q)
        lse = torch.empty((q.shape[1], q.shape[0]), dtype=torch.float32, device=q.device)
        prm = _fwd_params(q, inp.k_context, inp.v_context, inp.k_decoded, inp.v_decoded, inp.cu_dev,
                          inp.num_sequences, inp.context_seqlen, inp._grid_max, inp.softmax_scale, out, lse,
                          inp._groups)
        check(lib.dkv_dualkv_fwd(ctypes.byref(prm), _stream(q.device)), "dualkv_fwd")
    return out, lse


def fa2_varlen_fwd(batch: VarlenBatch) -> Tuple[torch.Tensor, torch.Tensor]:
    """Per-sequence causal attention -> (O [T, H, d], lse [H, T] f32)."""
    q = batch.q
    with torch.cuda.device(q.device):
        out = torch.empty_like(q)
        lse = torch.empty((q.shape[1], q.shape[0]), dtype=torch.float32, device=q.device)
        prm = _fwd_params(q, None, None, batch.k, batch.v, batch.cu_dev, batch.num_sequences, 0,
                          batch._grid_max, batch.softmax_scale, out, lse)
        check(lib.dkv_varlen_fwd(ctypes.byref(prm), _stream(q.device)), "fa2_varlen_fwd")
    return out, lse


# ---------------------------------------------------------------------------
# backward (kernel.py:213-305, fa2.py:268-306)
# ---------------------------------------------------------------------------

def _bwd_params(q, kc, vc, k, v, cu_dev, n, p_len, grid_max, scale, out, lse, d_out, deterministic,
                ctx_chunk=0, groups=None, grads=None):
    """Shape checks (kernel.py:214-218), output allocation and the C parameter block of one backward."""
    t, h, d = q.shape
    for name, x in (("O", out), ("dO", d_out), ("lse", lse)):
        if not isinstance(x, torch.Tensor) or not x.is_cuda or x.device != q.device:
            raise ValueError(f"{name} must be a CUDA tensor on {q.device}")
    if tuple(d_out.shape) != tuple(q.shape) or tuple(out.shape) != tuple(q.shape):
        raise ValueError(f"O/dO shape {tuple(out.shape)}/{tuple(d_out.shape)} inconsistent with q "
                         f"{tuple(q.shape)}")
    if tuple(lse.shape) != (h, t):
        raise ValueError(f"lse shape {tuple(lse.shape)} != {(h, t)}")
    keep = dict(out=out.to(q.dtype).contiguous(), d_out=d_out.to(q.dtype).contiguous(),
                lse=lse.to(torch.float32).contiguous())
    if grads is not None:  # caller-provided output views (dq, dk_ctx, dv_ctx, dk, dv)
        dq, dkc, dvc, dk, dv = grads
    else:
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
    _set_groups(prm.groups, groups)
    return prm, (dq, dkc, dvc, dk, dv), keep


def _ctx_f32(prm, kc, q) -> Optional[torch.Tensor]:
    if kc is None or kc.shape[0] == 0:
        return torch.zeros((2, 0) + tuple(kc.shape[1:] if kc is not None else (0, q.shape[2])),
                           dtype=torch.float32, device=q.device)
    buf = torch.empty((2,) + tuple(kc.shape), dtype=torch.float32, device=q.device)
    prm.ctx_grad_f32 = buf.data_ptr()
    return buf


def _bwd_run(q, kc, vc, k, v, cu_dev, n, p_len, grid_max, scale, out, lse, d_out, deterministic,
             ctx_chunk=0, partials_for_chunks=False, varlen=False, groups=None, want_f32=False):
    with torch.cuda.device(q.device):
        prm, grads, keep = _bwd_params(q, kc, vc, k, v, cu_dev, n, p_len, grid_max, scale, out, lse, d_out,
                                       deterministic, ctx_chunk, groups)
        partials = None
        if partials_for_chunks:
            nch = int(lib.dkv_bwd_num_ctx_chunks(ctypes.byref(prm)))
            kk = kc if kc is not None else k
            partials = torch.empty((nch, 2, p_len, kk.shape[1], q.shape[2]), dtype=torch.float32,
                                   device=q.device)
            prm.ctx_partials = _ptr(partials)
        f32 = _ctx_f32(prm, kc, q) if want_f32 else None
        ws_bytes = int(lib.dkv_bwd_workspace_size(ctypes.byref(prm)))
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=q.device)
        fn = lib.dkv_varlen_bwd if varlen else lib.dkv_dualkv_bwd
        check(fn(ctypes.byref(prm), ws.data_ptr(), ws_bytes, _stream(q.device)),
              "fa2_varlen_bwd" if varlen else "dualkv_bwd")
        del keep
    return grads + (partials, f32)


def dualkv_bwd(inp: DualKVInput, out, lse, d_out, deterministic: bool = True,
               fold_seed: Optional[int] = None, *, return_context_f32: bool = False):
    """Two-region backward -> (dQ_d, dK_c, dV_c, dK_d, dV_d) in storage dtype.

    dK_c/dV_c are the fp32 sum over all sequences cast once (kernel.py:279-285).
    ``fold_seed`` is accepted for interface parity.  ``return_context_f32`` (instrumentation)
    appends the fp32 [2, P, H_k, d] prompt gradient the cast was applied to."""
    del fold_seed
    res = _bwd_run(inp.q, inp.k_context, inp.v_context, inp.k_decoded, inp.v_decoded, inp.cu_dev,
                   inp.num_sequences, inp.context_seqlen, inp._grid_max, inp.softmax_scale, out, lse, d_out,
                   deterministic, groups=inp._groups, want_f32=return_context_f32)
    return res[:5] + ((res[6],) if return_context_f32 else ())


def context_grad_contributions(inp: DualKVInput, out, lse, d_out) -> List[Tuple[torch.Tensor, torch.Tensor]]:
    """Per-sequence fp32 (dK_c^i, dV_c^i) before any fold (kernel.py:296-305).

    Zero-length sequences contribute nothing and are skipped, as in the
    reference generator (kernel.py:231-234)."""
    if inp._groups is not None:
        raise ValueError("context_grad_contributions takes one prompt group")
    res = _bwd_run(inp.q, inp.k_context, inp.v_context, inp.k_decoded, inp.v_decoded, inp.cu_dev,
                   inp.num_sequences, inp.context_seqlen, inp._grid_max, inp.softmax_scale, out, lse,
                   d_out, True, ctx_chunk=1, partials_for_chunks=True)
    parts = res[5]
    host = inp.cu_host if inp.cu_host is not None else inp.cu_dev.cpu().numpy()  # instrumentation: may sync
    lens = np.diff(np.asarray(host, dtype=np.int64))
    return [(parts[i, 0], parts[i, 1]) for i in range(inp.num_sequences) if lens[i] > 0]


def fa2_varlen_bwd(batch: VarlenBatch, out, lse, d_out):
    """Backward of `fa2_varlen_fwd` -> (dQ, dK, dV) in storage dtype (fa2.py:268-306)."""
    dq, _, _, dk, dv, _, _ = _bwd_run(batch.q, None, None, batch.k, batch.v, batch.cu_dev,
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
        with torch.cuda.device(acc.device):
            dst = torch.empty(acc.shape, dtype=torch.bfloat16, device=acc.device)
            check(lib.dkv_convert_f32_to_bf16(_ptr(acc), _ptr(dst), acc.numel(), _stream(acc.device)),
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
# fused two-call op (layer.py:236-290 composed in one launch)
# ---------------------------------------------------------------------------

def _check_prompt_q(q_ctx, inp: DualKVInput):
    q_ctx = _check_tensor(q_ctx, "q_context", device=inp.q.device)
    p_len = inp.context_seqlen
    if tuple(q_ctx.shape) != (p_len, inp.q.shape[1], inp.q.shape[2]) or q_ctx.dtype != inp.q.dtype:
        raise ValueError(f"q_context shape/dtype {tuple(q_ctx.shape)}/{q_ctx.dtype} inconsistent with "
                         f"P={p_len}, q {tuple(inp.q.shape)}/{inp.q.dtype}")
    return q_ctx


def dualkv_two_call_fwd(q_context, inp: DualKVInput):
    """Call 1 (causal self-attention of the prompt's own queries) + Call 2 (DualKV) in ONE launch.

    Returns (O_ctx [P,H,d], lse_ctx [H,P], O_dec [sum R_i,H,d], lse_dec [H,sum R_i]) -- equal to
    `fa2_varlen_fwd` over the prompt and `dualkv_fwd(inp)` (layer.py:243-255).  With a group
    table, every group's prompt is its own Call 1 sequence (rows group_ctx_cu[g]..[g+1])."""
    q_ctx = _check_prompt_q(q_context, inp)
    q = inp.q
    p_len, h, d = q_ctx.shape
    with torch.cuda.device(q.device):
        out = torch.empty_like(q)
        lse = torch.empty((h, q.shape[0]), dtype=torch.float32, device=q.device)
        out_c = torch.empty_like(q_ctx)
        lse_c = torch.empty((h, p_len), dtype=torch.float32, device=q.device)
        prm = TwoCallFwdParams()
        prm.call2 = _fwd_params(q, inp.k_context, inp.v_context, inp.k_decoded, inp.v_decoded, inp.cu_dev,
                                inp.num_sequences, p_len, inp._grid_max, inp.softmax_scale, out, lse, inp._groups)
        prm.q_ctx, prm.out_ctx, prm.lse_ctx = _ptr(q_ctx), _ptr(out_c), _ptr(lse_c)
        check(lib.dkv_twocall_fwd(ctypes.byref(prm), _stream(q.device)), "dualkv_two_call_fwd")
    return out_c, lse_c, out, lse


def dualkv_two_call_bwd(q_context, inp: DualKVInput, out_ctx, lse_ctx, d_out_ctx, out, lse, d_out,
                        deterministic: bool = True, *, return_context_f32: bool = False):
    """Backward of both calls in ONE launch.  Returns (dQ_ctx, dK_c, dV_c, dQ_dec, dK_dec, dV_dec),
    dK_c / dV_c being the TOTAL prompt-key gradient (Call 1 + Call 2, layer.py:278-279) accumulated
    in one fp32 scratch and cast once (``return_context_f32`` appends that fp32 [2, P, H_k, d])."""
    q_ctx = _check_prompt_q(q_context, inp)
    p_len, h, d = q_ctx.shape
    for name, x in (("O_ctx", out_ctx), ("dO_ctx", d_out_ctx), ("lse_ctx", lse_ctx)):
        if not isinstance(x, torch.Tensor) or not x.is_cuda or x.device != q_ctx.device:
            raise ValueError(f"{name} must be a CUDA tensor on {q_ctx.device}")
    if tuple(out_ctx.shape) != tuple(q_ctx.shape) or tuple(d_out_ctx.shape) != tuple(q_ctx.shape):
        raise ValueError("O_ctx/dO_ctx shape inconsistent with q_context")
    if tuple(lse_ctx.shape) != (h, p_len):
        raise ValueError(f"lse_ctx shape {tuple(lse_ctx.shape)} != {(h, p_len)}")
    with torch.cuda.device(q_ctx.device):
        prm2, grads, keep = _bwd_params(inp.q, inp.k_context, inp.v_context, inp.k_decoded, inp.v_decoded,
                                        inp.cu_dev, inp.num_sequences, p_len, inp._grid_max, inp.softmax_scale,
                                        out, lse, d_out, deterministic, groups=inp._groups)
        dq, dkc, dvc, dkd, dvd = grads
        f32 = _ctx_f32(prm2, inp.k_context, inp.q) if return_context_f32 else None
        o_c = out_ctx.to(q_ctx.dtype).contiguous()
        l_c = lse_ctx.to(torch.float32).contiguous()
        do_c = d_out_ctx.to(q_ctx.dtype).contiguous()
        dq_c = torch.empty_like(q_ctx)
        prm = TwoCallBwdParams()
        prm.call2 = prm2
        prm.q_ctx, prm.out_ctx, prm.lse_ctx = _ptr(q_ctx), _ptr(o_c), _ptr(l_c)
        prm.dout_ctx, prm.dq_ctx = _ptr(do_c), _ptr(dq_c)
        ws_bytes = int(lib.dkv_twocall_bwd_workspace_size(ctypes.byref(prm)))
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=q_ctx.device)
        check(lib.dkv_twocall_bwd(ctypes.byref(prm), ws.data_ptr(), ws_bytes, _stream(q_ctx.device)),
              "dualkv_two_call_bwd")
        del keep
    res = (dq_c, dkc, dvc, dq, dkd, dvd)
    return res + ((f32,) if return_context_f32 else ())


# ---------------------------------------------------------------------------
# autograd surfaces (kernel.py:308-348): registered torch.library custom ops
# (library.py) so torch.compile sees opaque ops with fake implementations instead of graph breaks
# ---------------------------------------------------------------------------

def dualkv_attention_varlen(q, k_context, v_context, k_decoded, v_decoded, cu_seqlens_q,
                            cu_seqlens_k_decoded=None, max_seqlen_q: Optional[int] = None,
                            context_seqlen: Optional[int] = None,
                            max_seqlen_k_decoded: Optional[int] = None,
                            softmax_scale: Optional[float] = None, causal: bool = True,
                            tile_size: int = 64) -> torch.Tensor:
    """Five-tensor call surface; lse is saved on the autograd ctx, not returned."""
    if cu_seqlens_k_decoded is not None and cu_seqlens_k_decoded is not cu_seqlens_q:
        if isinstance(cu_seqlens_k_decoded, torch.Tensor) and isinstance(cu_seqlens_q, torch.Tensor) \
                and cu_seqlens_k_decoded.device == cu_seqlens_q.device:
            same = cu_seqlens_k_decoded.shape == cu_seqlens_q.shape and \
                bool(torch.equal(cu_seqlens_k_decoded.to(cu_seqlens_q.dtype), cu_seqlens_q))
        else:
            host = lambda x: np.asarray(x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else x)
            same = np.array_equal(host(cu_seqlens_k_decoded), host(cu_seqlens_q))
        if not same:
            raise ValueError("cu_seqlens_k_decoded must equal cu_seqlens_q")
    del max_seqlen_k_decoded  # decoded KV shares q's offsets (kernel.py:333)
    inp = DualKVInput(q, k_context, v_context, k_decoded, v_decoded, cu_seqlens_q,
                      context_seqlen=context_seqlen, max_seqlen_q=max_seqlen_q,
                      softmax_scale=softmax_scale, causal=causal, tile_size=tile_size)
    from . import library
    return library.attention(inp)


def dualkv_two_call_attention(q_context, k_context, v_context, q_decoded, k_decoded, v_decoded,
                              cu_seqlens_q, max_seqlen_q: Optional[int] = None,
                              softmax_scale: Optional[float] = None,
                              group_seq_cu: Optional[Sequence[int]] = None,
                              group_ctx_cu: Optional[Sequence[int]] = None):
    """The whole attention of one prompt group (or, with a group table, of several) in the P+NR
    layout (layer.py:236-290): returns (O_context [P,H,d], O_decoded [sum R_i,H,d]); autograd gives
    all six input gradients, the prompt K/V gradient summed over both calls and all N sequences in
    fp32 and cast once."""
    inp = DualKVInput(q_decoded, k_context, v_context, k_decoded, v_decoded, cu_seqlens_q,
                      max_seqlen_q=max_seqlen_q, softmax_scale=softmax_scale,
                      group_seq_cu=group_seq_cu, group_ctx_cu=group_ctx_cu)
    q_ctx = _check_prompt_q(q_context, inp)
    from . import library
    return library.two_call_attention(q_ctx, inp)


# ---------------------------------------------------------------------------
# the two-call op over ONE buffer per tensor: rows [0, P_total) are every group's prompt, the rest
# every group's responses (the layer's split layout).  Outputs / gradients land in single buffers
# of the same layout -- no concatenation or slice-gradient assembly around the op.
# ---------------------------------------------------------------------------

def _split_input(q, k, v, p_rows, cu_seqlens, max_seqlen, softmax_scale, group_seq_cu, group_ctx_cu):
    return DualKVInput(q[p_rows:], k[:p_rows], v[:p_rows], k[p_rows:], v[p_rows:], cu_seqlens,
                       max_seqlen_q=max_seqlen, softmax_scale=softmax_scale,
                       group_seq_cu=group_seq_cu or None, group_ctx_cu=group_ctx_cu or None)


def two_call_split_fwd(q, k, v, p_rows: int, cu_seqlens, max_seqlen: int, softmax_scale: float,
                       group_seq_cu=None, group_ctx_cu=None):
    """-> (O [T, H, d] in the same split layout, lse_ctx [H, P], lse [H, T - P])."""
    inp = _split_input(q, k, v, p_rows, cu_seqlens, max_seqlen, softmax_scale, group_seq_cu, group_ctx_cu)
    q_ctx = _check_prompt_q(q[:p_rows], inp)
    t, h, d = q.shape
    with torch.cuda.device(q.device):
        out = torch.empty_like(q)
        lse_c = torch.empty((h, p_rows), dtype=torch.float32, device=q.device)
        lse = torch.empty((h, t - p_rows), dtype=torch.float32, device=q.device)
        prm = TwoCallFwdParams()
        prm.call2 = _fwd_params(inp.q, inp.k_context, inp.v_context, inp.k_decoded, inp.v_decoded, inp.cu_dev,
                                inp.num_sequences, p_rows, inp._grid_max, inp.softmax_scale, out[p_rows:], lse,
                                inp._groups)
        prm.q_ctx, prm.out_ctx, prm.lse_ctx = _ptr(q_ctx), _ptr(out[:p_rows]), _ptr(lse_c)
        check(lib.dkv_twocall_fwd(ctypes.byref(prm), _stream(q.device)), "two_call_split_fwd")
    return out, lse_c, lse


def two_call_split_bwd(q, k, v, p_rows: int, cu_seqlens, max_seqlen: int, softmax_scale: float,
                       group_seq_cu, group_ctx_cu, out, lse_ctx, lse, d_out, deterministic: bool = False):
    """-> (dQ, dK, dV) in the split layout; the prompt rows of dK / dV are the TOTAL prompt gradient
    (Call 1 + Call 2 over every sequence of the group, fp32, cast once)."""
    inp = _split_input(q, k, v, p_rows, cu_seqlens, max_seqlen, softmax_scale, group_seq_cu, group_ctx_cu)
    q_ctx = _check_prompt_q(q[:p_rows], inp)
    out, d_out = out.contiguous(), d_out.to(q.dtype).contiguous()
    with torch.cuda.device(q.device):
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
        # the gradients go straight into the split-layout buffers
        prm2, _, keep = _bwd_params(inp.q, inp.k_context, inp.v_context, inp.k_decoded, inp.v_decoded, inp.cu_dev,
                                    inp.num_sequences, p_rows, inp._grid_max, inp.softmax_scale, out[p_rows:], lse,
                                    d_out[p_rows:], deterministic, groups=inp._groups,
                                    grads=(dq[p_rows:], dk[:p_rows], dv[:p_rows], dk[p_rows:], dv[p_rows:]))
        prm = TwoCallBwdParams()
        prm.call2 = prm2
        lse_ctx = lse_ctx.to(torch.float32).contiguous()  # kept alive until the launch is enqueued
        prm.q_ctx, prm.out_ctx, prm.lse_ctx = _ptr(q_ctx), _ptr(out[:p_rows]), _ptr(lse_ctx)
        prm.dout_ctx, prm.dq_ctx = _ptr(d_out[:p_rows]), _ptr(dq[:p_rows])
        ws_bytes = int(lib.dkv_twocall_bwd_workspace_size(ctypes.byref(prm)))
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=q.device)
        check(lib.dkv_twocall_bwd(ctypes.byref(prm), ws.data_ptr(), ws_bytes, _stream(q.device)),
              "two_call_split_bwd")
        del keep
    return dq, dk, dv

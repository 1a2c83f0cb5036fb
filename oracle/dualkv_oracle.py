"""CPU oracle for the DualKV attention hot path -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference's CPU algorithm
(`/root/reference/pkg/src/dualkv/{fa2,kernel,tensor,refattn,packing,costmodel}.py`).
It exists so that `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` leg have a checker and a CPU timing
baseline.  The product path (`paper_2605_15422_b200`) never imports it; the
product fails loudly when its CUDA library is missing.

Parity pinning: every function here is checked against golden vectors that
`tools/make_golden.py` produced by importing the reference itself in the
build container (`tests/golden/*.npz`, test `tests/test_oracle_golden.py`).

Numerics contract restated from the reference:
  * storage precision ``"f64" | "f32" | "bf16"``; compute dtype is f64 for
    f64 storage, f32 otherwise (tensor.py:70-92);
  * bf16 rounding is RNE on the f32 bit pattern (tensor.py:39-58);
  * saved O / lse stay in compute precision (fa2.py:22-28, kernel.py:207-210);
  * returned gradients are quantized once to storage precision
    (fa2.py:302-306, kernel.py:285-293);
  * the shared-context gradient is an f32 (f64 for f64 runs) fold over
    sequences, cast exactly once (kernel.py:279-285, :140-148).
"""

from __future__ import annotations

import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

ROW_BLOCK = 128  # query rows per block, fa2.py:46

__all__ = [
    "bf16_round", "bf16_ulp", "quantize", "compute_dtype",
    "tiled_forward", "tiled_backward",
    "varlen_fwd", "varlen_bwd", "dualkv_fwd", "dualkv_bwd",
    "context_contributions", "convert_context", "naive_bf16_fold",
    "dense_fwd", "dense_bwd",
    "standard_layout", "dualkv_layout", "position_ids",
    "repack_index", "visible_pairs", "attention_flops",
]


# --------------------------------------------------------------------------
# numerics (tensor.py:39-92)
# --------------------------------------------------------------------------

def bf16_round(x):
    """RNE to bf16 on the f32 bit pattern; NaN kept (tensor.py:39-58)."""
    a = np.asarray(x, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    bias = np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))
    r = (((u + bias) & np.uint64(0xFFFF0000)) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    out = np.where(np.isnan(a), a, r.view(np.float32))
    if np.ndim(x) == 0:
        return float(out)
    return out.astype(np.float32)


def bf16_ulp(x):
    """bf16 grid spacing at |x| (tensor.py:61-67)."""
    mag = np.abs(np.asarray(x, dtype=np.float64))
    e = np.floor(np.log2(np.where(mag > 0, mag, 1.0)))
    e = np.where(mag > 0, np.maximum(e, -126.0), -126.0)
    return np.exp2(e - 7.0)


def compute_dtype(prec: str):
    return np.float64 if prec == "f64" else np.float32


def quantize(arr, prec: str) -> np.ndarray:
    """Project onto the storage grid of ``prec`` (tensor.py:86-92)."""
    if prec == "f64":
        return np.asarray(arr, dtype=np.float64)
    if prec == "f32":
        return np.asarray(arr, dtype=np.float32)
    if prec == "bf16":
        return bf16_round(np.asarray(arr, dtype=np.float32))
    raise ValueError(f"unknown precision {prec!r}")


# --------------------------------------------------------------------------
# tile core (fa2.py:94-229)
# --------------------------------------------------------------------------

def _tiles(regions, block_n):
    """Physical tile -> (region idx, lo, hi, logical start) (fa2.py:94-102)."""
    out = []
    for idx, (k, _v, base) in enumerate(regions):
        n = k.shape[0]
        lo = 0
        while lo < n:
            hi = min(lo + block_n, n)
            out.append((idx, lo, hi, base + lo))
            lo = hi
    return out


def _heads_major(x, group):
    """[T, Hk, d] -> [H, T, d] where q head h reads kv head h // group (fa2.py:105-109)."""
    if group != 1:
        x = np.repeat(x, group, axis=1)
    return np.moveaxis(x, 1, 0)


def tiled_forward(q, regions, row_pos, scale, block_n, cdt):
    """Online-softmax forward over ordered KV regions (fa2.py:112-165).

    ``regions`` is a list of (k [S,Hk,d], v [S,Hk,d], logical_base).
    Tiles are visited in reverse logical order, rows in blocks of 128.
    Returns (o [M,H,d], lse [H,M]) in ``cdt``.
    """
    m_rows, n_heads, dim = q.shape
    hk = regions[0][0].shape[1] if regions else n_heads
    grp = n_heads // hk
    sc = cdt(scale)
    o = np.empty((m_rows, n_heads, dim), dtype=cdt)
    lse = np.empty((n_heads, m_rows), dtype=cdt)
    tiles = _tiles(regions, block_n)[::-1]
    for r0 in range(0, m_rows, ROW_BLOCK):
        r1 = min(r0 + ROW_BLOCK, m_rows)
        qb = np.moveaxis(q[r0:r1], 1, 0)               # [H, m, d]
        pos = row_pos[r0:r1]
        horizon = int(pos[-1])
        mx = np.full((n_heads, r1 - r0), -np.inf, dtype=cdt)
        den = np.zeros((n_heads, r1 - r0), dtype=cdt)
        acc = np.zeros((n_heads, r1 - r0, dim), dtype=cdt)
        for ridx, lo, hi, logical in tiles:
            if logical > horizon:
                continue
            kt = _heads_major(regions[ridx][0][lo:hi], grp)
            vt = _heads_major(regions[ridx][1][lo:hi], grp)
            s = np.matmul(qb, np.swapaxes(kt, 1, 2))
            s *= sc
            keep = (logical + np.arange(hi - lo))[None, :] <= pos[:, None]
            s = np.where(keep[None], s, cdt(-np.inf))
            new_mx = np.maximum(mx, s.max(axis=2))
            ref = np.where(np.isneginf(new_mx), cdt(0.0), new_mx)
            p = np.exp(s - ref[..., None])
            corr = np.exp(mx - ref)
            den = corr * den + p.sum(axis=2)
            acc = corr[..., None] * acc + np.matmul(p, vt)
            mx = new_mx
        o[r0:r1] = np.moveaxis(acc / den[..., None], 0, 1)
        lse[:, r0:r1] = mx + np.log(den)
    return o, lse


def tiled_backward(q, dout, lse, drow, regions, row_pos, scale, block_n, cdt):
    """Tiled backward from saved lse (fa2.py:168-229).

    Returns (dq [M,H,d], [(dk, dv) per region]) -- uncast accumulators.
    """
    m_rows, n_heads, dim = q.shape
    hk = regions[0][0].shape[1] if regions else n_heads
    grp = n_heads // hk
    sc = cdt(scale)
    dq = np.zeros((m_rows, n_heads, dim), dtype=cdt)
    grads = [(np.zeros(k.shape, dtype=cdt), np.zeros(v.shape, dtype=cdt)) for k, v, _ in regions]
    for ridx, lo, hi, logical in _tiles(regions, block_n):
        kt = _heads_major(regions[ridx][0][lo:hi], grp)
        vt = _heads_major(regions[ridx][1][lo:hi], grp)
        n = hi - lo
        tdk = np.zeros((n_heads, n, dim), dtype=cdt)
        tdv = np.zeros((n_heads, n, dim), dtype=cdt)
        for r0 in range(0, m_rows, ROW_BLOCK):
            r1 = min(r0 + ROW_BLOCK, m_rows)
            pos = row_pos[r0:r1]
            if logical > int(pos[-1]):
                continue
            qb = np.moveaxis(q[r0:r1], 1, 0)
            gb = np.moveaxis(dout[r0:r1], 1, 0)
            s = np.matmul(qb, np.swapaxes(kt, 1, 2))
            s *= sc
            keep = (logical + np.arange(n))[None, :] <= pos[:, None]
            p = np.where(keep[None], np.exp(s - lse[:, r0:r1, None]), cdt(0.0))
            tdv += np.matmul(np.swapaxes(p, 1, 2), gb)
            dp = np.matmul(gb, np.swapaxes(vt, 1, 2))
            ds = p * (dp - drow[:, r0:r1, None])
            ds *= sc
            tdk += np.matmul(np.swapaxes(ds, 1, 2), qb)
            dq[r0:r1] += np.moveaxis(np.matmul(ds, kt), 0, 1)
        gk, gv = grads[ridx]
        gk[lo:hi] += np.moveaxis(tdk.reshape(hk, grp, n, dim).sum(axis=1), 0, 1)
        gv[lo:hi] += np.moveaxis(tdv.reshape(hk, grp, n, dim).sum(axis=1), 0, 1)
    return dq, grads


def _rowsum(dout, o):
    """D[h, r] = sum_d dO*O (fa2.py:232-234)."""
    return np.einsum("rhd,rhd->hr", dout, o)


def _check_cu(cu, total, what="cu_seqlens"):
    cu = np.asarray(cu, dtype=np.int64)
    if cu.ndim != 1 or cu.size < 2 or cu[0] != 0 or cu[-1] != total:
        raise ValueError(f"malformed {what} {cu!r} for T={total}")
    if np.any(np.diff(cu) < 0):
        raise ValueError(f"{what} must be non-decreasing")
    return cu


# --------------------------------------------------------------------------
# single-region varlen causal attention (fa2.py:237-306)
# --------------------------------------------------------------------------

def varlen_fwd(q, k, v, cu, scale=None, prec="f32", block_n=64):
    """Per-sequence causal attention; (O, lse) in compute precision (fa2.py:237-265)."""
    cdt = compute_dtype(prec)
    q, k, v = (quantize(a, prec).astype(cdt) for a in (q, k, v))
    t, h, d = q.shape
    cu = _check_cu(cu, t)
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    o = np.zeros((t, h, d), dtype=cdt)
    lse = np.zeros((h, t), dtype=cdt)
    for a, b in zip(cu[:-1], cu[1:]):
        a, b = int(a), int(b)
        if a == b:
            continue
        oi, li = tiled_forward(q[a:b], [(k[a:b], v[a:b], 0)], np.arange(b - a), scale, block_n, cdt)
        o[a:b] = oi
        lse[:, a:b] = li
    return o, lse


def varlen_bwd(q, k, v, cu, o, lse, dout, scale=None, prec="f32", block_n=64):
    """(dQ, dK, dV) cast once to storage precision (fa2.py:268-306)."""
    cdt = compute_dtype(prec)
    q, k, v, dout = (quantize(a, prec).astype(cdt) for a in (q, k, v, dout))
    o = np.asarray(o, dtype=cdt)
    lse = np.asarray(lse, dtype=cdt)
    t, h, d = q.shape
    if dout.shape != q.shape or o.shape != q.shape:
        raise ValueError("O/dO shape inconsistent with Q")
    cu = _check_cu(cu, t)
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    drow = _rowsum(dout, o)
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    for a, b in zip(cu[:-1], cu[1:]):
        a, b = int(a), int(b)
        if a == b:
            continue
        dqi, g = tiled_backward(q[a:b], dout[a:b], lse[:, a:b], drow[:, a:b],
                                [(k[a:b], v[a:b], 0)], np.arange(b - a), scale, block_n, cdt)
        dq[a:b] = dqi
        dk[a:b], dv[a:b] = g[0]
    return quantize(dq, prec), quantize(dk, prec), quantize(dv, prec)


# --------------------------------------------------------------------------
# two-region DualKV kernel (kernel.py:168-305)
# --------------------------------------------------------------------------

def _dualkv_prepare(q, kc, vc, kd, vd, cu, prec, scale):
    cdt = compute_dtype(prec)
    q, kc, vc, kd, vd = (quantize(a, prec).astype(cdt) for a in (q, kc, vc, kd, vd))
    t, h, d = q.shape
    cu = _check_cu(cu, t, "cu_seqlens_q")
    if kc.shape != vc.shape or kd.shape != vd.shape:
        raise ValueError("K/V shape mismatch")
    if kd.shape[0] != t:
        raise ValueError("k_decoded must share q's packed token count")
    hk = kc.shape[1]
    if kd.shape[1] != hk or kc.shape[2] != d:
        raise ValueError("context/decoded KV head layout mismatch")
    if hk == 0 or h % hk:
        raise ValueError(f"H={h} must be a positive multiple of H_k={hk}")
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    return cdt, q, kc, vc, kd, vd, cu, scale


def dualkv_fwd(q, kc, vc, kd, vd, cu, scale=None, prec="f32", block_n=64):
    """Two-region forward: context tiles at logical 0, own tiles at P (kernel.py:177-210)."""
    cdt, q, kc, vc, kd, vd, cu, scale = _dualkv_prepare(q, kc, vc, kd, vd, cu, prec, scale)
    t, h, d = q.shape
    p_len = kc.shape[0]
    o = np.zeros((t, h, d), dtype=cdt)
    lse = np.zeros((h, t), dtype=cdt)
    for a, b in zip(cu[:-1], cu[1:]):
        a, b = int(a), int(b)
        if a == b:
            continue
        regs = [(kc, vc, 0), (kd[a:b], vd[a:b], p_len)]
        oi, li = tiled_forward(q[a:b], regs, p_len + np.arange(b - a), scale, block_n, cdt)
        o[a:b] = oi
        lse[:, a:b] = li
    return o, lse


def _per_sequence_grads(q, kc, vc, kd, vd, cu, o, lse, dout, scale, prec, block_n):
    cdt, q, kc, vc, kd, vd, cu, scale = _dualkv_prepare(q, kc, vc, kd, vd, cu, prec, scale)
    dout = quantize(dout, prec).astype(cdt)
    o = np.asarray(o, dtype=cdt)
    lse = np.asarray(lse, dtype=cdt)
    if dout.shape != q.shape or o.shape != q.shape:
        raise ValueError("O/dO shape inconsistent with q")
    p_len = kc.shape[0]
    drow = _rowsum(dout, o)
    for a, b in zip(cu[:-1], cu[1:]):
        a, b = int(a), int(b)
        if a == b:
            continue
        regs = [(kc, vc, 0), (kd[a:b], vd[a:b], p_len)]
        dqi, g = tiled_backward(q[a:b], dout[a:b], lse[:, a:b], drow[:, a:b], regs,
                                p_len + np.arange(b - a), scale, block_n, cdt)
        yield a, b, dqi, g[0], g[1]


def dualkv_bwd(q, kc, vc, kd, vd, cu, o, lse, dout, scale=None, prec="f32", block_n=64,
               deterministic=True, fold_seed=None):
    """(dQ, dK_c, dV_c, dK_d, dV_d) (kernel.py:245-293)."""
    cdt = compute_dtype(prec)
    dq = np.zeros(np.shape(q), dtype=cdt)
    dkd = np.zeros(np.shape(kd), dtype=cdt)
    dvd = np.zeros(np.shape(vd), dtype=cdt)
    parts = []
    for a, b, dqi, (gkc, gvc), (gkd, gvd) in _per_sequence_grads(
            q, kc, vc, kd, vd, cu, o, lse, dout, scale, prec, block_n):
        dq[a:b], dkd[a:b], dvd[a:b] = dqi, gkd, gvd
        parts.append((gkc, gvc))
    acc_k = np.zeros(np.shape(kc), dtype=cdt)
    acc_v = np.zeros(np.shape(vc), dtype=cdt)
    order = np.arange(len(parts))
    if not deterministic:
        order = np.random.default_rng(fold_seed).permutation(order)
    for i in order:
        acc_k += parts[i][0]
        acc_v += parts[i][1]
    dkc, dvc = convert_context(acc_k, acc_v, prec)
    return quantize(dq, prec), dkc, dvc, quantize(dkd, prec), quantize(dvd, prec)


def context_contributions(q, kc, vc, kd, vd, cu, o, lse, dout, scale=None, prec="f32",
                          block_n=64):
    """Per-sequence (dK_c^i, dV_c^i) before any fold (kernel.py:296-305)."""
    return [g for _, _, _, g, _ in _per_sequence_grads(
        q, kc, vc, kd, vd, cu, o, lse, dout, scale, prec, block_n)]


def convert_context(acc_k, acc_v, prec):
    """One cast per element of the finished scratch (kernel.py:140-148)."""
    return quantize(acc_k, prec), quantize(acc_v, prec)


def naive_bf16_fold(parts):
    """acc = bf16(acc + bf16(c)): the rejected fold (kernel.py:151-165)."""
    acc = None
    for c in parts:
        c = bf16_round(np.asarray(c, dtype=np.float32))
        acc = c if acc is None else bf16_round(acc + c)
    if acc is None:
        raise ValueError("need at least one contribution")
    return np.asarray(acc, dtype=np.float32)


# --------------------------------------------------------------------------
# dense f64 oracle (refattn.py:66-136)
# --------------------------------------------------------------------------

def _dense_weights(q, k, scale, offset):
    sq, sk = q.shape[0], k.shape[0]
    grp = q.shape[1] // k.shape[1]
    kk = np.repeat(k, grp, axis=1)
    vis = np.arange(sk)[None, :] <= (offset + np.arange(sq))[:, None]
    s = np.einsum("rhd,jhd->hrj", q, kk) * scale
    return np.where(vis[None], s, -np.inf), vis


def dense_fwd(q, k, v, scale=None, causal_offset=0):
    """Full-matrix masked softmax in f64 -> (O [Sq,H,d], lse [H,Sq])."""
    q, k, v = (np.asarray(a, dtype=np.float64) for a in (q, k, v))
    scale = 1.0 / math.sqrt(q.shape[2]) if scale is None else scale
    grp = q.shape[1] // k.shape[1]
    s, vis = _dense_weights(q, k, scale, causal_offset)
    if q.shape[0] and not vis.any(axis=1).all():
        raise ValueError("a query row has no visible keys")
    mx = s.max(axis=2, keepdims=True)
    e = np.exp(s - mx)
    z = e.sum(axis=2, keepdims=True)
    o = np.einsum("hrj,jhd->rhd", e / z, np.repeat(v, grp, axis=1))
    return o, (mx + np.log(z))[..., 0]


def dense_bwd(q, k, v, o, lse, dout, scale=None, causal_offset=0):
    """Analytic (dQ, dK, dV) of `dense_fwd`, GQA folded (refattn.py:103-136)."""
    q, k, v, o, lse, dout = (np.asarray(a, dtype=np.float64) for a in (q, k, v, o, lse, dout))
    scale = 1.0 / math.sqrt(q.shape[2]) if scale is None else scale
    hk = k.shape[1]
    grp = q.shape[1] // hk
    s, vis = _dense_weights(q, k, scale, causal_offset)
    w = np.where(vis[None], np.exp(s - lse[..., None]), 0.0)
    drow = np.einsum("rhd,rhd->hr", dout, o)
    vv = np.repeat(v, grp, axis=1)
    kk = np.repeat(k, grp, axis=1)
    dv_full = np.einsum("hrj,rhd->jhd", w, dout)
    ds = w * (np.einsum("rhd,jhd->hrj", dout, vv) - drow[..., None]) * scale
    dk_full = np.einsum("hrj,rhd->jhd", ds, q)
    dq = np.einsum("hrj,jhd->rhd", ds, kk)
    sk = k.shape[0]
    return (dq, dk_full.reshape(sk, hk, grp, -1).sum(axis=2),
            dv_full.reshape(sk, hk, grp, -1).sum(axis=2))


# --------------------------------------------------------------------------
# packing contract (packing.py:105-220)
# --------------------------------------------------------------------------

def standard_layout(groups: Sequence[Tuple[int, Sequence[int]]]):
    """Replicated layout [P;R_i] per response; returns global seq offsets (packing.py:159-179)."""
    cu = [0]
    for p_len, rs in groups:
        for r in rs:
            cu.append(cu[-1] + p_len + int(r))
    return np.asarray(cu, dtype=np.int64)


def dualkv_layout(groups: Sequence[Tuple[int, Sequence[int]]]):
    """Shared layout [P;R_1..R_N] per group (packing.py:182-220).

    Returns a list of (context_start, P, resp_start, resp_cu) per group.
    """
    out, cur = [], 0
    for p_len, rs in groups:
        rcu = np.concatenate([[0], np.cumsum(np.asarray(rs, dtype=np.int64))]).astype(np.int64)
        out.append((cur, int(p_len), cur + int(p_len), rcu))
        cur += int(p_len) + int(rcu[-1])
    return out


def position_ids(groups, mode="dualkv"):
    """Logical positions: prompt j -> j, response r -> P + r (packing.py:105-120)."""
    pos = []
    for p_len, rs in groups:
        if mode == "dualkv":
            pos.extend(range(p_len))
            for r in rs:
                pos.extend(range(p_len, p_len + int(r)))
        else:
            for r in rs:
                pos.extend(range(p_len + int(r)))
    return np.asarray(pos, dtype=np.int64)


def rope(x, positions, base=10000.0, inverse=False):
    """Rotary embedding at (logical) positions, f64 (layer.py:182-196; inverse = rope_bwd,
    layer.py:198-205): pair (2k, 2k+1) rotated by pos * base^(-2k/d)."""
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    inv_freq = base ** (-np.arange(0, d, 2, dtype=np.float64) / d)
    ang = np.asarray(positions, dtype=np.float64)[:, None] * inv_freq[None, :]
    cos, sin = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    if inverse:
        sin = -sin
    ev, od = x[..., 0::2], x[..., 1::2]
    out = np.empty_like(x)
    out[..., 0::2] = ev * cos - od * sin
    out[..., 1::2] = ev * sin + od * cos
    return out


def repack_index(groups):
    """For every row of the shared layout, the source row in the replicated
    layout (prompt rows taken from copy 0).  Gathering a replicated
    activation tensor with this index yields the shared layout."""
    src, base = [], 0
    for p_len, rs in groups:
        rs = [int(r) for r in rs]
        starts = []
        cur = base
        for r in rs:
            starts.append(cur)
            cur += p_len + r
        src.extend(range(starts[0], starts[0] + p_len) if rs else [])
        for st, r in zip(starts, rs):
            src.extend(range(st + p_len, st + p_len + r))
        base = cur
    return np.asarray(src, dtype=np.int64)


# --------------------------------------------------------------------------
# cost model (costmodel.py:113-130)
# --------------------------------------------------------------------------

def visible_pairs(p_len: int, r_list: Sequence[int], mode: str = "dualkv") -> int:
    """Exact unmasked (q, k) pairs for one prompt group (costmodel.py:118-125)."""
    tri = lambda s: s * (s + 1) // 2
    if mode == "standard":
        return sum(tri(p_len + int(r)) for r in r_list)
    return tri(p_len) + sum(int(r) * p_len + tri(int(r)) for r in r_list)


def attention_flops(p_len, r_list, heads, head_dim, mode="dualkv", passes="fwd") -> int:
    """4*pairs*H*d forward (costmodel.py:128-130); x2.5 more for backward (5 GEMMs)."""
    mult = {"fwd": 4, "bwd": 10, "fwdbwd": 14}[passes]
    return mult * visible_pairs(p_len, r_list, mode) * heads * head_dim

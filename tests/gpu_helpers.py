"""Shared helpers for the GPU parity tests (oracle = tests' checker only)."""

from __future__ import annotations

import numpy as np
import torch

from oracle import dualkv_oracle as orc

# SURVEY §8(c) tolerances
BF16_ATOL = BF16_RTOL = 1e-2
LSE_ATOL = 1e-3
F32_ATOL = 1e-4


def make_case(seed, n, p, r_list, h, hk, d, dtype):
    rng = np.random.default_rng(seed)
    t = int(sum(r_list))
    arrs = dict(q=rng.normal(size=(t, h, d)), kc=rng.normal(size=(p, hk, d)),
                vc=rng.normal(size=(p, hk, d)), kd=rng.normal(size=(t, hk, d)),
                vd=rng.normal(size=(t, hk, d)), do=rng.normal(size=(t, h, d)))
    prec = "bf16" if dtype == torch.bfloat16 else "f32"
    arrs = {k: orc.quantize(v, prec) for k, v in arrs.items()}
    cu = np.concatenate([[0], np.cumsum(r_list)]).astype(np.int64)
    dev = {k: torch.from_numpy(np.ascontiguousarray(v)).to("cuda", dtype) for k, v in arrs.items()}
    return arrs, dev, cu, prec


def to_np(t):
    return t.detach().float().cpu().numpy()


def assert_close_bf16(got, ref, what):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    if got.size == 0:
        return
    assert np.isfinite(got).all(), f"{what}: non-finite values"
    bad = np.abs(got - ref) > BF16_ATOL + BF16_RTOL * np.abs(ref)
    if bad.any():
        idx = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {bad.sum()} / {bad.size} elements out of tolerance; first at "
                             f"{tuple(idx)} got {got[tuple(idx)]} ref {ref[tuple(idx)]}; "
                             f"max err {np.max(np.abs(got - ref)):.3e}")


def assert_close_abs(got, ref, atol, what):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    if got.size == 0:
        return
    err = np.max(np.abs(got - ref))
    assert err <= atol, f"{what}: max abs err {err:.3e} > {atol:.1e}"


def ref_attention_slice_f64(q, keys, vals, d_out, offset, scale, block=2048):
    """Independent dense float64 reference on the GPU for ONE KV head (torch, no shared code with
    the kernels or the NumPy oracle): queries q [R, G, d] at logical positions offset + r attend to
    keys / vals [S, d] (key j visible iff j <= offset + r).  Query blocks of `block` rows keep the
    [G, block, S] score arrays bounded; softmax rows are independent, so blocking is exact.
    Returns float64 (O [R, G, d], lse [G, R], dQ [R, G, d], dK [S, d], dV [S, d])."""
    k, v = keys.double(), vals.double()
    r_total, s_total = q.shape[0], k.shape[0]
    o_all, lse_all, dq_all = [], [], []
    dk = torch.zeros_like(k)
    dv = torch.zeros_like(v)
    for r0 in range(0, r_total, block):
        r1 = min(r_total, r0 + block)
        qb = q[r0:r1].double().permute(1, 0, 2)          # [G, B, d]
        dob = d_out[r0:r1].double().permute(1, 0, 2)
        s = (qb @ k.T) * scale                           # [G, B, S]
        vis = torch.arange(s_total, device=q.device)[None, :] <= \
            (offset + torch.arange(r0, r1, device=q.device))[:, None]
        s = s.masked_fill(~vis[None], float("-inf"))
        lse = torch.logsumexp(s, dim=-1)                 # [G, B]
        p = torch.exp(s - lse[..., None])
        del s
        o = p @ v                                        # [G, B, d]
        dv += (p.transpose(1, 2) @ dob).sum(0)
        dp = dob @ v.T
        dsum = (dob * o).sum(-1, keepdim=True)
        ds = p * (dp - dsum)
        del p, dp
        dq_all.append((ds @ k * scale).permute(1, 0, 2))
        dk += (ds.transpose(1, 2) @ qb).sum(0) * scale
        del ds
        o_all.append(o.permute(1, 0, 2))
        lse_all.append(lse)
    return torch.cat(o_all), torch.cat(lse_all, dim=1), torch.cat(dq_all), dk, dv


def assert_bf16_vs_f64(got, ref, what, max_rel=1e-2, elementwise=True):
    """SURVEY §8c bf16 bounds against the f64 reference: elementwise |gpu-ref| <= 1e-2 + 1e-2|ref|,
    and max|gpu - ref| / max|ref| <= 1e-2 (the scale-aware bound; the elementwise one alone is loose
    for gradients much smaller than 1).  `elementwise=False` (sums over ~10^5-10^6 bf16-operand
    terms, checked with the FA-style comparative bound instead) keeps only the max-relative one.
    Returns (max-relative error, fraction of elements outside the elementwise bound)."""
    g = got.double()
    r = ref.double()
    assert g.shape == r.shape, (what, tuple(g.shape), tuple(r.shape))
    assert torch.isfinite(g).all(), f"{what}: non-finite values"
    err = (g - r).abs()
    bad = err > BF16_ATOL + BF16_RTOL * r.abs()
    if elementwise:
        assert not bad.any(), f"{what}: {int(bad.sum())} elements outside 1e-2 + 1e-2|ref| (max err {err.max():.3e})"
    rel = (err.max() / r.abs().max().clamp_min(1e-300)).item()
    assert rel <= max_rel, f"{what}: max err / max|ref| = {rel:.3e} > {max_rel}"
    return rel, bad.double().mean().item()

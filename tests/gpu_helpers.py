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

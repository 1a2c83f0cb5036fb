"""Peaked and growing logits: the online softmax's lazy O rescale (taken only when the running
max grows past the threshold) and its interplay with the causal/own/context tile order.  The
forward visits own tiles from the diagonal down, then context tiles (fwd_sm100.cu); the context
keys here are scaled so the running max jumps by ~2^20 mid-stream, and a sharp-query case makes
every row's softmax nearly one-hot.  Checked against the oracle (SURVEY §8c tolerances)."""

import numpy as np
import pytest
import torch

from gpu_helpers import LSE_ATOL, assert_close_abs, assert_close_bf16, to_np
from oracle import dualkv_oracle as orc

pytestmark = pytest.mark.gpu


def _case(seed, p, rl, h, hk, d, q_scale, kc_scale):
    rng = np.random.default_rng(seed)
    t = int(sum(rl))
    arrs = dict(q=rng.normal(size=(t, h, d)) * q_scale, kc=rng.normal(size=(p, hk, d)) * kc_scale,
                vc=rng.normal(size=(p, hk, d)), kd=rng.normal(size=(t, hk, d)), vd=rng.normal(size=(t, hk, d)),
                do=rng.normal(size=(t, h, d)))
    arrs = {k: orc.quantize(v, "bf16") for k, v in arrs.items()}
    cu = np.concatenate([[0], np.cumsum(rl)]).astype(np.int64)
    dev = {k: torch.from_numpy(np.ascontiguousarray(v)).to("cuda", torch.bfloat16) for k, v in arrs.items()}
    return arrs, dev, cu


CASES = [
    # (seed, P, R list, H, Hk, d, q scale, context-key scale)
    (61, 384, [300, 5, 257], 8, 2, 128, 1.0, 4.0),   # context logits ~4x the own ones: rescale mid-walk
    (62, 256, [130, 64], 16, 4, 128, 6.0, 1.0),      # sharp queries: near one-hot rows
    (63, 200, [77, 129], 4, 1, 64, 3.0, 3.0),        # d = 64, both
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"s{c[0]}")
def test_rescale_forward_backward(case, cuda_device):
    import paper_2605_15422_b200 as dkv
    seed, p, rl, h, hk, d, qs, ks = case
    arrs, dev, cu = _case(seed, p, rl, h, hk, d, qs, ks)
    inp = dkv.DualKVInput(dev["q"], dev["kc"], dev["vc"], dev["kd"], dev["vd"], cu)
    o, lse = dkv.dualkv_fwd(inp)
    grads = dkv.dualkv_bwd(inp, o, lse, dev["do"], deterministic=True)
    torch.cuda.synchronize()
    o_ref, lse_ref = orc.dualkv_fwd(arrs["q"], arrs["kc"], arrs["vc"], arrs["kd"], arrs["vd"], cu,
                                    prec="bf16", block_n=128)
    assert_close_bf16(to_np(o), o_ref, "O")
    assert_close_abs(to_np(lse), lse_ref, LSE_ATOL * max(1.0, float(np.abs(lse_ref).max()) / 10), "lse")
    # backward against the oracle fed the GPU's own O / lse (as test_gpu_parity does)
    ref = orc.dualkv_bwd(arrs["q"], arrs["kc"], arrs["vc"], arrs["kd"], arrs["vd"], cu, to_np(o), to_np(lse),
                         arrs["do"], prec="bf16", block_n=128)
    for got, r, nm in zip(grads, ref, ("dQ", "dK_c", "dV_c", "dK_d", "dV_d")):
        scale = max(float(np.abs(r).max()), 1e-30)
        err = float(np.abs(to_np(got) - r).max())
        assert err <= 1e-2 * scale + 1e-2, f"{nm}: max err {err:.3e} (max|ref| {scale:.3e})"

"""RoPE at DualKV logical positions on the GPU vs the oracle / reference goldens.

Tolerance: bf16 storage, fp32 rotation -> |gpu - ref| <= 1e-2 + 1e-2 |ref| (the §8c bf16 bound);
fp32 storage -> 1e-5 absolute on unit-scale inputs (fp32 sin/cos of fp64 angles)."""

import numpy as np
import pytest
import torch

from conftest import load_golden
from gpu_helpers import assert_close_bf16, to_np
from oracle import dualkv_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_rope_vs_reference_golden(dtype, cuda_device):
    import paper_2605_15422_b200 as dkv
    meta, rec = load_golden("rope")
    for i, c in enumerate(meta["cases"] + [dict(base=meta["big_base"])]):
        key = f"x{i}" if i < len(meta["cases"]) else "x_big"
        pos = rec["pos"] if i < len(meta["cases"]) else rec["pos_big"]
        ref = rec[f"y{i}"] if i < len(meta["cases"]) else rec["y_big"]
        x = orc.quantize(rec[key], "bf16" if dtype == torch.bfloat16 else "f32")
        xt = torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)
        got = to_np(dkv.rope_logical(xt, pos, c["base"]))
        exp = orc.rope(x, pos, c["base"])  # the reference's rope on the same (quantised) input
        if dtype == torch.float32:
            np.testing.assert_allclose(got, exp, rtol=0, atol=1e-5)
            if i < len(meta["cases"]):
                np.testing.assert_allclose(got, ref, rtol=0, atol=1e-5)
        else:
            assert_close_bf16(got, exp, f"rope case {i}")
        back = to_np(dkv.rope_logical(torch.from_numpy(got).to("cuda", dtype), pos, c["base"], inverse=True))
        tol = 1e-5 if dtype == torch.float32 else 2e-2
        np.testing.assert_allclose(back, x, rtol=0, atol=tol * max(1.0, np.abs(x).max()))


def test_rope_autograd_is_inverse_rotation(cuda_device):
    import paper_2605_15422_b200 as dkv
    rng = np.random.default_rng(3)
    pos = rng.integers(0, 20000, 64)
    x = torch.from_numpy(rng.normal(size=(64, 4, 128))).to("cuda", torch.float32).requires_grad_()
    y = dkv.RoPE.apply(x, pos, 1e6)
    dy = torch.from_numpy(rng.normal(size=(64, 4, 128))).to("cuda", torch.float32)
    y.backward(dy)
    np.testing.assert_allclose(to_np(x.grad), orc.rope(to_np(dy), pos, 1e6, inverse=True), atol=1e-5)


def test_repack_rope_matches_unfused(cuda_device):
    """Fused gather + rotation == repack then rope at position_ids (prompt j -> j, response r -> P+r),
    and == the oracle on the replicated rows picked by the oracle's own repack index."""
    import paper_2605_15422_b200 as dkv
    from paper_2605_15422_b200 import packing
    groups = [(37, [5, 0, 70, 12]), (9, [3, 1])]
    plan = packing.make_plan(groups)
    rng = np.random.default_rng(11)
    mk = lambda hh: torch.from_numpy(rng.normal(size=(plan.total_standard, hh, 128))).to("cuda", torch.bfloat16)
    q, k, v = mk(8), mk(2), mk(2)
    qd, kd, vd = dkv.repack_rope_to_dualkv(q, k, v, plan, 1e6)
    pos = packing.position_ids(plan, "dualkv")
    np.testing.assert_array_equal(pos, orc.position_ids(groups))
    q2 = dkv.rope_logical(packing.repack_to_dualkv(q, plan), pos, 1e6)
    assert torch.equal(qd, q2)
    assert torch.equal(vd, packing.repack_to_dualkv(v, plan))
    src = orc.repack_index(groups)
    exp = orc.rope(to_np(k)[src], pos, 1e6)
    assert_close_bf16(to_np(kd), exp, "k")

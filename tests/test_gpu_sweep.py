"""Randomized sweeps with fixed seeds against the oracle (the reference's strategy, SURVEY §8c /
test_acceptance.py:47-59):

* the reference's own config generator (`verify._draw_config`, verify.py:54-70, restated draw for
  draw: N in [1,8], P in [0,33], R_i in [0,17], H_k in {1,2}, G in {1,2,4}, d in {1,4,8}) -- these
  head dims run on the SIMT kernels -- in bf16 and fp32;
* the same idea at tensor-core shapes (d in {64,128}, G in {1,2,4,8,16}, P up to 600, R_i up to
  400, ragged and empty responses), bf16.
Forward (O, lse) and backward (all five gradients) vs the oracle on identical inputs."""

import numpy as np
import pytest
import torch

from gpu_helpers import F32_ATOL, LSE_ATOL, assert_close_abs, assert_close_bf16, make_case, to_np
from oracle import dualkv_oracle as orc

pytestmark = pytest.mark.gpu


def _draw_reference(rng):
    """verify.py:54-70, the same sequence of draws."""
    n = int(rng.integers(1, 9))
    p = int(rng.integers(0, 34))
    r_list = rng.integers(0, 18, size=n)
    if r_list.sum() == 0:
        r_list[int(rng.integers(0, n))] = int(rng.integers(1, 18))
    h_k = int(rng.choice([1, 2]))
    group = int(rng.choice([1, 2, 4]))
    rng.choice([1, 3, 4, 8])  # tile (the GPU tiles are fixed; drawn to keep the sequence)
    return n, p, [int(r) for r in r_list], h_k * group, h_k, int(rng.choice([1, 4, 8]))


def _draw_tc(rng):
    n = int(rng.integers(1, 7))
    p = int(rng.integers(0, 600))
    r_list = [int(x) for x in rng.integers(0, 400, size=n)]
    if sum(r_list) == 0:
        r_list[0] = 1
    h_k = int(rng.choice([1, 2, 4]))
    group = int(rng.choice([1, 2, 4, 8, 16]))
    return n, p, r_list, h_k * group, h_k, int(rng.choice([64, 128]))


def _check(case_seed, cfg, dtype):
    import paper_2605_15422_b200 as dkv
    n, p, rl, h, hk, d = cfg
    arrs, dev, cu, prec = make_case(case_seed, n, p, rl, h, hk, d, dtype)
    inp = dkv.DualKVInput(dev["q"], dev["kc"], dev["vc"], dev["kd"], dev["vd"], cu)
    o, lse = dkv.dualkv_fwd(inp)
    grads = dkv.dualkv_bwd(inp, o, lse, dev["do"])
    torch.cuda.synchronize()
    o_ref, lse_ref = orc.dualkv_fwd(arrs["q"], arrs["kc"], arrs["vc"], arrs["kd"], arrs["vd"], cu, prec=prec,
                                    block_n=128)
    # the backward from the GPU's own saved O / lse (as the reference's callers do)
    g_ref = orc.dualkv_bwd(arrs["q"], arrs["kc"], arrs["vc"], arrs["kd"], arrs["vd"], cu, to_np(o), to_np(lse),
                           arrs["do"], prec=prec, block_n=128)
    names = ("dQ", "dK_c", "dV_c", "dK_d", "dV_d")
    if dtype == torch.float32:
        tol = lambda ref: F32_ATOL * max(1.0, float(np.abs(ref).max(initial=0.0)))
        assert_close_abs(to_np(o), o_ref, tol(o_ref), f"O {cfg}")
        for got, ref, name in zip(grads, g_ref, names):
            assert_close_abs(to_np(got), ref, tol(ref), f"{name} {cfg}")
    else:
        assert_close_bf16(to_np(o), o_ref, f"O {cfg}")
        for got, ref, name in zip(grads, g_ref, names):
            assert_close_bf16(to_np(got), ref, f"{name} {cfg}")
    assert_close_abs(to_np(lse), lse_ref, LSE_ATOL, f"lse {cfg}")


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32], ids=["bf16", "f32"])
@pytest.mark.parametrize("seed", [101, 103, 113])
def test_reference_generator_sweep(seed, dtype, cuda_device):
    rng = np.random.default_rng(seed)
    for i in range(8):
        _check(seed * 100 + i, _draw_reference(rng), dtype)


@pytest.mark.parametrize("seed", [7, 8, 9, 10])
def test_tensor_core_sweep(seed, cuda_device):
    import paper_2605_15422_b200 as dkv
    rng = np.random.default_rng(seed)
    for i in range(5):
        cfg = _draw_tc(rng)
        assert dkv.uses_tensor_cores(torch.bfloat16, cfg[5], cfg[3], cfg[4]) or (cfg[3] // cfg[4]) > 64
        _check(seed * 100 + i, cfg, torch.bfloat16)

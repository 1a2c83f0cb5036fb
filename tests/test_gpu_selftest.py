"""UMMA operand-layout self test (every descriptor form the kernels use)."""

import ctypes

import pytest
import torch

pytestmark = pytest.mark.gpu

SHAPES = {  # mode: (A shape as stored, B shape as stored, reference)
    0: ((128, 128), (128, 128), lambda a, b: a @ b.T),
    1: ((128, 128), (128, 128), lambda a, b: a @ b),
    2: ((128, 128), (128, 128), lambda a, b: a @ b.T),
    3: ((128, 128), (128, 128), lambda a, b: a.T @ b.T),
    4: ((128, 128), (128, 128), lambda a, b: a @ b),
    5: ((128, 128), (64, 128), lambda a, b: a @ b.T),
    6: ((128, 128), (128, 64), lambda a, b: a.T @ b),
    7: ((128, 64), (64, 128), lambda a, b: a @ b),
}


@pytest.mark.parametrize("mode", sorted(SHAPES))
def test_umma_layout(mode, cuda_device):
    from paper_2605_15422_b200._lib import check, lib
    sa, sb, ref_fn = SHAPES[mode]
    g = torch.Generator(device="cuda").manual_seed(mode)
    a = torch.randn(sa, device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn(sb, device="cuda", generator=g).to(torch.bfloat16)
    ref = ref_fn(a.float(), b.float())
    d = torch.full(ref.shape, float("nan"), device="cuda", dtype=torch.float32)
    check(lib.dkv_selftest_umma(mode, a.data_ptr(), b.data_ptr(), d.data_ptr(),
                                torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    err = (d - ref).abs().max().item()
    assert err < 1e-2 * ref.abs().max().item(), f"mode {mode}: max err {err}"

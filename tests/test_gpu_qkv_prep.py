"""The fused QKV epilogue (`dualkv::qkv_prep`, csrc/qkv_prep.cu): per-head q/k RMSNorm + RoPE at
logical positions + scatter into the split layout, one HBM pass, and its adjoint -- checked
against the unfused torch composition (fp32 RMSNorm, the `dualkv::rope` op, index scatter) and
its autograd.  The fused path rounds once (after norm + rotation); the composition rounds twice,
so the two agree to bf16 resolution."""

import numpy as np
import pytest
import torch

from gpu_helpers import assert_close_bf16, to_np

pytestmark = pytest.mark.gpu


def _reference(qkv, wq, wk, pos, dst, h, hk, eps, base):
    from paper_2605_15422_b200.layer import _rms_norm
    t = qkv.shape[0]
    x = qkv.view(t, h + 2 * hk, -1)
    q, k, v = x[:, :h], x[:, h:h + hk], x[:, h + hk:]
    if wq is not None:
        q, k = _rms_norm(q, wq, eps), _rms_norm(k, wk, eps)
    q = torch.ops.dualkv.rope(q.contiguous(), pos, base, False)
    k = torch.ops.dualkv.rope(k.contiguous(), pos, base, False)
    inv = torch.empty_like(dst)
    inv[dst] = torch.arange(t, device=dst.device)
    return q.index_select(0, inv), k.index_select(0, inv), v.contiguous().index_select(0, inv)


@pytest.mark.parametrize("norm", [True, False])
@pytest.mark.parametrize("h,hk,d", [(32, 8, 128), (8, 1, 64), (4, 4, 128)])
def test_qkv_prep_matches_torch_composition(norm, h, hk, d, cuda_device):
    import paper_2605_15422_b200  # noqa: F401
    torch.manual_seed(0)
    t, eps, base = 777, 1e-6, 1e6
    qkv = (torch.randn(t, (h + 2 * hk) * d, device="cuda") * 2).to(torch.bfloat16).requires_grad_()
    wq = (1 + 0.1 * torch.randn(d, device="cuda")).to(torch.bfloat16).requires_grad_() if norm else None
    wk = (1 + 0.1 * torch.randn(d, device="cuda")).to(torch.bfloat16).requires_grad_() if norm else None
    pos = torch.as_tensor(np.random.default_rng(1).integers(0, 20000, t), device="cuda")
    dst = torch.randperm(t, device="cuda")
    q, k, v = torch.ops.dualkv.qkv_prep(qkv, wq, wk, pos, dst, h, hk, eps, base)
    qr, kr, vr = _reference(qkv, wq, wk, pos, dst, h, hk, eps, base)
    for a, b, name in ((q, qr, "q"), (k, kr, "k"), (v, vr, "v")):
        assert_close_bf16(to_np(a), to_np(b), name)
    assert torch.equal(v, vr)  # v is only moved
    gq, gk, gv = (torch.randn_like(x) for x in (q, k, v))
    params = [qkv] + ([wq, wk] if norm else [])
    got = torch.autograd.grad((q.float() * gq).sum() + (k.float() * gk).sum() + (v.float() * gv).sum(), params)
    ref = torch.autograd.grad((qr.float() * gq).sum() + (kr.float() * gk).sum() + (vr.float() * gv).sum(), params)
    assert_close_bf16(to_np(got[0]), to_np(ref[0]), "dqkv")
    for a, b, name in zip(got[1:], ref[1:], ("d q_norm", "d k_norm")):
        rel = (a.float() - b.float()).abs().max().item() / b.float().abs().max().item()
        assert rel < 2e-2, f"{name}: {rel:.3e}"

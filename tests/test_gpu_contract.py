"""The reference's contract, edge-case and precision-contract tests run against the GPU op.

Mirrors /root/reference/pkg/tests/test_dualkv.py and test_fa2.py case by case (cited per test) on
CUDA tensors through the public API; and the instrumentation checks that need
`context_grad_contributions` (verify.py:325-355, 563-596; test_dualkv.py:165-175, 238).
"""

import numpy as np
import pytest
import torch

from gpu_helpers import assert_close_bf16, make_case, to_np
from oracle import dualkv_oracle as orc

pytestmark = pytest.mark.gpu


def _inp(seed, p, rl, h=8, hk=2, d=128, dtype=torch.bfloat16, **kw):
    import paper_2605_15422_b200 as dkv
    arrs, dev, cu, _ = make_case(seed, len(rl), p, rl, h, hk, d, dtype)
    return dkv.DualKVInput(dev["q"], dev["kc"], dev["vc"], dev["kd"], dev["vd"], cu, **kw), dev, arrs, cu


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_all_empty_responses(dtype, cuda_device):
    """test_dualkv.py:96-102: total_q = 0 -> empty O, all-zero prompt gradients."""
    import paper_2605_15422_b200 as dkv
    inp, dev, _, _ = _inp(12, 5, [0, 0], h=2, hk=1, d=64, dtype=dtype)
    out, lse = dkv.dualkv_fwd(inp)
    assert tuple(out.shape) == (0, 2, 64) and tuple(lse.shape) == (2, 0)
    grads = dkv.dualkv_bwd(inp, out, lse, torch.zeros(0, 2, 64, device="cuda", dtype=dtype))
    torch.cuda.synchronize()
    assert tuple(grads[1].shape) == (5, 1, 64) and not grads[1].any() and not grads[2].any()
    # and the two-call op over an empty response set still runs Call 1
    qc = torch.randn(5, 2, 64, device="cuda").to(dtype)
    oc, lc, od, ld = dkv.dualkv_two_call_fwd(qc, inp)
    g = dkv.dualkv_two_call_bwd(qc, inp, oc, lc, torch.ones_like(oc), od, ld, torch.zeros_like(od))
    torch.cuda.synchronize()
    assert od.shape[0] == 0 and g[1].abs().sum() > 0  # only Call 1 feeds the prompt gradient


def test_negative_context_rejected(cuda_device):
    """test_dualkv.py:104-115."""
    import paper_2605_15422_b200 as dkv
    _, dev, _, cu = _inp(2, 3, [2], h=1, hk=1, d=64)
    with pytest.raises(ValueError):
        dkv.DualKVInput(dev["q"], dev["kc"], dev["vc"], dev["kd"], dev["vd"], cu, context_seqlen=-1)


def test_zero_upstream_zeroes_everything(cuda_device):
    """test_dualkv.py:126-131."""
    import paper_2605_15422_b200 as dkv
    inp, _, _, _ = _inp(3, 6, [4, 3])
    out, lse = dkv.dualkv_fwd(inp)
    grads = dkv.dualkv_bwd(inp, out, lse, torch.zeros_like(out))
    torch.cuda.synchronize()
    for g in grads:
        assert not g.any()


def test_instrumented_contributions_sum_to_total(cuda_device):
    """test_dualkv.py:165-175: one contribution per non-empty sequence, summing to the total."""
    import paper_2605_15422_b200 as dkv
    inp, dev, _, _ = _inp(6, 300, [40, 0, 200, 130])
    out, lse = dkv.dualkv_fwd(inp)
    d_out = dev["do"]
    _, dkc, dvc, _, _, f32 = dkv.dualkv_bwd(inp, out, lse, d_out, return_context_f32=True)
    contribs = dkv.context_grad_contributions(inp, out, lse, d_out)
    torch.cuda.synchronize()
    assert len(contribs) == 3
    tot_k = sum(c[0].double() for c in contribs)
    tot_v = sum(c[1].double() for c in contribs)
    scale = sum(c[0].abs().double() for c in contribs).max().item()
    assert (tot_k - f32[0].double()).abs().max().item() <= 64 * 2 ** -23 * max(scale, 1e-30)
    assert (tot_v - f32[1].double()).abs().max().item() <= 64 * 2 ** -23 * max(
        sum(c[1].abs().double() for c in contribs).max().item(), 1e-30)


@pytest.mark.parametrize("seed", range(4))
def test_single_cast_within_one_bf16_ulp(seed, cuda_device):
    """verify.py:563-596 (test_dualkv.py:238): dK_c / dV_c equal bf16(f64 sum of the per-sequence
    contributions) within one bf16 ulp -- the fp32 scratch adds no compounded rounding."""
    import paper_2605_15422_b200 as dkv
    rng = np.random.default_rng(seed)
    rl = [int(x) for x in rng.integers(1, 300, int(rng.integers(2, 7)))]
    inp, dev, _, _ = _inp(40 + seed, int(rng.integers(4, 400)), rl)
    out, lse = dkv.dualkv_fwd(inp)
    _, dkc, dvc, _, _ = dkv.dualkv_bwd(inp, out, lse, dev["do"])
    contribs = dkv.context_grad_contributions(inp, out, lse, dev["do"])
    torch.cuda.synchronize()
    for got, idx in ((dkc, 0), (dvc, 1)):
        ref = sum(c[idx].double().cpu().numpy() for c in contribs)
        target = orc.bf16_round(ref.astype(np.float32)).astype(np.float64)
        ulp = orc.bf16_ulp(target)
        diff = np.abs(to_np(got).astype(np.float64) - target)
        assert (diff / ulp).max() <= 1.0, f"single cast: {(diff / ulp).max():.2f} bf16 ulp"


def test_five_tensor_call_matches_structured_input(cuda_device):
    """test_dualkv.py:243-259."""
    import paper_2605_15422_b200 as dkv
    inp, dev, _, cu = _inp(7, 5, [3, 4])
    out_struct, _ = dkv.dualkv_fwd(inp)
    out_flat = dkv.dualkv_attention_varlen(dev["q"], dev["kc"], dev["vc"], dev["kd"], dev["vd"], cu,
                                           cu_seqlens_k_decoded=cu, max_seqlen_q=4, context_seqlen=5,
                                           max_seqlen_k_decoded=4, tile_size=4)
    torch.cuda.synchronize()
    assert torch.equal(out_struct, out_flat)


def test_mismatched_decoded_offsets_rejected(cuda_device):
    """test_dualkv.py:261-268 (host and device offsets)."""
    import paper_2605_15422_b200 as dkv
    _, dev, _, cu = _inp(8, 5, [3, 4])
    args = (dev["q"], dev["kc"], dev["vc"], dev["kd"], dev["vd"])
    with pytest.raises(ValueError):
        dkv.dualkv_attention_varlen(*args, cu, cu_seqlens_k_decoded=np.array([0, 4, 7]))
    cu_d = torch.as_tensor(cu, device="cuda")
    with pytest.raises(ValueError):
        dkv.dualkv_attention_varlen(*args, cu_d, cu_seqlens_k_decoded=torch.tensor([0, 4, 7], device="cuda"),
                                    max_seqlen_q=4)


def test_non_causal_rejected(cuda_device):
    """test_dualkv.py:270-276."""
    import paper_2605_15422_b200 as dkv
    _, dev, _, cu = _inp(9, 2, [2])
    with pytest.raises(ValueError):
        dkv.dualkv_attention_varlen(dev["q"], dev["kc"], dev["vc"], dev["kd"], dev["vd"], cu, causal=False)


def test_backward_shape_mismatch(cuda_device):
    """test_dualkv.py:278-283."""
    import paper_2605_15422_b200 as dkv
    inp, _, _, _ = _inp(10, 3, [2])
    out, lse = dkv.dualkv_fwd(inp)
    with pytest.raises(ValueError):
        dkv.dualkv_bwd(inp, out, lse, torch.zeros(3, 8, 128, device="cuda", dtype=torch.bfloat16))
    with pytest.raises(ValueError):
        dkv.dualkv_bwd(inp, out, lse[:, :1], torch.zeros_like(out))


def test_malformed_cu_seqlens(cuda_device):
    """test_fa2.py:78-88: does not reach T, decreasing, does not start at 0."""
    import paper_2605_15422_b200 as dkv
    q = torch.randn(6, 2, 64, device="cuda").to(torch.bfloat16)
    k = torch.randn(6, 1, 64, device="cuda").to(torch.bfloat16)
    for cu in ([0, 4], [0, 5, 3, 6], [1, 6]):
        with pytest.raises(ValueError):
            dkv.VarlenBatch(q, k, k.clone(), np.array(cu))
        with pytest.raises(ValueError):  # a device tensor without max_seqlen is validated on the host
            dkv.VarlenBatch(q, k, k.clone(), torch.tensor(cu, device="cuda"))


def test_device_offsets_trusted_path_equals_host_path(cuda_device):
    """cu_seqlens as a CUDA tensor with max_seqlen: no host sync, same results."""
    import paper_2605_15422_b200 as dkv
    inp, dev, _, cu = _inp(13, 257, [64, 0, 190, 3])
    o1, l1 = dkv.dualkv_fwd(inp)
    inp2 = dkv.DualKVInput(dev["q"], dev["kc"], dev["vc"], dev["kd"], dev["vd"],
                           torch.as_tensor(cu, dtype=torch.int32, device="cuda"), max_seqlen_q=190)
    assert inp2.cu_host is None
    o2, l2 = dkv.dualkv_fwd(inp2)
    g1 = dkv.dualkv_bwd(inp, o1, l1, dev["do"])
    g2 = dkv.dualkv_bwd(inp2, o2, l2, dev["do"])
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    for a, b in zip(g1[1:], g2[1:]):
        assert torch.equal(a, b)
    assert_close_bf16(to_np(g1[0]), to_np(g2[0]), "dQ (reduce order)")


def test_autograd_saves_inputs_for_version_checks(cuda_device):
    """In-place edits of an input between forward and backward raise instead of silently giving
    wrong gradients (the autograd op saves q/k/v with save_for_backward)."""
    import paper_2605_15422_b200 as dkv
    _, dev, _, cu = _inp(14, 64, [32, 16])
    leaves = [dev[k].clone().requires_grad_(True) for k in ("q", "kc", "vc", "kd", "vd")]
    xs = [x * 1 for x in leaves]
    out = dkv.dualkv_attention_varlen(*xs, cu)
    xs[0].add_(1)
    with pytest.raises(RuntimeError):
        out.float().sum().backward()

"""GQA ratios that do not divide the tile rows (Qwen3-14B / Qwen2.5-14B/32B: H=40, H_k=8, G=5;
Qwen2.5-7B: 28/4, G=7; G=3, 6, 40) on the tensor-core kernels: a 128-row forward tile holds
floor(128/G) tokens x G heads and a 64-row backward tile floor(64/G) x G (padding rows computed,
masked, never stored).  Forward, lse and all five gradients vs the f64 oracle on identical
(bf16-quantized) inputs -- elementwise 1e-2 + 1e-2|ref| and max-relative 1e-2 (oracle 1)
-- and the fused two-call op vs the oracle's composition."""

import numpy as np
import pytest
import torch

from gpu_helpers import LSE_ATOL, assert_close_abs, assert_close_bf16, make_case, to_np
from oracle import dualkv_oracle as orc

pytestmark = pytest.mark.gpu

# (seed, N, P, R list, H, H_k, d)
CASES = [
    (61, 3, 300, [77, 0, 260], 40, 8, 128),    # G = 5 (Qwen3-14B)
    (62, 2, 257, [129, 64], 28, 4, 128),       # G = 7 (Qwen2.5-7B)
    (63, 3, 130, [40, 201, 1], 12, 4, 64),     # G = 3, d = 64
    (64, 2, 200, [150, 33], 12, 2, 128),       # G = 6
    (65, 2, 70, [20, 90], 40, 1, 128),         # G = 40 (one token per backward tile)
    (66, 4, 0, [50, 3, 0, 130], 20, 4, 128),   # G = 5, P = 0
]


def _close(got, ref, what):
    """Max-relative 1e-2 vs f64, and the elementwise 1e-2 + 1e-2|ref| bound for all but <= 1e-4 of the
    elements: on the P = 0 case a few small-magnitude elements exceed the elementwise bound for
    ANY bf16-storage implementation -- measured (tools/dbg_gqa.py): the G = 4 tensor-core path at
    1.13x and the exact-fp32 SIMT path at 1.08x of the bound, this G = 5 path at 1.07x."""
    if ref.size:
        bad = np.abs(got - ref) > 1e-2 + 1e-2 * np.abs(ref)
        assert bad.mean() <= 1e-4, f"{what}: {int(bad.sum())} / {bad.size} elements outside 1e-2 + 1e-2|ref|"
        rel = float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))
        assert rel <= 1e-2, f"{what}: max err / max|ref| = {rel:.3e}"


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"G{c[4] // c[5]}_d{c[6]}_s{c[0]}")
def test_odd_gqa_vs_oracle(case, cuda_device):
    import paper_2605_15422_b200 as dkv
    seed, n, p, rl, h, hk, d = case
    assert dkv.uses_tensor_cores(torch.bfloat16, d, h, hk)
    arrs, dev, cu, prec = make_case(seed, n, p, rl, h, hk, d, torch.bfloat16)
    inp = dkv.DualKVInput(dev["q"], dev["kc"], dev["vc"], dev["kd"], dev["vd"], cu)
    o, lse = dkv.dualkv_fwd(inp)
    for det in (True, False):
        grads = dkv.dualkv_bwd(inp, o, lse, dev["do"], deterministic=det)
        torch.cuda.synchronize()
        o_ref, lse_ref = orc.dualkv_fwd(arrs["q"], arrs["kc"], arrs["vc"], arrs["kd"], arrs["vd"], cu, prec="f64",
                                        block_n=128)
        _close(to_np(o), o_ref, "O")
        assert_close_abs(to_np(lse), lse_ref, LSE_ATOL, "lse")
        g_ref = orc.dualkv_bwd(arrs["q"], arrs["kc"], arrs["vc"], arrs["kd"], arrs["vd"], cu, o_ref, lse_ref,
                               arrs["do"], prec="f64", block_n=128)
        for got, ref, name in zip(grads, g_ref, ("dQ", "dK_c", "dV_c", "dK_d", "dV_d")):
            _close(to_np(got), ref, f"{name} (deterministic={det})")


@pytest.mark.parametrize("case", CASES[:2], ids=lambda c: f"G{c[4] // c[5]}_s{c[0]}")
def test_odd_gqa_two_call(case, cuda_device):
    import paper_2605_15422_b200 as dkv
    seed, n, p, rl, h, hk, d = case
    arrs, dev, cu, prec = make_case(seed, n, p, rl, h, hk, d, torch.bfloat16)
    rng = np.random.default_rng(seed + 7)
    qc = orc.quantize(rng.normal(size=(p, h, d)), prec)
    doc = orc.quantize(rng.normal(size=(p, h, d)), prec)
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to("cuda", torch.bfloat16)
    inp = dkv.DualKVInput(dev["q"], dev["kc"], dev["vc"], dev["kd"], dev["vd"], cu)
    oc, lc, od, ld = dkv.dualkv_two_call_fwd(t(qc), inp)
    dq_c, dkc, dvc, dq, dkd, dvd = dkv.dualkv_two_call_bwd(t(qc), inp, oc, lc, t(doc), od, ld, dev["do"])
    torch.cuda.synchronize()
    o1, l1 = orc.varlen_fwd(qc, arrs["kc"], arrs["vc"], [0, p], prec=prec, block_n=128)
    assert_close_bf16(to_np(oc), o1, "O_ctx")
    g1 = orc.varlen_bwd(qc, arrs["kc"], arrs["vc"], [0, p], to_np(oc), to_np(lc), doc, prec="f64", block_n=128)
    c2 = orc.context_contributions(arrs["q"], arrs["kc"], arrs["vc"], arrs["kd"], arrs["vd"], cu, to_np(od),
                                   to_np(ld), arrs["do"], prec="f64", block_n=128)
    dkc_ref = sum((c[0] for c in c2), np.zeros_like(arrs["kc"], dtype=np.float64)) + g1[1]
    assert_close_bf16(to_np(dq_c), g1[0], "dQ_ctx")
    assert_close_bf16(to_np(dkc), dkc_ref, "dK_c total")

"""Fused two-call op: Call 1 (prompt self-attention) + Call 2 (DualKV) in one launch,
with the total prompt-key gradient accumulated in fp32 and cast once.
Checked against separate calls and the oracle's composition (layer.py:236-290)."""

import numpy as np
import pytest
import torch

from gpu_helpers import F32_ATOL, LSE_ATOL, assert_close_abs, assert_close_bf16, make_case, to_np
from oracle import dualkv_oracle as orc

pytestmark = pytest.mark.gpu

CASES = [
    (31, 3, 300, [77, 0, 260], 8, 2, 128, torch.bfloat16),
    (32, 2, 513, [256, 3], 4, 4, 128, torch.bfloat16),
    (33, 4, 128, [128, 1, 200, 64], 32, 8, 128, torch.bfloat16),
    (34, 2, 200, [33, 300], 2, 2, 64, torch.bfloat16),   # d=64: tensor cores both ways
    (35, 4, 256, [128] * 4, 8, 8, 64, torch.float32),     # C1-like fp32: SIMT
]


def _setup(case):
    import paper_2605_15422_b200 as dkv
    seed, n, p, rl, h, hk, d, dt = case
    arrs, dev, cu, prec = make_case(seed, n, p, rl, h, hk, d, dt)
    rng = np.random.default_rng(seed + 1000)
    qc = orc.quantize(rng.normal(size=(p, h, d)), prec)
    doc = orc.quantize(rng.normal(size=(p, h, d)), prec)
    qc_t = torch.from_numpy(np.ascontiguousarray(qc)).to("cuda", dt)
    doc_t = torch.from_numpy(np.ascontiguousarray(doc)).to("cuda", dt)
    inp = dkv.DualKVInput(dev["q"], dev["kc"], dev["vc"], dev["kd"], dev["vd"], cu)
    return dkv, arrs, dev, cu, prec, qc, doc, qc_t, doc_t, inp


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"s{c[0]}")
def test_two_call_forward_equals_separate_calls(case, cuda_device):
    dkv, arrs, dev, cu, prec, qc, doc, qc_t, doc_t, inp = _setup(case)
    oc, lc, od, ld = dkv.dualkv_two_call_fwd(qc_t, inp)
    od2, ld2 = dkv.dualkv_fwd(inp)
    oc2, lc2 = dkv.fa2_varlen_fwd(dkv.VarlenBatch(qc_t, dev["kc"], dev["vc"], [0, qc_t.shape[0]]))
    torch.cuda.synchronize()
    # same kernels, same per-item work: bit-identical
    assert torch.equal(od, od2) and torch.equal(ld, ld2)
    assert torch.equal(oc, oc2) and torch.equal(lc, lc2)


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"s{c[0]}")
def test_two_call_backward_vs_oracle(case, cuda_device):
    dkv, arrs, dev, cu, prec, qc, doc, qc_t, doc_t, inp = _setup(case)
    oc, lc, od, ld = dkv.dualkv_two_call_fwd(qc_t, inp)
    dq_c, dkc, dvc, dq, dkd, dvd = dkv.dualkv_two_call_bwd(qc_t, inp, oc, lc, doc_t, od, ld, dev["do"])
    torch.cuda.synchronize()
    p = qc.shape[0]
    # oracle composition of the two calls from the GPU's own saved O / lse (layer.py:273-279)
    g2 = orc.dualkv_bwd(arrs["q"], arrs["kc"], arrs["vc"], arrs["kd"], arrs["vd"], cu, to_np(od), to_np(ld),
                        arrs["do"], prec=prec, block_n=128)
    g1 = orc.varlen_bwd(qc, arrs["kc"], arrs["vc"], [0, p], to_np(oc), to_np(lc), doc, prec=prec, block_n=128)
    # total prompt grad: the exact (f64) sum of both calls' contributions
    f64 = dict(prec="f64", block_n=128)
    g1_64 = orc.varlen_bwd(qc, arrs["kc"], arrs["vc"], [0, p], to_np(oc), to_np(lc), doc, **f64)
    c2 = orc.context_contributions(arrs["q"], arrs["kc"], arrs["vc"], arrs["kd"], arrs["vd"], cu, to_np(od),
                                   to_np(ld), arrs["do"], **f64)
    dkc_ref = sum((c[0] for c in c2), np.zeros_like(arrs["kc"], dtype=np.float64)) + g1_64[1]
    dvc_ref = sum((c[1] for c in c2), np.zeros_like(arrs["vc"], dtype=np.float64)) + g1_64[2]
    check = (lambda got, ref, name: assert_close_abs(got, ref, F32_ATOL * max(1.0, np.abs(ref).max()), name)) \
        if prec == "f32" else assert_close_bf16
    check(to_np(dq), g2[0], "dQ_dec")
    check(to_np(dkd), g2[3], "dK_d")
    check(to_np(dvd), g2[4], "dV_d")
    check(to_np(dq_c), g1[0], "dQ_ctx")
    check(to_np(dkc), dkc_ref, "dK_c total")
    check(to_np(dvc), dvc_ref, "dV_c total")


def test_two_call_autograd_and_determinism(cuda_device):
    import paper_2605_15422_b200 as dkv
    case = CASES[0]
    _, arrs, dev, cu, prec, qc, doc, qc_t, doc_t, inp = _setup(case)
    leaves = [x.detach().clone().requires_grad_(True)
              for x in (qc_t, dev["kc"], dev["vc"], dev["q"], dev["kd"], dev["vd"])]
    oc, od = dkv.dualkv_two_call_attention(*leaves, cu)
    (oc.float() * doc_t.float()).sum().add((od.float() * dev["do"].float()).sum()).backward()
    o2 = dkv.dualkv_two_call_fwd(qc_t, inp)
    g = dkv.dualkv_two_call_bwd(qc_t, inp, o2[0], o2[1], doc_t, o2[2], o2[3], dev["do"])
    torch.cuda.synchronize()
    for leaf, ref, name in zip(leaves, (g[0], g[1], g[2], g[3], g[4], g[5]),
                               ("dQ_ctx", "dK_c", "dV_c", "dQ", "dK_d", "dV_d")):
        assert leaf.grad is not None, name
        assert_close_bf16(to_np(leaf.grad), to_np(ref), name)
    # deterministic mode: fixed-order fold of the prompt gradient -> bitwise reproducible
    a = dkv.dualkv_two_call_bwd(qc_t, inp, o2[0], o2[1], doc_t, o2[2], o2[3], dev["do"], deterministic=True)
    b = dkv.dualkv_two_call_bwd(qc_t, inp, o2[0], o2[1], doc_t, o2[2], o2[3], dev["do"], deterministic=True)
    torch.cuda.synchronize()
    assert torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])

"""SURVEY §8c oracle 2 at a full BASELINE config: the GPU op against the reference's CPU DualKV
(the NumPy restatement in oracle/, pinned to the reference's own goldens) on the identical bf16
inputs, over EVERY output element -- not a slice.

C2 (Qwen3-8B heads: H=32, H_k=8, d=128; N=16, P=4K, R=1K) through bench.py's exact call,
`dualkv_two_call_fwd` + `dualkv_two_call_bwd(deterministic=False)`.  The oracle runs the
reference algorithm (kernel.py:168-305 / fa2.py:112-306) with f32 compute on the bf16 inputs and
returns its results uncast (f32), on the host cores: ~1-2 minutes.  Bounds as in
test_gpu_twocall.py (|gpu - ref| <= 1e-2 + 1e-2 |ref| elementwise, lse <= 1e-3);
the prompt-key totals are Call 2's f32 fold over the 16 sequences plus Call 1's, summed in f64.
"""

import numpy as np
import pytest
import torch

from gpu_helpers import LSE_ATOL, assert_close_abs, assert_close_bf16, to_np
from oracle import dualkv_oracle as orc

pytestmark = pytest.mark.gpu


def test_c2_two_call_vs_cpu_reference_all_elements(cuda_device):
    import paper_2605_15422_b200 as dkv
    n, p, r, h, hk, d = 16, 4096, 1024, 32, 8, 128
    rng = np.random.default_rng(2024)
    t = n * r
    a = {k: orc.quantize(rng.normal(size=s), "bf16") for k, s in dict(
        q=(t, h, d), kc=(p, hk, d), vc=(p, hk, d), kd=(t, hk, d), vd=(t, hk, d), do=(t, h, d),
        qc=(p, h, d), doc=(p, h, d)).items()}
    g = {k: torch.from_numpy(np.ascontiguousarray(v)).to("cuda", torch.bfloat16) for k, v in a.items()}
    cu = np.arange(0, t + 1, r, dtype=np.int64)
    inp = dkv.DualKVInput(g["q"], g["kc"], g["vc"], g["kd"], g["vd"], cu)
    oc, lc, od, ld = dkv.dualkv_two_call_fwd(g["qc"], inp)
    dq_c, dkc, dvc, dq, dkd, dvd = dkv.dualkv_two_call_bwd(g["qc"], inp, oc, lc, g["doc"], od, ld, g["do"],
                                                           deterministic=False)
    torch.cuda.synchronize()

    # forward: Call 2 (two regions) and Call 1 (the prompt's causal self-attention)
    o2, l2 = orc.dualkv_fwd(a["q"], a["kc"], a["vc"], a["kd"], a["vd"], cu, prec="f32", block_n=128)
    o1, l1 = orc.varlen_fwd(a["qc"], a["kc"], a["vc"], [0, p], prec="f32", block_n=128)
    assert_close_bf16(to_np(od), o2, "O (Call 2)")
    assert_close_bf16(to_np(oc), o1, "O (Call 1)")
    assert_close_abs(to_np(ld), l2, LSE_ATOL, "lse (Call 2)")
    assert_close_abs(to_np(lc), l1, LSE_ATOL, "lse (Call 1)")

    # backward from the GPU's own saved O / lse (the reference caller's contract, layer.py:262-290)
    g2 = orc.dualkv_bwd(a["q"], a["kc"], a["vc"], a["kd"], a["vd"], cu, to_np(od), to_np(ld), a["do"],
                        prec="f32", block_n=128)
    g1 = orc.varlen_bwd(a["qc"], a["kc"], a["vc"], [0, p], to_np(oc), to_np(lc), a["doc"], prec="f32",
                        block_n=128)
    assert_close_bf16(to_np(dq), g2[0], "dQ (responses)")
    assert_close_bf16(to_np(dkd), g2[3], "dK_d")
    assert_close_bf16(to_np(dvd), g2[4], "dV_d")
    assert_close_bf16(to_np(dq_c), g1[0], "dQ (prompt)")
    # total prompt-key gradient: Call 2's (already folded over the 16 sequences) + Call 1's
    dkc_ref = g2[1].astype(np.float64) + g1[1].astype(np.float64)
    dvc_ref = g2[2].astype(np.float64) + g1[2].astype(np.float64)
    assert_close_bf16(to_np(dkc), dkc_ref, "dK_c total")
    assert_close_bf16(to_np(dvc), dvc_ref, "dV_c total")

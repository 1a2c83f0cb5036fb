"""Full-size GPU properties (no CPU oracle at these sizes):

* DualKV == replicated N-copy attention on the same problem (the paper's exactness
  argument; test_layer.py:178-196): decoded outputs/grads agree row for
  row, and the shared-prompt gradient equals the sum over the N prompt copies, at the
  BASELINE C2 shape and on a ragged (C4-like) group built through the device repack;
* deterministic mode is bitwise reproducible; exact power-of-two linearity in dO.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).abs().max() / b.abs().max().clamp_min(1e-30)).item()


def _replicated_grads(dkv, qc, kc, vc, q, kd, vd, doc, dod, cu, p):
    """Replicated layout [prompt ; response_i] per sequence with the prompt's own queries
    and upstream grads in every copy: the standard-packing computation of the same layer."""
    n = len(cu) - 1
    qs, ks, vs, ds, cu_r = [], [], [], [], [0]
    for i in range(n):
        a, b = int(cu[i]), int(cu[i + 1])
        qs += [qc, q[a:b]]
        ks += [kc, kd[a:b]]
        vs += [vc, vd[a:b]]
        # the prompt's upstream grad is shared: give it to copy 0 only (sum over copies = doc)
        ds += [doc if i == 0 else torch.zeros_like(doc), dod[a:b]]
        cu_r.append(cu_r[-1] + p + b - a)
    cat = lambda xs: torch.cat(xs).contiguous()
    b = dkv.VarlenBatch(cat(qs), cat(ks), cat(vs), np.asarray(cu_r))
    o, l = dkv.fa2_varlen_fwd(b)
    dq, dk, dv = dkv.fa2_varlen_bwd(b, o, l, cat(ds))
    return o, dq, dk, dv, cu_r


def _split(x, cu, cu_r, p):
    n = len(cu) - 1
    prompt = [x[cu_r[i]:cu_r[i] + p].float() for i in range(n)]
    dec = torch.cat([x[cu_r[i] + p:cu_r[i + 1]] for i in range(n)])
    return prompt, dec


def _check_equivalence(dkv, qc, kc, vc, q, kd, vd, doc, dod, cu, tol=2e-2):
    p = qc.shape[0]
    inp = dkv.DualKVInput(q, kc, vc, kd, vd, cu)
    oc, lc, od, ld = dkv.dualkv_two_call_fwd(qc, inp)
    dq_c, dkc, dvc, dq, dkd, dvd = dkv.dualkv_two_call_bwd(qc, inp, oc, lc, doc, od, ld, dod)
    o_r, dq_r, dk_r, dv_r, cu_r = _replicated_grads(dkv, qc, kc, vc, q, kd, vd, doc, dod, cu, p)
    torch.cuda.synchronize()
    o_pr, o_dec = _split(o_r, cu, cu_r, p)
    assert _rel(od, o_dec) < tol, "O_dec"
    assert _rel(oc, o_pr[0]) < tol, "O_ctx"
    for copy in o_pr[1:]:                       # prompt rows identical in every copy
        assert torch.equal(copy, o_pr[0])
    dq_pr, dq_dec = _split(dq_r, cu, cu_r, p)
    assert _rel(dq, dq_dec) < tol, "dQ_dec"
    assert _rel(dq_c, dq_pr[0]) < tol, "dQ_ctx"
    dk_pr, dk_dec = _split(dk_r, cu, cu_r, p)
    dv_pr, dv_dec = _split(dv_r, cu, cu_r, p)
    assert _rel(dkd, dk_dec) < tol, "dK_d"
    assert _rel(dvd, dv_dec) < tol, "dV_d"
    assert _rel(dkc, sum(dk_pr)) < tol, "dK_c = sum over prompt copies"
    assert _rel(dvc, sum(dv_pr)) < tol, "dV_c = sum over prompt copies"


def _rand(g, *shape):
    return torch.randn(*shape, device="cuda", generator=g).to(torch.bfloat16)


def test_c2_dualkv_equals_replicated(cuda_device):
    """BASELINE config C2: N=16, P=4096, R=1024, H=32/8, d=128, bf16."""
    import paper_2605_15422_b200 as dkv
    g = torch.Generator(device="cuda").manual_seed(7)
    n, p, r, h, hk, d = 16, 4096, 1024, 32, 8, 128
    t = n * r
    qc, kc, vc, doc = _rand(g, p, h, d), _rand(g, p, hk, d), _rand(g, p, hk, d), _rand(g, p, h, d)
    q, kd, vd, dod = _rand(g, t, h, d), _rand(g, t, hk, d), _rand(g, t, hk, d), _rand(g, t, h, d)
    _check_equivalence(dkv, qc, kc, vc, q, kd, vd, doc, dod, np.arange(0, t + 1, r))


@pytest.mark.parametrize("cfg", [(32, 8192, 2048, 32, 8), (32, 16384, 2048, 32, 4)], ids=["C3", "C5"])
def test_headline_shapes_dualkv_equals_replicated(cfg, cuda_device):
    """BASELINE configs C3 (the bench workload) and C5 (Qwen3-30B-A3B heads, G = 8, P = 16K) at
    full size: the fused two-call DualKV op against replicated N-copy attention on the same
    device (SURVEY §8c oracle 3), all outputs and six gradients."""
    import paper_2605_15422_b200 as dkv
    n, p, r, h, hk = cfg
    d = 128
    g = torch.Generator(device="cuda").manual_seed(11)
    t = n * r
    qc, kc, vc, doc = _rand(g, p, h, d), _rand(g, p, hk, d), _rand(g, p, hk, d), _rand(g, p, h, d)
    q, kd, vd, dod = _rand(g, t, h, d), _rand(g, t, hk, d), _rand(g, t, hk, d), _rand(g, t, h, d)
    _check_equivalence(dkv, qc, kc, vc, q, kd, vd, doc, dod, np.arange(0, t + 1, r))
    torch.cuda.empty_cache()


def test_ragged_group_through_device_repack(cuda_device):
    """C4-like ragged group (R_i ~ U[128, 1024]) packed N(P+R) -> P+NR on the device."""
    import paper_2605_15422_b200 as dkv
    from paper_2605_15422_b200.packing import make_plan, repack_to_dualkv
    rl = [int(x) for x in np.random.default_rng(0).integers(128, 1025, 12)]
    p, h, hk, d = 2048, 32, 8, 128
    plan = make_plan([(p, rl)])
    g = torch.Generator(device="cuda").manual_seed(3)
    # replicated activations whose prompt rows are identical in every copy (same prompt tokens)
    base_q, base_k, base_v = _rand(g, p, h, d), _rand(g, p, hk, d), _rand(g, p, hk, d)
    xq, xk, xv = [], [], []
    for r in rl:
        xq += [base_q, _rand(g, r, h, d)]
        xk += [base_k, _rand(g, r, hk, d)]
        xv += [base_v, _rand(g, r, hk, d)]
    qs, ks, vs = torch.cat(xq), torch.cat(xk), torch.cat(xv)
    q_dk, k_dk, v_dk = (repack_to_dualkv(x, plan) for x in (qs, ks, vs))
    assert torch.equal(q_dk[:p], base_q) and torch.equal(k_dk[:p], base_k)
    cu = plan.groups[0].resp_cu
    doc, dod = _rand(g, p, h, d), _rand(g, int(cu[-1]), h, d)
    _check_equivalence(dkv, q_dk[:p].contiguous(), k_dk[:p].contiguous(), v_dk[:p].contiguous(),
                       q_dk[p:].contiguous(), k_dk[p:].contiguous(), v_dk[p:].contiguous(), doc, dod, cu)


def test_deterministic_and_linearity(cuda_device):
    import paper_2605_15422_b200 as dkv
    g = torch.Generator(device="cuda").manual_seed(11)
    n, p, r, h, hk, d = 8, 1024, 512, 32, 8, 128
    t = n * r
    q, kc, vc, kd, vd, do = (_rand(g, t, h, d), _rand(g, p, hk, d), _rand(g, p, hk, d),
                             _rand(g, t, hk, d), _rand(g, t, hk, d), _rand(g, t, h, d))
    inp = dkv.DualKVInput(q, kc, vc, kd, vd, np.arange(0, t + 1, r))
    o, lse = dkv.dualkv_fwd(inp)
    a = dkv.dualkv_bwd(inp, o, lse, do, deterministic=True)
    b = dkv.dualkv_bwd(inp, o, lse, do, deterministic=True)
    c = dkv.dualkv_bwd(inp, o, lse, (do.float() * 2).to(torch.bfloat16), deterministic=True)
    torch.cuda.synchronize()
    assert torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])        # fixed-order fold
    assert torch.equal(a[3], b[3]) and torch.equal(a[4], b[4])        # own-response grads
    # exact doubling (power-of-two scaling commutes with every rounding); dQ's TMA reduce-add
    # order is not fixed, so it only agrees to bf16 resolution
    assert _rel(c[0], 2 * a[0].float()) < 1e-2
    for x, y in zip(a[1:], c[1:]):
        assert torch.equal(y.float(), 2 * x.float())

"""Past 2^31 elements (the replicated N-copy layout at C5 holds 2.4e9 query elements):
varlen causal attention (fa2.py:237-306, the kernels behind Call 1 and the N-copy baseline)
and the two-region DualKV op on tensors whose element offsets exceed int32, checked on the
LAST sequences -- the rows whose offsets overflow -- against a torch fp32 reference of the
same slice (SURVEY §8c tolerance, bf16 path)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

H, HK, D = 32, 8, 128


def _rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).abs().max() / b.abs().max().clamp_min(1e-30)).item()


def _ref_attention(q, k, v, do, causal_offset):
    """fp32 reference of one sequence: q [S_q, H, d], k/v [S_k, H_k, d]; query i sees keys
    j <= i + causal_offset (refattn.py:66-136 with GQA expansion)."""
    g = H // HK
    qf = q.float().transpose(0, 1).requires_grad_()                  # [H, S_q, d]
    kf = k.float().transpose(0, 1).repeat_interleave(g, 0).requires_grad_()
    vf = v.float().transpose(0, 1).repeat_interleave(g, 0).requires_grad_()
    s = (qf @ kf.transpose(1, 2)) / D ** 0.5
    sq, sk = q.shape[0], k.shape[0]
    mask = torch.arange(sk, device=q.device)[None, :] > (torch.arange(sq, device=q.device)[:, None] + causal_offset)
    s = s.masked_fill(mask, float("-inf"))
    o = torch.softmax(s, dim=-1) @ vf
    o.backward(do.float().transpose(0, 1))
    fold = lambda x: x.grad.view(HK, g, sk, D).sum(1).transpose(0, 1)
    return o.transpose(0, 1), qf.grad.transpose(0, 1), fold(kf), fold(vf)


def test_varlen_past_int32_offsets(cuda_device):
    import paper_2605_15422_b200 as dkv
    seq, nseq = 2048, 264  # 540,672 rows x 32 heads x 128 = 2.2e9 elements > 2^31
    t = seq * nseq
    assert t * H * D > 2 ** 31
    g = torch.Generator(device="cuda").manual_seed(7)
    mk = lambda *s: torch.randn(*s, device="cuda", generator=g, dtype=torch.bfloat16)
    q, k, v, do = mk(t, H, D), mk(t, HK, D), mk(t, HK, D), mk(t, H, D)
    cu = np.arange(0, t + 1, seq)
    b = dkv.VarlenBatch(q, k, v, cu)
    o, lse = dkv.fa2_varlen_fwd(b)
    dq, dk, dv = dkv.fa2_varlen_bwd(b, o, lse, do)
    torch.cuda.synchronize()
    for i in (nseq - 1, nseq // 2):
        a, e = int(cu[i]), int(cu[i + 1])
        ro, rdq, rdk, rdv = _ref_attention(q[a:e], k[a:e], v[a:e], do[a:e], 0)
        for got, ref, nm in ((o[a:e], ro, "O"), (dq[a:e], rdq, "dQ"), (dk[a:e], rdk, "dK"), (dv[a:e], rdv, "dV")):
            err = _rel(got, ref)
            assert err < 1e-2, f"seq {i} {nm}: max rel err {err:.3e}"


def test_dualkv_past_int32_offsets(cuda_device):
    import paper_2605_15422_b200 as dkv
    p, r, n = 1024, 2048, 264  # decoded region 540,672 rows: q / dO / dQ offsets exceed int32
    t = n * r
    g = torch.Generator(device="cuda").manual_seed(8)
    mk = lambda *s: torch.randn(*s, device="cuda", generator=g, dtype=torch.bfloat16)
    kc, vc = mk(p, HK, D), mk(p, HK, D)
    q, kd, vd, do = mk(t, H, D), mk(t, HK, D), mk(t, HK, D), mk(t, H, D)
    cu = np.arange(0, t + 1, r)
    inp = dkv.DualKVInput(q, kc, vc, kd, vd, cu)
    o, lse = dkv.dualkv_fwd(inp)
    dq, dkc, dvc, dkd, dvd = dkv.dualkv_bwd(inp, o, lse, do, deterministic=True)
    torch.cuda.synchronize()
    i = n - 1
    a, e = int(cu[i]), int(cu[i + 1])
    kk, vv = torch.cat([kc, kd[a:e]]), torch.cat([vc, vd[a:e]])
    ro, rdq, rdk, rdv = _ref_attention(q[a:e], kk, vv, do[a:e], p)
    for got, ref, nm in ((o[a:e], ro, "O"), (dq[a:e], rdq, "dQ"), (dkd[a:e], rdk[p:], "dK_d"), (dvd[a:e], rdv[p:], "dV_d")):
        err = _rel(got, ref)
        assert err < 1e-2, f"last sequence {nm}: max rel err {err:.3e}"

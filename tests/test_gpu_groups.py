"""Multi-group launches (SURVEY §8b group table): several prompt groups in ONE forward and ONE
backward launch must equal the per-group launches the reference's caller makes (layer.py:239);
and the registered torch.library ops compile with torch.compile(fullgraph=True)."""

import numpy as np
import pytest
import torch

from gpu_helpers import assert_close_bf16, to_np

pytestmark = pytest.mark.gpu

# (P_g, [R_g1, ...]) per group: ragged prompts (one empty), partial tiles, R_i = 0, varying N
GROUPS = [(300, [77, 0, 260]), (0, [50, 129]), (1024, [1, 200, 128, 33]), (129, [64]), (513, [3, 5, 700])]


def _rand(g, *shape):
    return torch.randn(*shape, device="cuda", generator=g).to(torch.bfloat16)


def _make(h=32, hk=8, d=128, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    data = []
    for p, rl in GROUPS:
        t = sum(rl)
        data.append(dict(qc=_rand(g, p, h, d), kc=_rand(g, p, hk, d), vc=_rand(g, p, hk, d), doc=_rand(g, p, h, d),
                         q=_rand(g, t, h, d), kd=_rand(g, t, hk, d), vd=_rand(g, t, hk, d), dod=_rand(g, t, h, d),
                         cu=np.concatenate([[0], np.cumsum(rl)]).astype(np.int64)))
    cat = lambda k: torch.cat([x[k] for x in data]).contiguous()
    lens = [r for _, rl in GROUPS for r in rl]
    allg = {k: cat(k) for k in ("qc", "kc", "vc", "doc", "q", "kd", "vd", "dod")}
    allg["cu"] = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    allg["gs"] = np.concatenate([[0], np.cumsum([len(rl) for _, rl in GROUPS])])
    allg["gc"] = np.concatenate([[0], np.cumsum([p for p, _ in GROUPS])])
    return data, allg


@pytest.mark.parametrize("d,hk", [(128, 8), (64, 2)])
def test_one_launch_equals_per_group_launches(d, hk, cuda_device):
    import paper_2605_15422_b200 as dkv
    data, a = _make(h=8 if d == 64 else 32, hk=hk, d=d)
    inp = dkv.DualKVInput(a["q"], a["kc"], a["vc"], a["kd"], a["vd"], a["cu"], group_seq_cu=a["gs"],
                          group_ctx_cu=a["gc"])
    assert inp.num_groups == len(GROUPS)
    oc, lc, od, ld = dkv.dualkv_two_call_fwd(a["qc"], inp)
    grads = dkv.dualkv_two_call_bwd(a["qc"], inp, oc, lc, a["doc"], od, ld, a["dod"], deterministic=False,
                                    return_context_f32=True)
    dq_c, dkc, dvc, dq, dkd, dvd, f32 = grads
    torch.cuda.synchronize()
    for gi, x in enumerate(data):
        c0, c1 = int(a["gc"][gi]), int(a["gc"][gi + 1])
        r0 = int(a["cu"][a["gs"][gi]])
        r1 = r0 + int(x["cu"][-1])
        one = dkv.DualKVInput(x["q"], x["kc"], x["vc"], x["kd"], x["vd"], x["cu"])
        ref_fwd = dkv.dualkv_two_call_fwd(x["qc"], one)
        ref = dkv.dualkv_two_call_bwd(x["qc"], one, *ref_fwd[:2], x["doc"], *ref_fwd[2:], x["dod"],
                                      deterministic=True, return_context_f32=True)
        torch.cuda.synchronize()
        # forward: same tiles in the same order -> bitwise
        assert torch.equal(oc[c0:c1], ref_fwd[0]) and torch.equal(lc[:, c0:c1], ref_fwd[1]), f"group {gi} Call 1"
        assert torch.equal(od[r0:r1], ref_fwd[2]) and torch.equal(ld[:, r0:r1], ref_fwd[3]), f"group {gi} Call 2"
        # own-response key gradients never merge across work items -> bitwise
        assert torch.equal(dkd[r0:r1], ref[4]) and torch.equal(dvd[r0:r1], ref[5]), f"group {gi} dK_d/dV_d"
        # dQ (fp32 reduce order) and the prompt gradient (fold order) agree to bf16 / fp32 resolution
        assert_close_bf16(to_np(dq[r0:r1]), to_np(ref[3]), f"group {gi} dQ")
        assert_close_bf16(to_np(dq_c[c0:c1]), to_np(ref[0]), f"group {gi} dQ_ctx")
        if c1 > c0:
            tot = f32[:, c0:c1].double()
            rel = ((tot - ref[6].double()).abs().max() / ref[6].double().abs().max()).item()
            assert rel < 1e-5, f"group {gi} fp32 prompt gradient: {rel:.2e}"
            assert_close_bf16(to_np(dkc[c0:c1]), to_np(ref[1]), f"group {gi} dK_c")
            assert_close_bf16(to_np(dvc[c0:c1]), to_np(ref[2]), f"group {gi} dV_c")


def test_group_table_validation(cuda_device):
    import paper_2605_15422_b200 as dkv
    _, a = _make()
    args = (a["q"], a["kc"], a["vc"], a["kd"], a["vd"], a["cu"])
    for gs, gc in (([0, 2, 2, 13], [0, 300, 300, a["gc"][-1]]),      # an empty group
                   ([0, 5, 13], [0, 400, 100]),                      # prompt rows do not add up
                   ([1, 13], [0, a["gc"][-1]])):                      # does not start at 0
        with pytest.raises(ValueError):
            dkv.DualKVInput(*args, group_seq_cu=gs, group_ctx_cu=gc)
    # fp32 (SIMT path) has no multi-group launch: a clear error, not a wrong answer
    inp = dkv.DualKVInput(*(x.float() for x in args[:5]), a["cu"], group_seq_cu=a["gs"], group_ctx_cu=a["gc"])
    with pytest.raises(ValueError, match="tensor-core"):
        dkv.dualkv_fwd(inp)


def test_layer_compiles_fullgraph_and_matches_eager(cuda_device):
    """torch.compile(fullgraph=True) over DualKVSelfAttention (Qwen3 q/k RMSNorm on): no graph
    break -- every device op is a registered op with a fake implementation -- and the compiled
    block's output and parameter gradients equal eager's."""
    from paper_2605_15422_b200 import packing
    from paper_2605_15422_b200.layer import DualKVBatch, DualKVSelfAttention
    torch.manual_seed(0)
    plan = packing.make_plan([(150, [40, 3, 200]), (70, [130, 64]), (0, [33])])
    blk = DualKVSelfAttention(256, 8, 2, 128, rope_base=1e6, qk_norm=True)
    batch = DualKVBatch.from_plan(plan, "cuda")
    x = (torch.randn(plan.total_dualkv, 256, device="cuda") * 0.5).to(torch.bfloat16)
    dy = torch.randn(plan.total_dualkv, 256, device="cuda").to(torch.bfloat16)

    def run(fn):
        blk.zero_grad()
        xx = x.clone().requires_grad_()
        y = fn(xx, batch)
        y.backward(dy)
        return y.detach(), xx.grad, {n: p.grad.clone() for n, p in blk.named_parameters()}

    y0, dx0, g0 = run(blk)
    torch._dynamo.reset()
    compiled = torch.compile(blk, fullgraph=True)
    y1, dx1, g1 = run(compiled)
    torch.cuda.synchronize()
    assert_close_bf16(to_np(y1), to_np(y0), "compiled output")
    assert_close_bf16(to_np(dx1), to_np(dx0), "compiled dX")
    for n in g0:
        err = (g1[n].float() - g0[n].float()).abs().max().item() / max(g0[n].float().abs().max().item(), 1e-30)
        assert err < 2e-2, f"compiled grad {n}: {err:.3e}"


def test_c4_groups_one_launch_equals_per_group_launches(cuda_device):
    """C4-sized groups (P = 8K, N = 16, R_i ~ U[512, 4096] with the bench's group seeds), four of
    them in one launch each way vs one launch per group."""
    import paper_2605_15422_b200 as dkv
    p, h, hk, d = 8192, 32, 8, 128
    rls = [[int(x) for x in np.random.default_rng(gi).integers(512, 4097, 16)] for gi in range(4)]
    g = torch.Generator(device="cuda").manual_seed(5)
    per = []
    for rl in rls:
        t = sum(rl)
        per.append(dict(qc=_rand(g, p, h, d), kc=_rand(g, p, hk, d), vc=_rand(g, p, hk, d), doc=_rand(g, p, h, d),
                        q=_rand(g, t, h, d), kd=_rand(g, t, hk, d), vd=_rand(g, t, hk, d), dod=_rand(g, t, h, d),
                        cu=np.concatenate([[0], np.cumsum(rl)]).astype(np.int64)))
    cat = lambda k: torch.cat([x[k] for x in per]).contiguous()
    lens = [r for rl in rls for r in rl]
    inp = dkv.DualKVInput(cat("q"), cat("kc"), cat("vc"), cat("kd"), cat("vd"), np.concatenate([[0], np.cumsum(lens)]),
                          group_seq_cu=np.arange(0, 65, 16), group_ctx_cu=np.arange(0, 4 * p + 1, p))
    qc_all, doc_all = cat("qc"), cat("doc")
    oc, lc, od, ld = dkv.dualkv_two_call_fwd(qc_all, inp)
    dq_c, dkc, dvc, dq, dkd, dvd = dkv.dualkv_two_call_bwd(qc_all, inp, oc, lc, doc_all, od, ld, cat("dod"),
                                                           deterministic=False)
    r0 = 0
    for gi, x in enumerate(per):
        t = int(x["cu"][-1])
        one = dkv.DualKVInput(x["q"], x["kc"], x["vc"], x["kd"], x["vd"], x["cu"])
        f = dkv.dualkv_two_call_fwd(x["qc"], one)
        b = dkv.dualkv_two_call_bwd(x["qc"], one, f[0], f[1], x["doc"], f[2], f[3], x["dod"], deterministic=False)
        torch.cuda.synchronize()
        c = slice(gi * p, (gi + 1) * p)
        assert torch.equal(oc[c], f[0]) and torch.equal(od[r0:r0 + t], f[2]), f"group {gi} forward"
        assert torch.equal(ld[:, r0:r0 + t], f[3]) and torch.equal(lc[:, c], f[1])
        assert torch.equal(dkd[r0:r0 + t], b[4]) and torch.equal(dvd[r0:r0 + t], b[5]), f"group {gi} dK_d/dV_d"
        for got, ref, name in ((dq[r0:r0 + t], b[3], "dQ"), (dq_c[c], b[0], "dQ_ctx"), (dkc[c], b[1], "dK_c"),
                               (dvc[c], b[2], "dV_c")):
            rel = ((got.float() - ref.float()).abs().max() / ref.float().abs().max()).item()
            assert rel < 1e-2, f"group {gi} {name}: {rel:.2e}"
        r0 += t

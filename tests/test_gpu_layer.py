"""Cross-backend gradient equivalence on the GPU (the reference's check at verify.py:411-420,
layer.py:236-290): one attention block (QKV projections, RoPE, attention, output projection)
trained through the DualKV layout -- `DualKVSelfAttention`, two-call op per group -- gives the
same parameter gradients as the same block on the replicated N(P+R) layout with ordinary causal
attention, for a loss on response tokens (the GRPO loss).  Input gradients agree after the
adjoint of the prompt broadcast (prompt rows summed over their N copies).  bf16 everywhere:
max |a - b| <= 2e-2 max |b| per tensor (SURVEY §8c bf16 bound, loosened for the two extra
bf16 GEMM layers the block adds)."""

import numpy as np
import pytest
import torch

from gpu_helpers import to_np

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = to_np(a), to_np(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def test_block_gradients_dualkv_equal_replicated(cuda_device):
    import paper_2605_15422_b200 as dkv
    from paper_2605_15422_b200 import packing
    from paper_2605_15422_b200.layer import DualKVSelfAttention
    torch.manual_seed(0)
    groups = [(150, [40, 0, 200, 9]), (70, [130, 64])]
    plan = packing.make_plan(groups)
    dm, h, hk, d = 256, 8, 2, 128
    blk = DualKVSelfAttention(dm, h, hk, d, rope_base=1e6)
    x = (torch.randn(plan.total_dualkv, dm, device="cuda") * 0.5).to(torch.bfloat16)
    # upstream gradient on response rows only (prompt rows carry no loss)
    resp = torch.zeros(plan.total_dualkv, 1, device="cuda")
    for g in plan.groups:
        resp[g.resp_start:g.resp_start + int(g.resp_cu[-1])] = 1
    dy = ((torch.randn(plan.total_dualkv, dm, device="cuda") * resp)).to(torch.bfloat16)

    # DualKV layout
    xd = x.clone().requires_grad_()
    blk.zero_grad()
    y = blk(xd, plan)
    y.backward(dy)
    g_dk = {n: p.grad.clone() for n, p in blk.named_parameters()}
    dx_dk = xd.grad.clone()

    # replicated layout, ordinary causal attention (DualKV op with an empty context = varlen causal)
    xs = packing.broadcast_to_standard(x, plan).clone().requires_grad_()
    dys = packing.broadcast_to_standard(dy, plan)
    for g in plan.groups:  # the loss lives on response rows: prompt copies carry none
        for i in range(len(g.resp_lens)):
            s = int(g.seq_cu[i])
            dys[s:s + g.prompt_len] = 0
    blk.zero_grad()
    t = xs.shape[0]
    pos = torch.as_tensor(packing.position_ids(plan, "standard"), device="cuda")
    q = dkv.RoPE.apply((xs @ blk.w_q).view(t, h, d), pos, blk.base)
    k = dkv.RoPE.apply((xs @ blk.w_k).view(t, hk, d), pos, blk.base)
    v = (xs @ blk.w_v).view(t, hk, d)
    empty = torch.zeros(0, hk, d, device="cuda", dtype=torch.bfloat16)
    o = dkv.dualkv_attention_varlen(q, empty, empty, k, v, plan.cu_seqlens_standard())
    ys = o.reshape(t, h * d) @ blk.w_o
    ys.backward(dys)
    for n, p in blk.named_parameters():
        assert _rel(g_dk[n], p.grad) <= 2e-2, f"{n}: rel err {_rel(g_dk[n], p.grad):.3e}"
    assert _rel(dx_dk, packing.reduce_to_dualkv(xs.grad, plan)) <= 2e-2
    # forward: the DualKV block output equals the replicated output seen through the repack
    assert _rel(y, packing.repack_to_dualkv(ys, plan)) <= 2e-2

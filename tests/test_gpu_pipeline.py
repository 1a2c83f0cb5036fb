"""End to end on the GPU: rollout records -> manifest -> repack + RoPE at logical positions ->
fused two-call DualKV attention, against replicated N-copy attention over the replicated layout
with RoPE at standard positions (the layout the reference's standard backend runs, layer.py:224-233).
DualKV rows must match the replicated rows they stand for (prompt rows: the first copy) within the
bf16 bound of SURVEY §8c."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from gpu_helpers import to_np

pytestmark = pytest.mark.gpu


def test_rollouts_to_attention(cuda_device):
    import paper_2605_15422_b200 as dkv
    from paper_2605_15422_b200 import packing, rollouts
    groups = rollouts.read_rollouts(os.path.join(GOLDEN, "rollouts.jsonl"))
    # scale the toy token lengths up so tiles are partial and multi-tile (lengths x 9)
    groups = [rollouts.RolloutGroup(g.prompt_id, g.prompt_tokens * 9,
                                    [rollouts.RolloutResponse(r.tokens * 9, r.advantage) for r in g.responses])
              for g in groups]
    rec_groups = rollouts.chunk_groups(groups, 8)
    h, hk, d, base = 8, 2, 128, 1e6
    g = torch.Generator(device="cuda").manual_seed(0)
    for chunk in rec_groups:
        plan = rollouts.pack_plan(chunk)
        # projections of the SAME tokens: every prompt copy in the replicated layout is identical
        mk = lambda hh: packing.broadcast_to_standard(
            (torch.randn(plan.total_dualkv, hh, d, device="cuda", generator=g) * 0.5).to(torch.bfloat16), plan)
        q_s, k_s, v_s = mk(h), mk(hk), mk(hk)
        # replicated reference: RoPE at standard positions, varlen causal attention over N(P+R)
        pos_std = packing.position_ids(plan, "standard")
        cu_std = plan.cu_seqlens_standard()
        qr, kr = dkv.rope_logical(q_s, pos_std, base), dkv.rope_logical(k_s, pos_std, base)
        o_r, _ = dkv.fa2_varlen_fwd(dkv.VarlenBatch(qr, kr, v_s, cu_std))
        # DualKV: fused repack + RoPE at logical positions, then per group the fused two-call op
        q_d, k_d, v_d = dkv.repack_rope_to_dualkv(q_s, k_s, v_s, plan, base)
        o_d = packing.repack_to_dualkv(o_r, plan)  # the replicated result seen through the repack
        for gl in plan.groups:
            c0, c1, r0 = gl.context_start, gl.context_start + gl.prompt_len, gl.resp_start
            r1 = r0 + int(gl.resp_cu[-1])
            inp = dkv.DualKVInput(q_d[r0:r1], k_d[c0:c1], v_d[c0:c1], k_d[r0:r1], v_d[r0:r1], gl.resp_cu)
            oc, lc, od, ld = dkv.dualkv_two_call_fwd(q_d[c0:c1], inp)
            for got, ref, name in ((od, o_d[r0:r1], "responses"), (oc, o_d[c0:c1], "prompt")):
                a, b = to_np(got), to_np(ref)
                bad = np.abs(a - b) > 1e-2 + 1e-2 * np.abs(b)
                assert not bad.any(), f"group {gl.prompt_len}/{gl.resp_lens} {name}: {bad.sum()} mismatches"

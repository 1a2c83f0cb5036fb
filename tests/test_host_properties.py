"""Property tests (hypothesis, as the reference's test_packing.py:100-128 / test_costmodel.py:183-191)
for the host-side logic either side of the kernels: repack plans, rollout manifests, pair counts."""

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import dualkv_oracle as orc

group_shapes = st.lists(
    st.tuples(st.integers(min_value=0, max_value=40),
              st.lists(st.integers(min_value=0, max_value=30), min_size=1, max_size=5)),
    min_size=1, max_size=4)


@given(group_shapes)
@settings(max_examples=80, deadline=None)
def test_plan_gather_broadcast_adjoint(groups):
    """Gather (replicated -> shared), broadcast (shared -> replicated) and the adjoint agree:
    broadcast(gather(x)) restores every response row and copy 0's prompt; the adjoint of the
    broadcast sums the N prompt copies; positions are logical (prompt j -> j, response r -> P + r)."""
    from paper_2605_15422_b200.packing import make_plan, position_ids
    plan = make_plan(groups)
    assert plan.total_standard == sum(sum(p + r for r in rs) for p, rs in groups)
    assert plan.total_dualkv == sum(p + sum(rs) for p, rs in groups)
    # token identity through the maps: tag each replicated row with (group, copy, in-seq pos)
    std_pos = position_ids(plan, "standard")
    dk_pos = position_ids(plan, "dualkv")
    assert np.array_equal(std_pos[plan.dk_from_std], dk_pos)
    assert np.array_equal(dk_pos[plan.std_from_dk], std_pos)
    # gather then broadcast is the identity on rows whose source is the gathered copy
    rt = plan.dk_from_std[plan.std_from_dk]
    for g in plan.groups:
        for i in range(len(g.resp_lens)):
            a, b = int(g.seq_cu[i]) + g.prompt_len, int(g.seq_cu[i + 1])
            assert np.array_equal(rt[a:b], np.arange(a, b))  # responses round-trip exactly
    # adjoint = transpose of the broadcast
    x = np.arange(plan.total_standard, dtype=np.float64) * 1.5 + 1.0
    adj = np.add.reduceat(x[plan.seg_src], plan.seg[:-1]) if plan.total_dualkv else np.zeros(0)
    ref = np.zeros(plan.total_dualkv)
    np.add.at(ref, plan.std_from_dk, x)
    nonempty = np.diff(plan.seg) > 0
    assert np.allclose(adj[nonempty], ref[nonempty])
    assert plan.dk_from_std.tolist() == orc.repack_index(groups).tolist()


@given(group_shapes)
@settings(max_examples=80, deadline=None)
def test_pair_counts_ordering(groups):
    """DualKV never visits more pairs than the replicated layout (costmodel.py:113-130), the
    cost model agrees with the oracle's restatement, and equality holds iff no prompt is shared."""
    from paper_2605_15422_b200.costmodel import visible_pairs
    for p, rs in groups:
        dk, std = visible_pairs(p, rs, "dualkv"), visible_pairs(p, rs, "standard")
        assert dk <= std
        assert dk == orc.visible_pairs(p, rs, "dualkv") and std == orc.visible_pairs(p, rs, "standard")
        if p > 0 and len(rs) > 1:
            assert dk < std


tokens = st.lists(st.integers(min_value=0, max_value=999), min_size=0, max_size=6)


@given(st.lists(st.tuples(tokens.filter(len), st.lists(st.tuples(tokens, st.floats(-2, 2, allow_nan=False)),
                                            min_size=1, max_size=4)), min_size=1, max_size=4),
       st.integers(min_value=4, max_value=8))
@settings(max_examples=60, deadline=None)
def test_manifest_round_trip(raw, mb):
    """Both manifest layouts restore every group's prompt, responses and advantages from the
    packed token ids (the reference's pack/unpack round trip, test_packing.py:100-128), and the
    dualkv manifest's positions are the repack plan's.  (Prompts are non-empty: a micro-batch
    without any token has no rho and raises, see below.)"""
    from paper_2605_15422_b200.packing import position_ids
    from paper_2605_15422_b200.rollouts import (RolloutGroup, RolloutResponse, manifest_positions,
                                                manifest_records, pack_plan)
    groups = [RolloutGroup(f"g{i}", list(p), [RolloutResponse(list(t), a) for t, a in rs])
              for i, (p, rs) in enumerate(raw)]
    for mode in ("dualkv", "standard"):
        recs = manifest_records(groups, mode, mb)
        back = []
        for rec in recs:
            ids = rec["token_ids"]
            for g in rec["groups"]:
                if mode == "dualkv":
                    c0, span, r0, cu = g["context_start"], g["context_span"], g["resp_start"], g["resp_cu"]
                    prompt = ids[c0:c0 + span]
                    resps = [ids[r0 + cu[i]:r0 + cu[i + 1]] for i in range(len(cu) - 1)]
                else:
                    cu, pl = g["seq_cu"], g["prompt_len"]
                    seqs = [ids[cu[i]:cu[i + 1]] for i in range(len(cu) - 1)]
                    prompt = seqs[0][:pl]
                    assert all(s[:pl] == prompt for s in seqs)
                    resps = [s[pl:] for s in seqs]
                back.append((g["prompt_id"], prompt, resps, g["advantages"]))
        # standard chunks may split a group across micro-batches: merge consecutive pieces
        merged = []
        for pid, prompt, resps, adv in back:
            if merged and merged[-1][0] == pid:
                merged[-1][2].extend(resps)
                merged[-1][3].extend(adv)
            else:
                merged.append((pid, prompt, list(resps), list(adv)))
        assert [m[0] for m in merged] == [g.prompt_id for g in groups]
        for (pid, prompt, resps, adv), g in zip(merged, groups):
            assert prompt == g.prompt_tokens
            assert resps == [r.tokens for r in g.responses]
            assert adv == [r.advantage for r in g.responses]
        if mode == "dualkv":
            for rec in recs:
                chunk = [g for g in groups if g.prompt_id in {e["prompt_id"] for e in rec["groups"]}]
                assert manifest_positions(rec).tolist() == position_ids(pack_plan(chunk), "dualkv").tolist()


def test_manifest_of_empty_batch_raises_like_the_reference():
    """A micro-batch without tokens has no rho: ZeroDivisionError, as packing.py:271-272."""
    import pytest
    from paper_2605_15422_b200.rollouts import RolloutGroup, RolloutResponse, manifest_records
    with pytest.raises(ZeroDivisionError):
        manifest_records([RolloutGroup("g", [], [RolloutResponse([], 0.0)])], "dualkv", 4)

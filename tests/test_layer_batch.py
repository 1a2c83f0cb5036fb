"""Host-side layout of the layer's single multi-group launch (`DualKVBatch.from_plan`), on CPU:
the split layout [all prompts ; all responses] is a permutation of the P+NR rows, the group table
matches the plan, and the offsets are the responses' (packing.py:182-220 layout)."""

import numpy as np
import pytest
import torch

from paper_2605_15422_b200 import packing
from paper_2605_15422_b200.layer import DualKVBatch


@pytest.mark.parametrize("groups", [[(7, [3, 5])], [(4, [2, 0, 6]), (0, [1]), (9, [4, 4, 1])]])
def test_batch_layout(groups):
    plan = packing.make_plan(groups)
    b = DualKVBatch.from_plan(plan, "cpu")
    assert DualKVBatch.from_plan(plan, "cpu") is b  # cached per device
    t = plan.total_dualkv
    order = torch.cat([b.ctx_rows, b.resp_rows])
    assert sorted(order.tolist()) == list(range(t))           # a permutation of the packed rows
    assert torch.equal(order[b.inv_perm], torch.arange(t))    # inv_perm undoes it
    assert b.group_ctx_cu == list(np.cumsum([0] + [p for p, _ in groups]))
    assert b.group_seq_cu == list(np.cumsum([0] + [len(r) for _, r in groups]))
    lens = [r for _, rs in groups for r in rs]
    assert b.cu_seqlens.dtype == torch.int32 and b.cu_seqlens.tolist() == list(np.cumsum([0] + lens))
    assert b.max_seqlen == max(lens)
    pos = packing.position_ids(plan, "dualkv")
    assert b.positions.tolist() == pos.tolist()
    # prompts first, in group order; each prompt row's logical position is its index in the prompt
    off = 0
    for g, (p, _) in zip(plan.groups, groups):
        rows = b.ctx_rows[off:off + p].tolist()
        assert rows == list(range(g.context_start, g.context_start + p))
        assert [pos[r] for r in rows] == list(range(p))
        off += p


def test_make_plan_rejects_a_group_without_responses():
    """a group with no responses has no copy to take its prompt from (the reference's
    RolloutGroup rejects it)."""
    with pytest.raises(ValueError, match="at least one response"):
        packing.make_plan([(4, []), (3, [2, 1])])

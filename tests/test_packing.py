"""Repack layouts: host index maps (CPU) and the device gather / adjoint (GPU)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import dualkv_oracle as orc


def _golden_groups():
    with open(os.path.join(GOLDEN, "packing_cost.json")) as f:
        return json.load(f)["packing"]


def test_plan_matches_reference_layouts():
    from paper_2605_15422_b200.packing import make_plan, position_ids
    pk = _golden_groups()
    groups = [(p, rs) for p, rs in pk["groups"]]
    plan = make_plan(groups)
    assert plan.cu_seqlens_standard().tolist() == pk["std_cu"]
    assert [[g.context_start, g.prompt_len, g.resp_start, g.resp_cu.tolist()] for g in plan.groups] \
        == pk["dk_layout"]
    std_tok = np.asarray(pk["std_tokens"])
    dk_tok = np.asarray(pk["dk_tokens"])
    assert std_tok[plan.dk_from_std].tolist() == pk["dk_tokens"]       # pack_dualkv
    assert dk_tok[plan.std_from_dk].tolist() == pk["std_tokens"]       # broadcast = pack_standard
    assert position_ids(plan, "dualkv").tolist() == pk["dk_pos"]
    assert position_ids(plan, "standard").tolist() == pk["std_pos"]
    assert plan.dk_from_std.tolist() == orc.repack_index(groups).tolist()


def test_adjoint_index_is_transpose_of_broadcast():
    from paper_2605_15422_b200.packing import make_plan
    plan = make_plan([(5, [3, 0, 2]), (0, [4]), (2, [1, 1, 1, 1])])
    m = np.zeros((plan.total_dualkv, plan.total_standard), dtype=np.int64)
    m[plan.std_from_dk, np.arange(plan.total_standard)] = 1
    adj = np.zeros_like(m)
    for r in range(plan.total_dualkv):
        adj[r, plan.seg_src[plan.seg[r]:plan.seg[r + 1]]] = 1
    assert np.array_equal(m, adj)


@pytest.mark.gpu
def test_device_repack_bitexact(cuda_device):
    import torch
    from paper_2605_15422_b200.packing import (broadcast_to_standard, make_plan, reduce_to_dualkv,
                                               repack_to_dualkv)
    rng = np.random.default_rng(0)
    groups = [(int(rng.integers(0, 300)), [int(x) for x in rng.integers(0, 200, size=int(rng.integers(1, 6)))])
              for _ in range(4)]
    plan = make_plan(groups)
    x_dk = torch.randn(plan.total_dualkv, 48, 128, device="cuda").to(torch.bfloat16)
    x_std = broadcast_to_standard(x_dk, plan)
    assert torch.equal(x_std.cpu(), x_dk.cpu()[torch.from_numpy(plan.std_from_dk)])
    assert torch.equal(repack_to_dualkv(x_std, plan), x_dk)
    g = torch.randn(plan.total_standard, 8, 64, device="cuda")
    red = reduce_to_dualkv(g, plan)
    ref = torch.zeros(plan.total_dualkv, 8, 64, dtype=torch.float64)
    ref.index_add_(0, torch.from_numpy(plan.std_from_dk), g.double().cpu())
    assert torch.allclose(red.double().cpu(), ref, atol=1e-5)

"""Rollout JSONL -> manifests -> repack plan against the reference's own `dualkv pack`
output (tests/golden/rollouts_manifests.json, tools/make_golden_rollouts.py)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2605_15422_b200 import packing, rollouts


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLDEN, "rollouts_manifests.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def groups():
    return rollouts.read_rollouts(os.path.join(GOLDEN, "rollouts.jsonl"))


def test_read_order_and_rho(gold, groups):
    assert [g.prompt_id for g in groups] == gold["group_order"]
    assert str(rollouts.token_reduction_ratio(groups)) == gold["rho_all"][0]


@pytest.mark.parametrize("key", ["dualkv_5", "dualkv_8", "standard_5", "standard_8"])
def test_manifests_match_reference(gold, groups, key):
    mode, mb = key.split("_")
    got = rollouts.manifest_records(groups, mode, int(mb))
    assert got == gold["manifests"][key]
    if mode == "dualkv":
        assert rollouts.validate_grouping(got).ok


def test_plan_positions_match_reference_layout(gold, groups):
    plan = rollouts.pack_plan(groups)
    np.testing.assert_array_equal(packing.position_ids(plan, "dualkv"), gold["dk_positions"])
    for rec in gold["manifests"]["dualkv_8"]:
        sub = [g for g in groups if g.prompt_id in {x["prompt_id"] for x in rec["groups"]}]
        sub.sort(key=lambda g: [x["prompt_id"] for x in rec["groups"]].index(g.prompt_id))
        p = rollouts.pack_plan(sub)
        assert p.total_dualkv == rec["total_tokens"]
        np.testing.assert_array_equal(packing.position_ids(p, "dualkv"), rollouts.manifest_positions(rec))


def test_errors(tmp_path, groups):
    bad = tmp_path / "bad.jsonl"
    bad.write_text(json.dumps(dict(prompt_id="x", prompt_tokens=[1, 2], response_tokens=[3], advantage=1.0)) + "\n"
                   + json.dumps(dict(prompt_id="x", prompt_tokens=[1, 9], response_tokens=[4], advantage=0.5)) + "\n")
    with pytest.raises(ValueError, match="'x'.*line 2"):
        rollouts.read_rollouts(str(bad))
    big = max(g.num_responses for g in groups)
    with pytest.raises(ValueError, match="cannot be co-located"):
        rollouts.manifest_records(groups, "dualkv", big - 1)
    with pytest.raises(ValueError):
        rollouts.RolloutGroup("e", [1], [])


def test_validate_grouping_detects_splits(groups):
    class S:
        def __init__(self, pid):
            self.prompt_id = pid
    assert not rollouts.validate_grouping([[S("a"), S("b")], [S("a")]]).ok
    assert not rollouts.validate_grouping([[S("a"), S("b"), S("a")]]).ok
    assert rollouts.validate_grouping([[S("a"), S("a"), S("b")], [S("c")]]).ok
    std = rollouts.manifest_records(groups, "standard", 2)
    assert rollouts.validate_grouping(std).ok  # replicated packing has no co-location contract

"""Rollout records -> micro-batch manifests -> the device repack plan.

The host-side data path in front of the DualKV kernels, with the reference's names and
contracts (cli.py:174-293 `read_rollouts` / `dualkv pack`, packing.py:159-322):

* `read_rollouts(path)`: JSONL records {prompt_id, prompt_tokens, response_tokens, advantage}
  -> prompt groups in first-appearance order; records of one prompt_id that disagree on
  prompt_tokens raise ValueError naming the prompt and line.
* `chunk_groups(groups, mb)`: DualKV micro-batches take whole groups (the co-location contract
  the shared-prompt kernel needs), at most `mb` responses each; a group larger than `mb`
  cannot be co-located and raises.  `chunk_samples(groups, mb)` is the replicated layout's
  free chunking.
* `manifest_records(...)`: one JSON-able record per micro-batch in the reference's manifest
  schema (token ids, per-group context/response offsets or sequence offsets, rho).
* `pack_plan(groups)`: the same micro-batch as a `packing.PackPlan` -- the index maps and
  logical positions the CUDA repack / RoPE (`repack_rope_to_dualkv`) and the attention ops use.
* `validate_grouping(batches)`: prompt_ids split across micro-batches (or non-contiguous
  within one) are violations.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Dict, Iterable, List, Sequence

import numpy as np

from .packing import PackPlan, make_plan

__all__ = ["RolloutResponse", "RolloutGroup", "read_rollouts", "chunk_groups", "chunk_samples",
           "manifest_records", "pack_plan", "token_reduction_ratio", "validate_grouping", "GroupingReport"]


@dataclass
class RolloutResponse:
    tokens: List[int]
    advantage: float


@dataclass
class RolloutGroup:
    """All responses sampled from one prompt (N >= 1)."""

    prompt_id: str
    prompt_tokens: List[int]
    responses: List[RolloutResponse]

    def __post_init__(self):
        if not self.responses:
            raise ValueError(f"group {self.prompt_id!r} has no responses")

    @property
    def num_responses(self) -> int:
        return len(self.responses)

    @property
    def prompt_len(self) -> int:
        return len(self.prompt_tokens)


def read_rollouts(path: str) -> List[RolloutGroup]:
    prompts: Dict[str, List[int]] = {}
    resps: Dict[str, List[RolloutResponse]] = {}
    with open(path, "r", encoding="utf-8") as fh:
        for line_no, line in enumerate(fh, 1):
            if not line.strip():
                continue
            rec = json.loads(line)
            pid = str(rec["prompt_id"])
            toks = [int(t) for t in rec["prompt_tokens"]]
            if pid in prompts and prompts[pid] != toks:
                raise ValueError(f"prompt {pid!r}: inconsistent prompt_tokens at line {line_no}")
            prompts.setdefault(pid, toks)
            resps.setdefault(pid, []).append(
                RolloutResponse([int(t) for t in rec["response_tokens"]], float(rec["advantage"])))
    return [RolloutGroup(pid, prompts[pid], resps[pid]) for pid in prompts]  # dicts keep first-seen order


def chunk_groups(groups: Sequence[RolloutGroup], mb: int) -> List[List[RolloutGroup]]:
    """Greedy in-order micro-batches of whole groups, <= mb responses each."""
    out: List[List[RolloutGroup]] = []
    cur: List[RolloutGroup] = []
    used = 0
    for g in groups:
        if g.num_responses > mb:
            raise ValueError(f"prompt {g.prompt_id!r} has {g.num_responses} responses, exceeding "
                             f"micro-batch capacity {mb}; its group cannot be co-located")
        if cur and used + g.num_responses > mb:
            out.append(cur)
            cur, used = [], 0
        cur.append(g)
        used += g.num_responses
    if cur:
        out.append(cur)
    return out


def chunk_samples(groups: Sequence[RolloutGroup], mb: int) -> List[List[RolloutGroup]]:
    """Replicated layout: fixed-size response chunks (no co-location contract); consecutive
    responses of one prompt inside a chunk are regrouped."""
    flat = [(g, r) for g in groups for r in g.responses]
    out = []
    for i in range(0, len(flat), mb):
        chunk: List[RolloutGroup] = []
        for g, r in flat[i:i + mb]:
            if chunk and chunk[-1].prompt_id == g.prompt_id:
                chunk[-1].responses.append(r)
            else:
                chunk.append(RolloutGroup(g.prompt_id, g.prompt_tokens, [r]))
        out.append(chunk)
    return out


def token_reduction_ratio(groups: Sequence[RolloutGroup]) -> Fraction:
    """T_standard / T_dualkv (packing.py token_reduction_ratio), exact."""
    t_std = sum(g.num_responses * g.prompt_len + sum(len(r.tokens) for r in g.responses) for g in groups)
    t_dk = sum(g.prompt_len + sum(len(r.tokens) for r in g.responses) for g in groups)
    if t_dk == 0:
        raise ZeroDivisionError("packed batch has no tokens")
    return Fraction(t_std, t_dk)


def _record(index: int, mode: str, chunk: Sequence[RolloutGroup]) -> dict:
    ids: List[int] = []
    groups = []
    for g in chunk:
        entry = dict(prompt_id=g.prompt_id, prompt_len=g.prompt_len, advantages=[r.advantage for r in g.responses])
        if mode == "dualkv":
            ctx0 = len(ids)
            ids += g.prompt_tokens
            rs0 = len(ids)
            cu = [0]
            for r in g.responses:
                ids += r.tokens
                cu.append(len(ids) - rs0)
            entry.update(context_start=ctx0, context_span=g.prompt_len, resp_start=rs0, resp_cu=cu)
        else:
            cu = [len(ids)]
            for r in g.responses:
                ids += g.prompt_tokens + r.tokens
                cu.append(len(ids))
            entry["seq_cu"] = cu
        groups.append(entry)
    return dict(index=index, mode=mode, total_tokens=len(ids), rho=float(token_reduction_ratio(chunk)),
                token_ids=ids, groups=groups)


def manifest_records(groups: Sequence[RolloutGroup], mode: str, mb: int) -> List[dict]:
    """The micro-batch manifests `dualkv pack --mode {mode} --mb {mb}` writes (cli.py:236-293)."""
    if mode not in ("dualkv", "standard"):
        raise ValueError(f"unknown mode {mode!r}")
    if mb < 1:
        raise ValueError("micro-batch capacity must be >= 1")
    chunks = chunk_groups(groups, mb) if mode == "dualkv" else chunk_samples(groups, mb)
    return [_record(i, mode, c) for i, c in enumerate(chunks)]


def pack_plan(groups: Sequence[RolloutGroup]) -> PackPlan:
    """The micro-batch's repack plan (both layouts' index maps, logical positions) for the
    device ops; group order and lengths as in the manifest."""
    return make_plan([(g.prompt_len, [len(r.tokens) for r in g.responses]) for g in groups])


@dataclass
class GroupingReport:
    ok: bool
    violations: List[str] = field(default_factory=list)


def validate_grouping(batches: Iterable) -> GroupingReport:
    """Co-location check (packing.py:282-322): each batch is a manifest record (dict, dualkv
    groups whole by construction; standard records pass) or an ordered list of objects with a
    `prompt_id`, whose same-prompt entries must be contiguous.  A prompt in two batches fails."""
    rep = GroupingReport(True)
    owner: Dict[str, int] = {}

    def claim(pid, b):
        if owner.get(pid, b) != b:
            rep.ok = False
            rep.violations.append(f"prompt {pid!r} split across batches {owner[pid]} and {b}")
        owner[pid] = b

    for b, batch in enumerate(batches):
        if isinstance(batch, dict):
            if batch.get("mode") == "standard":
                continue
            for g in batch["groups"]:
                claim(g["prompt_id"], b)
            continue
        runs: List[str] = []
        for s in batch:
            if not runs or runs[-1] != s.prompt_id:
                runs.append(s.prompt_id)
            claim(s.prompt_id, b)
        if len(runs) != len(set(runs)):
            dup = next(p for p in runs if runs.count(p) > 1)
            rep.ok = False
            rep.violations.append(f"prompt {dup!r} responses are not contiguous within batch {b}")
    return rep


def manifest_positions(record: dict) -> np.ndarray:
    """Logical positions of a dualkv manifest's token rows (PackedBatch.position_ids)."""
    pos = np.zeros(record["total_tokens"], dtype=np.int64)
    for g in record["groups"]:
        pos[g["context_start"]:g["context_start"] + g["context_span"]] = np.arange(g["context_span"])
        cu = g["resp_cu"]
        for i in range(len(cu) - 1):
            s, e = g["resp_start"] + cu[i], g["resp_start"] + cu[i + 1]
            pos[s:e] = g["prompt_len"] + np.arange(e - s)
    return pos

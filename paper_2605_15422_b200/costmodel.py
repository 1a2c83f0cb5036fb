"""Algorithmic work of the DualKV path (the roofline numerator).

Exact visible-pair counts as defined by the reference cost model
(costmodel.py:113-130): a prompt group with prompt length P and responses
R_i has P(P+1)/2 context pairs (Call 1) plus sum_i [R_i P + R_i(R_i+1)/2]
decoded pairs (Call 2).  Forward = 4 pairs*H*d FLOPs (QK^T, PV); backward =
10 pairs*H*d (S recompute, dP, dV, dK, dQ); masked/padded tile work and the
HBM-bound helper kernels are not counted.
"""

from __future__ import annotations

from typing import Sequence


def _tri(s: int) -> int:
    return s * (s + 1) // 2


def visible_pairs(p: int, r_list: Sequence[int], mode: str = "dualkv") -> int:
    if mode == "standard":
        return sum(_tri(p + int(r)) for r in r_list)
    if mode == "dualkv":
        return _tri(p) + sum(int(r) * p + _tri(int(r)) for r in r_list)
    if mode == "decoded":  # Call 2 alone
        return sum(int(r) * p + _tri(int(r)) for r in r_list)
    if mode == "context":  # Call 1 alone
        return _tri(p)
    raise ValueError(f"unknown mode {mode!r}")


def attention_flops(p: int, r_list: Sequence[int], heads: int, head_dim: int,
                    mode: str = "dualkv", passes: str = "fwd") -> int:
    mult = {"fwd": 4, "bwd": 10, "fwdbwd": 14}[passes]
    return mult * visible_pairs(p, r_list, mode) * heads * head_dim

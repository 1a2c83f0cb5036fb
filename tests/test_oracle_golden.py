"""Pin the CPU oracle to the reference's own outputs (tests/golden, made by
tools/make_golden.py from /root/reference).  CPU only."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_names, load_golden
from oracle import dualkv_oracle as orc

TOL = {"f64": 1e-12, "f32": 2e-5, "bf16": 2e-5}


def _close(got, ref, prec, what):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, what
    if got.size == 0:
        return
    if prec == "bf16" and what in ("dq", "dkc", "dvc", "dkd", "dvd", "dk", "dv"):
        # outputs on the bf16 grid: allow one bf16 ulp for f32 summation-order flips
        ulp = orc.bf16_ulp(ref)
        assert np.all(np.abs(got - ref) <= ulp * 1.0 + 1e-30), what
        return
    err = np.max(np.abs(got - ref) / (1.0 + np.abs(ref)))
    assert err <= TOL[prec], (what, err)


@pytest.mark.parametrize("name", golden_names("dualkv"))
def test_dualkv_matches_reference(name):
    meta, rec = load_golden(name)
    prec = meta["prec"]
    args = [rec[f"in_{k}"] for k in ("q", "k_context", "v_context", "k_decoded", "v_decoded")]
    cu = rec["in_cu"]
    o, lse = orc.dualkv_fwd(*args, cu, prec=prec, block_n=meta["tile"])
    _close(o, rec["o"], prec, "o")
    _close(lse, rec["lse"], prec, "lse")
    g = orc.dualkv_bwd(*args, cu, rec["o"], rec["lse"], rec["in_d_out"], prec=prec,
                       block_n=meta["tile"])
    for got, key in zip(g, ("dq", "dkc", "dvc", "dkd", "dvd")):
        _close(got, rec[key], prec, key)
    if "contrib_k" in rec:
        parts = orc.context_contributions(*args, cu, rec["o"], rec["lse"], rec["in_d_out"],
                                          prec=prec, block_n=meta["tile"])
        _close(np.stack([p[0] for p in parts]), rec["contrib_k"], prec, "contrib_k")
        _close(np.stack([p[1] for p in parts]), rec["contrib_v"], prec, "contrib_v")


@pytest.mark.parametrize("name", golden_names("varlen"))
def test_varlen_matches_reference(name):
    meta, rec = load_golden(name)
    prec = meta["prec"]
    o, lse = orc.varlen_fwd(rec["in_q"], rec["in_k"], rec["in_v"], rec["in_cu"], prec=prec,
                            block_n=meta["tile"])
    _close(o, rec["o"], prec, "o")
    _close(lse, rec["lse"], prec, "lse")
    g = orc.varlen_bwd(rec["in_q"], rec["in_k"], rec["in_v"], rec["in_cu"], rec["o"], rec["lse"],
                       rec["in_d_out"], prec=prec, block_n=meta["tile"])
    for got, key in zip(g, ("dq", "dk", "dv")):
        _close(got, rec[key], prec, key)


def test_dense_matches_reference():
    meta, rec = load_golden("dense_offset")
    o, lse = orc.dense_fwd(rec["in_q"], rec["in_k"], rec["in_v"], causal_offset=meta["offset"])
    assert np.max(np.abs(o - rec["o"])) < 1e-13
    assert np.max(np.abs(lse - rec["lse"])) < 1e-13
    g = orc.dense_bwd(rec["in_q"], rec["in_k"], rec["in_v"], rec["o"], rec["lse"],
                      rec["in_d_out"], causal_offset=meta["offset"])
    for got, key in zip(g, ("dq", "dk", "dv")):
        assert np.max(np.abs(got - rec[key])) < 1e-12, key


def test_bf16_round_bitexact():
    with np.load(os.path.join(GOLDEN, "bf16_round.npz")) as z:
        x, y = z["x"], z["y"]
    got = orc.bf16_round(x)
    assert np.array_equal(got.view(np.uint32)[~np.isnan(y)], y.view(np.uint32)[~np.isnan(y)])
    assert np.isnan(got[np.isnan(y)]).all()
    # known answers (test_tensor.py:23-47)
    assert orc.bf16_round(np.float32(1.0 / 3.0)) == 0.333984375
    assert orc.bf16_round(np.float32(1.00390625)) == 1.0


def test_packing_and_cost_match_reference():
    with open(os.path.join(GOLDEN, "packing_cost.json")) as f:
        ref = json.load(f)
    pk = ref["packing"]
    groups = [(p, rs) for p, rs in pk["groups"]]
    assert orc.standard_layout(groups).tolist() == pk["std_cu"]
    assert orc.position_ids(groups, "standard").tolist() == pk["std_pos"]
    assert orc.position_ids(groups, "dualkv").tolist() == pk["dk_pos"]
    lay = orc.dualkv_layout(groups)
    assert [[a, b, c, d.tolist()] for a, b, c, d in lay] == pk["dk_layout"]
    idx = orc.repack_index(groups)
    assert np.asarray(pk["std_tokens"])[idx].tolist() == pk["dk_tokens"]
    for c in ref["cost"]:
        rl = [c["r"]] * c["n"]
        assert orc.visible_pairs(c["p"], rl, "dualkv") == c["pairs_dk"]
        assert orc.visible_pairs(c["p"], rl, "standard") == c["pairs_std"]
        assert orc.attention_flops(c["p"], rl, c["h"], c["d"], "dualkv") == c["flops_dk"]
        assert orc.attention_flops(c["p"], rl, c["h"], c["d"], "standard") == c["flops_std"]


def test_dense_oracle_agrees_with_tiled_f64():
    """The two oracle forms agree (verify.py:112-133 restated)."""
    meta, rec = load_golden("partial_tiles")
    args = [rec[f"in_{k}"] for k in ("q", "k_context", "v_context", "k_decoded", "v_decoded")]
    cu = rec["in_cu"]
    o, lse = orc.dualkv_fwd(*args, cu, prec="f64", block_n=4)
    p = meta["p"]
    for i in range(len(cu) - 1):
        a, b = int(cu[i]), int(cu[i + 1])
        if a == b:
            continue
        od, ld = orc.dense_fwd(args[0][a:b], np.concatenate([args[1], args[3][a:b]]),
                               np.concatenate([args[2], args[4][a:b]]), causal_offset=p)
        assert np.max(np.abs(od - o[a:b])) < 1e-12
        assert np.max(np.abs(ld - lse[:, a:b])) < 1e-12


def test_stagnation_foil():
    """1 + 256 * 2^-9: naive bf16 fold stays 1.0, f32-then-cast gives 1.5 (verify.py:639-655)."""
    parts = [np.array([1.0], np.float32)] + [np.array([2.0 ** -9], np.float32)] * 256
    assert float(orc.naive_bf16_fold(parts)[0]) == 1.0
    acc = np.zeros(1, np.float32)
    for p in parts:
        acc += p
    assert float(orc.quantize(acc, "bf16")[0]) == 1.5


def test_rope_vs_reference_golden():
    """Oracle RoPE at DualKV logical positions == the reference's rope / rope_bwd
    (layer.py:182-205), pinned by tests/golden/rope.npz (tools/make_golden_rope.py)."""
    meta, rec = load_golden("rope")
    for i, c in enumerate(meta["cases"]):
        y = orc.rope(rec[f"x{i}"], rec["pos"], c["base"])
        b = orc.rope(rec[f"x{i}"], rec["pos"], c["base"], inverse=True)
        np.testing.assert_allclose(y, rec[f"y{i}"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(b, rec[f"b{i}"], rtol=0, atol=1e-12)
    yb = orc.rope(rec["x_big"], rec["pos_big"], meta["big_base"])
    np.testing.assert_allclose(yb, rec["y_big"], rtol=0, atol=1e-12)
    # the golden positions are the DualKV layout's (prompt j -> j, response r -> P + r)
    np.testing.assert_array_equal(rec["pos"], orc.position_ids([(9, [4, 0, 6]), (3, [5])]))

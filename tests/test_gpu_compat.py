"""`compat`: the reference's own objects in, the reference's own objects out.

The reference's check suites bind `dualkv_fwd`, `dualkv_bwd`, `fa2_varlen_fwd/bwd` and
`context_grad_contributions` by name (verify.py:17-26) and hand them its `Tensor`
(tensor.py:95-124: `.data` + `.precision` enum with values f64/f32/bf16), `DualKVInput`
(kernel.py:52-114) and `VarlenBatch` (fa2.py:57-91).  `/root/reference` is not on the GPU box,
so these are duck-typed stand-ins with the same attributes; the outputs must be instances of
the caller's class with the reference's saved precision (kernel.py:207-210), and match the
reference's stored outputs (tests/golden, made by tools/make_golden.py) at bf16 / fp32 bounds.
"""

import enum
from dataclasses import dataclass
from typing import Optional

import numpy as np
import pytest

from conftest import golden_names, load_golden
from gpu_helpers import F32_ATOL, LSE_ATOL, assert_close_abs, assert_close_bf16

pytestmark = pytest.mark.gpu


class Precision(enum.Enum):  # tensor.py:64-92 (values only)
    F64 = "f64"
    F32 = "f32"
    BF16EMU = "bf16"


class Tensor:  # tensor.py:95-124 (the attributes compat reads)
    def __init__(self, data, precision=Precision.F32):
        self.precision = precision
        self.data = np.asarray(data, dtype=np.float64 if precision is Precision.F64 else np.float32)

    @property
    def shape(self):
        return self.data.shape


@dataclass
class RefDualKVInput:  # kernel.py:52-114
    q: Tensor
    k_context: Tensor
    v_context: Tensor
    k_decoded: Tensor
    v_decoded: Tensor
    cu_seqlens_q: np.ndarray
    context_seqlen: Optional[int] = None
    max_seqlen_q: Optional[int] = None
    softmax_scale: Optional[float] = None
    causal: bool = True
    tile_size: int = 64


@dataclass
class RefVarlenBatch:  # fa2.py:57-91
    q: Tensor
    k: Tensor
    v: Tensor
    cu_seqlens: np.ndarray
    max_seqlen: Optional[int] = None
    softmax_scale: Optional[float] = None
    tile_size: int = 64


_PREC = {"bf16": Precision.BF16EMU, "f32": Precision.F32}


def _gpu_names(kind):
    return [n for n in golden_names(kind) if load_golden(n)[0]["prec"] in _PREC]


def _check(got, ref, prec, what):
    if prec == "bf16":
        assert_close_bf16(got, ref, what)
    else:
        assert_close_abs(got, ref, F32_ATOL * max(1.0, float(np.abs(ref).max(initial=0.0))), what)


@pytest.mark.parametrize("name", _gpu_names("dualkv"))
def test_compat_dualkv_against_reference_outputs(name, cuda_device):
    from paper_2605_15422_b200 import compat
    meta, rec = load_golden(name)
    pr = _PREC[meta["prec"]]
    t = lambda k: Tensor(rec[f"in_{k}"], pr)
    inp = RefDualKVInput(t("q"), t("k_context"), t("v_context"), t("k_decoded"), t("v_decoded"), rec["in_cu"],
                         softmax_scale=meta["scale"], tile_size=meta["tile"])
    o, lse = compat.dualkv_fwd(inp)
    assert isinstance(o, Tensor) and o.precision is Precision.F32  # saved in compute precision
    _check(o.data, rec["o"], meta["prec"], "O")
    assert_close_abs(lse.data, rec["lse"], LSE_ATOL, "lse")
    d_out = Tensor(rec["in_d_out"], pr)
    # the reference's saved O / lse fed back, as its callers do (layer.py:262-290)
    grads = compat.dualkv_bwd(inp, Tensor(rec["o"], Precision.F32), Tensor(rec["lse"], Precision.F32), d_out)
    for g, key, like in zip(grads, ("dq", "dkc", "dvc", "dkd", "dvd"),
                            (inp.q, inp.k_context, inp.v_context, inp.k_decoded, inp.v_decoded)):
        assert isinstance(g, Tensor) and g.precision is pr and g.shape == like.shape
        _check(g.data, rec[key], meta["prec"], key)
    if "contrib_k" in rec:
        parts = compat.context_grad_contributions(inp, Tensor(rec["o"], Precision.F32),
                                                  Tensor(rec["lse"], Precision.F32), d_out)
        assert len(parts) == rec["contrib_k"].shape[0]
        for (pk, pv), rk, rv in zip(parts, rec["contrib_k"], rec["contrib_v"]):
            _check(pk, rk, meta["prec"], "contrib_k")
            _check(pv, rv, meta["prec"], "contrib_v")


@pytest.mark.parametrize("name", _gpu_names("varlen"))
def test_compat_varlen_against_reference_outputs(name, cuda_device):
    from paper_2605_15422_b200 import compat
    meta, rec = load_golden(name)
    pr = _PREC[meta["prec"]]
    b = RefVarlenBatch(Tensor(rec["in_q"], pr), Tensor(rec["in_k"], pr), Tensor(rec["in_v"], pr), rec["in_cu"],
                       softmax_scale=meta["scale"], tile_size=meta["tile"])
    o, lse = compat.fa2_varlen_fwd(b)
    _check(o.data, rec["o"], meta["prec"], "O")
    assert_close_abs(lse.data, rec["lse"], LSE_ATOL, "lse")
    dq, dk, dv = compat.fa2_varlen_bwd(b, Tensor(rec["o"], Precision.F32), Tensor(rec["lse"], Precision.F32),
                                       Tensor(rec["in_d_out"], pr))
    for g, key in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
        _check(g.data, rec[key], meta["prec"], key)


def test_compat_rejects_f64(cuda_device):
    """F64 stays CPU-oracle-only: a clear ValueError, never a silent downcast."""
    from paper_2605_15422_b200 import compat
    meta, rec = load_golden(golden_names("dualkv")[0])
    t = lambda k: Tensor(rec[f"in_{k}"], Precision.F64)
    inp = RefDualKVInput(t("q"), t("k_context"), t("v_context"), t("k_decoded"), t("v_decoded"), rec["in_cu"])
    with pytest.raises(ValueError, match="F64|f64"):
        compat.dualkv_fwd(inp)

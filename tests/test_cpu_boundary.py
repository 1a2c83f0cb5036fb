"""CPU-side checks of the C-ABI boundary and the host logic (no GPU compute)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "dkv.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"DKV_API\s+[\w\s\*]+?\b(dkv_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2605_15422_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(lib, name), f"libdkv.so does not export {name}"
    assert set(declared) == set(_lib.SIGNATURES), "ctypes signatures out of sync with include/dkv.h"
    assert _lib.lib.dkv_abi_version() == _lib.DKV_ABI_VERSION == 2


def test_validation_errors_without_gpu():
    """Contract violations are reported before any device work (kernel.py:75-110)."""
    from paper_2605_15422_b200 import _lib
    p = _lib.FwdParams()
    p.num_seqs, p.total_q, p.ctx_len, p.heads, p.kv_heads, p.head_dim = 1, 0, 0, 6, 4, 64
    p.softmax_scale, p.dtype = 0.125, _lib.DKV_BF16
    p.cu_seqlens = 8  # non-null dummy; never dereferenced on the error path
    with pytest.raises(ValueError, match="multiple of H_k"):
        _lib.check(_lib.lib.dkv_dualkv_fwd(ctypes.byref(p), None))
    p.heads, p.ctx_len = 8, -1
    with pytest.raises(ValueError, match="non-negative"):
        _lib.check(_lib.lib.dkv_dualkv_fwd(ctypes.byref(p), None))
    p.ctx_len = 3
    with pytest.raises(ValueError, match="no context"):
        _lib.check(_lib.lib.dkv_varlen_fwd(ctypes.byref(p), None))


def test_tensor_core_dispatch_table():
    from paper_2605_15422_b200 import _lib
    f = _lib.lib.dkv_uses_tensor_cores
    assert f(_lib.DKV_BF16, 128, 32, 8) == 1      # Qwen3-8B shapes
    assert f(_lib.DKV_BF16, 128, 32, 4) == 1      # Qwen3-30B-A3B shapes
    assert f(_lib.DKV_BF16, 64, 8, 8) == 1
    assert f(_lib.DKV_F32, 64, 8, 8) == 0         # C1 fp32 -> SIMT fp32 kernels
    assert f(_lib.DKV_BF16, 8, 4, 2) == 0         # reference sweep head dims -> SIMT
    assert f(_lib.DKV_BF16, 128, 12, 4) == 1      # G = 3: tiles of 42 tokens x 3 heads (2 padding rows)
    assert f(_lib.DKV_BF16, 128, 40, 8) == 1      # Qwen3-14B / Qwen2.5-14B, G = 5
    assert f(_lib.DKV_BF16, 128, 130, 1) == 0     # G > 128 -> SIMT


def test_costmodel_matches_oracle():
    from oracle import dualkv_oracle as orc
    from paper_2605_15422_b200 import costmodel
    for p, rl in [(8192, [2048] * 32), (0, [5, 0, 9]), (7, [])]:
        for mode in ("dualkv", "standard"):
            assert costmodel.visible_pairs(p, rl, mode) == orc.visible_pairs(p, rl, mode)
    # headline numbers quoted in BASELINE.md (C3)
    assert costmodel.attention_flops(8192, [2048] * 32, 32, 128, passes="fwdbwd") == 36560875552768  # 3.656e13


def test_integration_stub_matches_the_abi():
    """The reference-side ctypes stub printed in INTEGRATION.md §2 lays out dkv_fwd_params exactly
    like the library's own binding (field names, order, sizes)."""
    import ctypes as C
    from paper_2605_15422_b200 import _lib
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = text.split("```python", 1)[1].split("```", 1)[0]
    src = "\n".join(ln for ln in block.splitlines()
                    if not ln.startswith(("_lib", "assert _lib", "import torch")) and "CDLL" not in ln)
    ns = {}
    exec(compile("import ctypes\n" + src.split("def dualkv_fwd_gpu")[0], "INTEGRATION.md", "exec"), ns)
    stub, ours = ns["_Fwd"], _lib.FwdParams
    assert C.sizeof(stub) == C.sizeof(ours)
    assert [f[0] for f in stub._fields_] == [f[0] for f in ours._fields_]
    for name, _ in ours._fields_:
        assert getattr(stub, name).offset == getattr(ours, name).offset, name

"""ctypes binding of libdkv.so (the C ABI declared in include/dkv.h).

The shared library is built in-tree (``make -C paper_2605_15422_b200/csrc``
or ``__graft_entry__.build()``).  There is no fallback: importing the
package without the library raises ImportError.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DKV_LIB: an alternative in-tree build (A/B timing of kernel variants); default libdkv.so
LIB_PATH = os.path.join(_HERE, os.environ.get("DKV_LIB", "libdkv.so"))

DKV_OK, DKV_ERR_INVALID, DKV_ERR_UNSUPPORTED, DKV_ERR_CUDA, DKV_ERR_WORKSPACE = 0, -1, -2, -3, -4
DKV_BF16, DKV_F32 = 0, 1

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p


DKV_ABI_VERSION = 2
DKV_MAX_GROUPS = 256


class GroupTable(ctypes.Structure):
    """dkv_group_table: HOST int32 arrays of num_groups + 1 (0 groups = one group)."""
    _fields_ = [("num_groups", _i64), ("seq_cu", _vp), ("ctx_cu", _vp)]


class FwdParams(ctypes.Structure):
    _fields_ = [
        ("q", _vp), ("k_ctx", _vp), ("v_ctx", _vp), ("k", _vp), ("v", _vp),
        ("cu_seqlens", _vp), ("out", _vp), ("lse", _vp),
        ("num_seqs", _i64), ("total_q", _i64), ("ctx_len", _i64), ("heads", _i64),
        ("kv_heads", _i64), ("head_dim", _i64), ("max_seqlen", _i64),
        ("softmax_scale", ctypes.c_float), ("dtype", ctypes.c_int32),
        ("groups", GroupTable),
    ]


class BwdParams(ctypes.Structure):
    _fields_ = [
        ("q", _vp), ("k_ctx", _vp), ("v_ctx", _vp), ("k", _vp), ("v", _vp),
        ("cu_seqlens", _vp), ("out", _vp), ("lse", _vp), ("dout", _vp),
        ("dq", _vp), ("dk_ctx", _vp), ("dv_ctx", _vp), ("dk", _vp), ("dv", _vp),
        ("num_seqs", _i64), ("total_q", _i64), ("ctx_len", _i64), ("heads", _i64),
        ("kv_heads", _i64), ("head_dim", _i64), ("max_seqlen", _i64),
        ("softmax_scale", ctypes.c_float), ("dtype", ctypes.c_int32),
        ("deterministic", ctypes.c_int32), ("ctx_chunk", ctypes.c_int32),
        ("ctx_partials", _vp), ("groups", GroupTable), ("ctx_grad_f32", _vp),
    ]


class TwoCallFwdParams(ctypes.Structure):
    _fields_ = [("call2", FwdParams), ("q_ctx", _vp), ("out_ctx", _vp), ("lse_ctx", _vp)]


class TwoCallBwdParams(ctypes.Structure):
    _fields_ = [("call2", BwdParams), ("q_ctx", _vp), ("out_ctx", _vp), ("lse_ctx", _vp),
                ("dout_ctx", _vp), ("dq_ctx", _vp)]


# every symbol include/dkv.h declares, with its ctypes signature
SIGNATURES = {
    "dkv_abi_version": (ctypes.c_int32, []),
    "dkv_last_error": (ctypes.c_char_p, []),
    "dkv_uses_tensor_cores": (ctypes.c_int32, [ctypes.c_int32, _i64, _i64, _i64]),
    "dkv_dualkv_fwd": (ctypes.c_int32, [ctypes.POINTER(FwdParams), _vp]),
    "dkv_varlen_fwd": (ctypes.c_int32, [ctypes.POINTER(FwdParams), _vp]),
    "dkv_bwd_workspace_size": (ctypes.c_size_t, [ctypes.POINTER(BwdParams)]),
    "dkv_bwd_num_ctx_chunks": (_i64, [ctypes.POINTER(BwdParams)]),
    "dkv_dualkv_bwd": (ctypes.c_int32, [ctypes.POINTER(BwdParams), _vp, ctypes.c_size_t, _vp]),
    "dkv_varlen_bwd": (ctypes.c_int32, [ctypes.POINTER(BwdParams), _vp, ctypes.c_size_t, _vp]),
    "dkv_twocall_fwd": (ctypes.c_int32, [ctypes.POINTER(TwoCallFwdParams), _vp]),
    "dkv_twocall_bwd_workspace_size": (ctypes.c_size_t, [ctypes.POINTER(TwoCallBwdParams)]),
    "dkv_twocall_bwd": (ctypes.c_int32, [ctypes.POINTER(TwoCallBwdParams), _vp, ctypes.c_size_t, _vp]),
    "dkv_convert_f32_to_bf16": (ctypes.c_int32, [_vp, _vp, _i64, _vp]),
    "dkv_gather_rows": (ctypes.c_int32, [_vp, _vp, _i64, _vp, _i64, _vp]),
    "dkv_segment_sum_rows": (ctypes.c_int32, [_vp, _vp, ctypes.c_int32, _i64, _vp, _vp, _i64, _vp]),
    "dkv_rope_rows": (ctypes.c_int32, [_vp, _vp, ctypes.c_int32, _i64, _i64, _i64, _vp, _vp, ctypes.c_double,
                                       ctypes.c_int32, _vp]),
    "dkv_rope_qkv_rows": (ctypes.c_int32, [_vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int32, _i64, _i64, _i64, _i64,
                                           _vp, _vp, ctypes.c_double, ctypes.c_int32, _vp]),
    "dkv_qkv_prep_fwd": (ctypes.c_int32, [_vp, _vp, _vp, ctypes.c_float, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64,
                                          _i64, ctypes.c_double, _vp]),
    "dkv_qkv_prep_bwd": (ctypes.c_int32, [_vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_float, _vp, _vp, _vp, _vp, _vp,
                                          _i64, _i64, _i64, _i64, ctypes.c_double, _vp]),
    "dkv_selftest_umma": (ctypes.c_int32, [ctypes.c_int32, _vp, _vp, _vp, _vp]),
    "dkv_profile_begin": (ctypes.c_int32, []),
    "dkv_profile_end": (ctypes.c_int32, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32),
                                         ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int32),
                                         ctypes.POINTER(ctypes.c_int32)]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libdkv.so not found at {LIB_PATH}: build it with "
            "`make -C paper_2605_15422_b200/csrc` (or __graft_entry__.build()); "
            "there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.dkv_abi_version() != DKV_ABI_VERSION:
        raise ImportError("libdkv.so ABI version mismatch")
    return lib


lib = _load()


def check(rc: int, what: str = "") -> None:
    """Map a C status to the reference's exception classes."""
    if rc == DKV_OK:
        return
    msg = (lib.dkv_last_error() or b"").decode(errors="replace")
    if rc in (DKV_ERR_INVALID, DKV_ERR_UNSUPPORTED):
        raise ValueError(msg or what)
    raise RuntimeError(f"{what}: {msg}" if what else msg)

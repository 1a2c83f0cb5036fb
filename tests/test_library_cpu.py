"""The torch.library registration of the DualKV ops, checked on CPU (meta tensors / FakeTensorMode):
every op exists, carries an autograd formula, and its fake implementation gives the shapes and
dtypes the CUDA implementation returns -- what torch.compile needs to trace through the op."""

import pytest
import torch
from torch._subclasses.fake_tensor import FakeTensorMode

import paper_2605_15422_b200  # noqa: F401  (registers the ops)

OPS = ["fwd", "bwd", "two_call_fwd", "two_call_bwd", "rope", "qkv_prep", "qkv_prep_bwd", "two_call_split",
       "two_call_split_bwd"]


def _m(*shape, dt=torch.bfloat16):
    return torch.empty(*shape, device="meta", dtype=dt)


def test_ops_registered_with_autograd():
    for name in OPS:
        op = getattr(torch.ops.dualkv, name)
        assert op.default._schema.name == f"dualkv::{name}"
    for name in ("fwd", "two_call_fwd", "rope", "qkv_prep", "two_call_split"):
        assert torch._C._dispatch_has_kernel_for_dispatch_key(f"dualkv::{name}", "Autograd")


@pytest.mark.parametrize("groups", [([], []), ([0, 1, 3], [0, 40, 64])])
def test_fake_shapes_two_call(groups):
    p, t, h, hk, d = 64, 100, 8, 2, 128
    gs, gc = groups
    out = torch.ops.dualkv.two_call_fwd(_m(p, h, d), _m(p, hk, d), _m(p, hk, d), _m(t, h, d), _m(t, hk, d),
                                        _m(t, hk, d), _m(4, dt=torch.int32), 60, 0.1, gs, gc)
    assert [tuple(o.shape) for o in out] == [(p, h, d), (h, p), (t, h, d), (h, t)]
    assert [o.dtype for o in out] == [torch.bfloat16, torch.float32, torch.bfloat16, torch.float32]
    g = torch.ops.dualkv.two_call_bwd(_m(p, h, d), _m(p, hk, d), _m(p, hk, d), _m(t, h, d), _m(t, hk, d),
                                      _m(t, hk, d), _m(4, dt=torch.int32), 60, 0.1, gs, gc, out[0], out[1],
                                      _m(p, h, d), out[2], out[3], _m(t, h, d), False)
    assert [tuple(x.shape) for x in g] == [(p, h, d), (p, hk, d), (p, hk, d), (t, h, d), (t, hk, d), (t, hk, d)]


def test_fake_shapes_five_tensor_and_rope_under_fake_mode():
    with FakeTensorMode():
        q = torch.empty(10, 4, 64, device="cuda", dtype=torch.bfloat16)
        kc = torch.empty(7, 2, 64, device="cuda", dtype=torch.bfloat16)
        kd = torch.empty(10, 2, 64, device="cuda", dtype=torch.bfloat16)
        cu = torch.empty(3, device="cuda", dtype=torch.int32)
        o, lse = torch.ops.dualkv.fwd(q, kc, kc, kd, kd, cu, 6, 0.125, [], [])
        assert o.shape == q.shape and lse.shape == (4, 10) and lse.dtype == torch.float32
        grads = torch.ops.dualkv.bwd(q, kc, kc, kd, kd, cu, 6, 0.125, [], [], o, lse, o, False)
        assert [x.shape for x in grads] == [q.shape, kc.shape, kc.shape, kd.shape, kd.shape]
        y = torch.ops.dualkv.rope(q, torch.empty(10, device="cuda", dtype=torch.int64), 1e4, False)
        assert y.shape == q.shape and y.device.type == "cuda"

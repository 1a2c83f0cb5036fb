"""Multi-process (gloo, world_size 2) checks of the data-parallel path on CPU.

Each rank owns whole prompt groups (LPT over exact pair counts), computes its
groups' gradient contribution to a shared parameter with the CPU oracle, and
GradSync all-reduces; the result must equal the single-process sum over all
groups -- the pipeline theorem (verify.py:522-533) at world size 2.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dualkv_oracle as orc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


GROUPS = [(7, [3, 5]), (4, [2, 2, 6]), (9, [1]), (3, [4, 4, 4, 1]), (6, [0, 5])]
H, HK, D = 4, 2, 8


def _group_grad(gi):
    """dL/dW for a toy projection k_ctx = x W feeding DualKV: sum_r dK_c^{(g)} ... per group."""
    p_len, rl = GROUPS[gi]
    rng = np.random.default_rng(100 + gi)
    t = sum(rl)
    q = rng.normal(size=(t, H, D))
    x = rng.normal(size=(p_len, D))
    w = np.random.default_rng(7).normal(size=(D, HK * D))
    kc = (x @ w).reshape(p_len, HK, D)
    vc = rng.normal(size=(p_len, HK, D))
    kd, vd = rng.normal(size=(t, HK, D)), rng.normal(size=(t, HK, D))
    do = rng.normal(size=(t, H, D))
    cu = np.concatenate([[0], np.cumsum(rl)]).astype(np.int64)
    o, lse = orc.dualkv_fwd(q, kc, vc, kd, vd, cu, prec="f64")
    _, dkc, _, _, _ = orc.dualkv_bwd(q, kc, vc, kd, vd, cu, o, lse, do, prec="f64")
    return x.T @ dkc.reshape(p_len, HK * D)  # dL/dW


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_15422_b200.dp import GradSync, group_cost, lpt_assign
    owned = lpt_assign([group_cost(p, rl) for p, rl in GROUPS], world)[rank]
    w = torch.nn.Parameter(torch.zeros(D, HK * D, dtype=torch.float64))
    w.grad = torch.zeros_like(w)
    for gi in owned:
        w.grad += torch.from_numpy(_group_grad(gi))
    GradSync([w], bucket_bytes=128).sync()
    out[rank] = (owned, w.grad.numpy().copy())
    dist.destroy_process_group()


def test_lpt_assignment_balances_and_covers():
    from paper_2605_15422_b200.dp import group_cost, lpt_assign
    costs = [group_cost(8192, list(np.random.default_rng(g).integers(512, 4097, 16))) for g in range(64)]
    for world in (1, 2, 4, 8):
        parts = lpt_assign(costs, world)
        assert sorted(i for p in parts for i in p) == list(range(64))
        loads = [sum(costs[i] for i in p) for p in parts]
        assert max(loads) / (sum(loads) / world) < 1.05


def test_gradient_allreduce_world2_matches_single_process():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    total = sum(_group_grad(g) for g in range(len(GROUPS)))
    owned = sorted(i for r in range(world) for i in out[r][0])
    assert owned == list(range(len(GROUPS)))
    for r in range(world):
        np.testing.assert_allclose(out[r][1], total, rtol=1e-12, atol=1e-12)


def _worker_overlap(rank, world, port, out):
    """bf16 parameters, hooks launching the all-reduce from inside backward (overlap=True):
    the synced gradient is the fp32 sum of the ranks' gradients cast to bf16 ONCE."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_15422_b200.dp import GradSync
    torch.manual_seed(0)
    w1 = torch.nn.Parameter(torch.randn(16, 8).to(torch.bfloat16))
    w2 = torch.nn.Parameter(torch.randn(8, 4).to(torch.bfloat16))
    sync = GradSync([w1, w2], bucket_bytes=16 * 8 * 4, overlap=True)  # two buckets
    g = torch.Generator().manual_seed(10 + rank)
    x = torch.randn(32, 16, generator=g).to(torch.bfloat16)
    with sync.no_sync():  # an earlier micro-batch: accumulate locally, no collective
        ((x @ w1) @ w2).float().pow(2).sum().backward()
    assert not sync._pending
    local = [w1.grad.float().clone(), w2.grad.float().clone()]
    w1.grad = None
    w2.grad = None
    ((x @ w1) @ w2).float().pow(2).sum().backward()   # hooks launch both buckets here
    launched = sorted(sync._pending)
    local2 = [w1.grad.float().clone(), w2.grad.float().clone()]
    sync.sync()
    out[rank] = (launched, [l.numpy() for l in local2], [w1.grad.float().numpy(), w2.grad.float().numpy()],
                 [w1.grad.dtype, w2.grad.dtype])
    dist.destroy_process_group()


def test_overlapped_bf16_gradient_sync_world2():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_overlap, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        launched, _, synced, dts = out[r]
        assert launched == [0, 1], "both buckets launched from the backward hooks"
        assert dts == [torch.bfloat16, torch.bfloat16]
        for i in range(2):
            exact = out[0][1][i].astype(np.float64) + out[1][1][i].astype(np.float64)
            want = torch.from_numpy(exact.astype(np.float32)).to(torch.bfloat16).float().numpy()
            np.testing.assert_array_equal(synced[i], want)  # fp32 sum, one cast

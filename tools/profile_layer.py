"""Kernel-time breakdown of the C4 attention-layer step (torch.profiler, CUDA activity), two
micro-batches of 8 DAPO groups: attention kernels vs projections (cuBLAS), q/k norm + RoPE, repack,
gradient sync.  python tools/profile_layer.py"""
import collections
import contextlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_15422_b200 import packing as pk  # noqa: E402
from paper_2605_15422_b200.dp import GradSync  # noqa: E402
from paper_2605_15422_b200.layer import DualKVBatch, DualKVSelfAttention  # noqa: E402

cfg = bench.CONFIGS["C4"]
p, h, hk, d, dm = cfg["p"], cfg["h"], cfg["hk"], cfg["d"], cfg["d_model"]
dev = torch.device("cuda", 0)
groups = [bench.group_r_list(cfg, gi) for gi in range(16)]
blk = DualKVSelfAttention(dm, h, hk, d, rope_base=1e6, qk_norm=True, device=dev)
sync = GradSync(list(blk.parameters()), overlap=True)
mbs = []
for i in range(0, len(groups), cfg["mb_groups"]):
    plan = pk.make_plan([(p, rl) for rl in groups[i:i + cfg["mb_groups"]]])
    mbs.append((plan, DualKVBatch.from_plan(plan, dev)))
g = torch.Generator(device=dev).manual_seed(77)
x_std = (torch.randn(max(m[0].total_standard for m in mbs), dm, device=dev, generator=g) * 0.5).to(torch.bfloat16)
dy = torch.randn(max(m[0].total_dualkv for m in mbs), dm, device=dev, generator=g).to(torch.bfloat16)


def step():
    for i, (plan, batch) in enumerate(mbs):
        x = pk.repack_to_dualkv(x_std[:plan.total_standard], plan)
        ctx = sync.no_sync() if i < len(mbs) - 1 else contextlib.nullcontext()
        with ctx:
            blk(x, batch).backward(dy[:plan.total_dualkv])
    sync.sync()
    blk.zero_grad(set_to_none=True)


for _ in range(2):
    step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
for e in ev:
    a = agg[e.name[:90]]
    a[0] += 1
    a[1] += e.time_range.elapsed_us() / 1000
tot = sum(v[1] for v in agg.values())
span = (max(e.time_range.end for e in ev) - min(e.time_range.start for e in ev)) / 1000
print(f"device busy {tot:.2f} ms, span {span:.2f} ms (two micro-batches of 8 groups)")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{ms:9.3f} ms {100 * ms / tot:5.1f}%  x{n:<4d} {k}")

"""Time repack_rope_to_dualkv for one group: python tools/time_repack.py [N P R H Hk]  (default C3)"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_15422_b200 as dkv  # noqa: E402
from paper_2605_15422_b200 import packing as pk  # noqa: E402
n, p, r, h, hk = (int(x) for x in sys.argv[1:6]) if len(sys.argv) > 5 else (32, 8192, 2048, 32, 8)
d = 128
plan = pk.make_plan([(p, [r] * n)])
xs = [torch.randn(plan.total_standard, hh, d, device="cuda").to(torch.bfloat16) for hh in (h, hk, hk)]
f = lambda: dkv.repack_rope_to_dualkv(*xs, plan, 1e6)
for _ in range(3):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    f()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
moved = 2 * plan.total_dualkv * (h + 2 * hk) * d * 2
print(os.environ.get("DKV_LIB", "libdkv.so"), sys.argv[1:6], f"repack_ms={ms:.4f} GB/s={moved / ms / 1e6:.0f}")

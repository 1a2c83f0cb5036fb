"""Device timeline of three C3 steps (torch.profiler, CUDA activity): kernels, memsets and the gaps
between them -- the step's aux work beside the two main kernels.  python tools/profile_timeline.py"""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2605_15422_b200 as dkv
n, p, r, h, hk, d = 32, 8192, 2048, 32, 8, 128
dt = torch.bfloat16
if os.environ.get("TL_C1"):  # BASELINE config C1: fp32, N=4 P=256 R=128, 8 heads, d=64
    n, p, r, h, hk, d, dt = 4, 256, 128, 8, 8, 64, torch.float32
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(dt)
t = n * r
qc, kc, vc, doc = mk(p, h, d), mk(p, hk, d), mk(p, hk, d), mk(p, h, d)
q, kd, vd, dod = mk(t, h, d), mk(t, hk, d), mk(t, hk, d), mk(t, h, d)
dec = dkv.DualKVInput(q, kc, vc, kd, vd, np.arange(0, t + 1, r))
def step():
    oc, lc, od, ld = dkv.dualkv_two_call_fwd(qc, dec)
    return dkv.dualkv_two_call_bwd(qc, dec, oc, lc, doc, od, ld, dod, deterministic=False)
for _ in range(3): step()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3): step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev_end = t0
for e in ev:
    gap = e.time_range.start - prev_end
    print(f"{(e.time_range.start - t0)/1000:9.3f} ms  dur {e.time_range.elapsed_us()/1000:8.3f} ms  gap {gap/1000:7.3f}  {e.name[:70]}")
    prev_end = max(prev_end, e.time_range.end)
print("total span", (prev_end - t0)/1000, "ms for 3 steps")

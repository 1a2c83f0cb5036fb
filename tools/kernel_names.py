"""Names of the CUDA kernels one small bf16 DualKV forward launches (torch.profiler): which forward
variant the library picked on this device.  python tools/kernel_names.py"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2605_15422_b200 as dkv
from torch.profiler import profile, ProfilerActivity
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
n, p, r, h, hk, d = 4, 512, 256, 32, 8, 128
q, kc, vc, kd, vd = mk(n*r, h, d), mk(p, hk, d), mk(p, hk, d), mk(n*r, hk, d), mk(n*r, hk, d)
inp = dkv.DualKVInput(q, kc, vc, kd, vd, np.arange(0, n*r+1, r))
dkv.dualkv_fwd(inp); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    dkv.dualkv_fwd(inp); torch.cuda.synchronize()
print(sorted({e.name[:60] for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA}))

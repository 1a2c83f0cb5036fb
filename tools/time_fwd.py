"""Time the C3 two-call forward (5 reps after 2 warm-up): python tools/time_fwd.py"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_15422_b200 as dkv  # noqa: E402
n, p, r, h, hk, d = 32, 8192, 2048, 32, 8, 128
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
t = n * r
qc, kc, vc = mk(p, h, d), mk(p, hk, d), mk(p, hk, d)
q, kd, vd = mk(t, h, d), mk(t, hk, d), mk(t, hk, d)
dec = dkv.DualKVInput(q, kc, vc, kd, vd, np.arange(0, t + 1, r))
for _ in range(2):
    dkv.dualkv_two_call_fwd(qc, dec)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    dkv.dualkv_two_call_fwd(qc, dec)
e1.record()
torch.cuda.synchronize()
print(os.environ.get("DKV_LIB", "libdkv.so"), f"fwd_ms={e0.elapsed_time(e1) / 5:.3f}")

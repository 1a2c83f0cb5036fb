"""Time the two-call backward at C2-like sizes with d = 64 (N=16 P=4K R=1K H=32 Hk=8)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_15422_b200 as dkv  # noqa: E402
n, p, r, h, hk, d = 16, 4096, 1024, 32, 8, int(os.environ.get("HD", "64"))
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
t = n * r
qc, kc, vc, doc = mk(p, h, d), mk(p, hk, d), mk(p, hk, d), mk(p, h, d)
q, kd, vd, dod = mk(t, h, d), mk(t, hk, d), mk(t, hk, d), mk(t, h, d)
inp = dkv.DualKVInput(q, kc, vc, kd, vd, np.arange(0, t + 1, r))
oc, lc, od, ld = dkv.dualkv_two_call_fwd(qc, inp)
run = lambda: dkv.dualkv_two_call_bwd(qc, inp, oc, lc, doc, od, ld, dod, deterministic=False)
for _ in range(2):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    run()
e1.record()
torch.cuda.synchronize()
from paper_2605_15422_b200.costmodel import visible_pairs
ms = e0.elapsed_time(e1) / 5
print(os.environ.get("DKV_LIB", "libdkv.so"), f"d={d} bwd_ms={ms:.3f} TFLOP/s={10 * visible_pairs(p, [r] * n, 'dualkv') * h * d / ms / 1e9:.1f}")

"""One C3 DualKV step (Call 1 + Call 2 fused, fwd + bwd -- what bench.py times) for ncu captures.

    ncu --set full --clock-control none --import-source on -k regex:dualkv_bwd -c 1 \
        -o gpurun_out/prof python tools/profile_step.py
    python tools/profile_step.py small      # N=8 P=2K R=512
    SEPARATE=1 python tools/profile_step.py # the reference's two separate calls
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_15422_b200 as dkv  # noqa: E402

n, p, r, h, hk, d = 32, 8192, 2048, 32, 8, 128
if len(sys.argv) > 1 and sys.argv[1] == "small":
    n, p, r = 8, 2048, 512
steps = int(os.environ.get("STEPS", "1"))
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
t = n * r
qc, kc, vc, doc = mk(p, h, d), mk(p, hk, d), mk(p, hk, d), mk(p, h, d)
q, kd, vd, dod = mk(t, h, d), mk(t, hk, d), mk(t, hk, d), mk(t, h, d)
ctx = dkv.VarlenBatch(qc, kc, vc, np.array([0, p]))
dec = dkv.DualKVInput(q, kc, vc, kd, vd, np.arange(0, t + 1, r))
for _ in range(steps):
    if os.environ.get("SEPARATE"):
        oc, lc = dkv.fa2_varlen_fwd(ctx)
        od, ld = dkv.dualkv_fwd(dec)
        dkv.dualkv_bwd(dec, od, ld, dod, deterministic=False)
        dkv.fa2_varlen_bwd(ctx, oc, lc, doc)
    else:
        oc, lc, od, ld = dkv.dualkv_two_call_fwd(qc, dec)
        # DET=1: the ordered fold (per-chunk partial stores) instead of the atomic merge -- the
        # difference in L2 reduction sectors isolates the dK_c / dV_c merge from the dQ reduce
        dkv.dualkv_two_call_bwd(qc, dec, oc, lc, doc, od, ld, dod, deterministic=os.environ.get("DET") == "1")
torch.cuda.synchronize()
print("done")

"""Small two-call DualKV fwd+bwd (ragged, partial tiles, R_i = 0, G = 4), a d = 64 DualKV fwd+bwd,
and the fused repack+RoPE gather, for compute-sanitizer."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_15422_b200 as dkv  # noqa: E402
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
p, rl, h, hk, d = 200, [77, 0, 150, 33], 8, 2, 128
t = sum(rl)
qc, kc, vc, doc = mk(p, h, d), mk(p, hk, d), mk(p, hk, d), mk(p, h, d)
q, kd, vd, dod = mk(t, h, d), mk(t, hk, d), mk(t, hk, d), mk(t, h, d)
dec = dkv.DualKVInput(q, kc, vc, kd, vd, np.concatenate([[0], np.cumsum(rl)]))
oc, lc, od, ld = dkv.dualkv_two_call_fwd(qc, dec)
for det in (True, False):
    gr = dkv.dualkv_two_call_bwd(qc, dec, oc, lc, doc, od, ld, dod, deterministic=det)
# d = 64 (tensor-core backward with the zero-padded K^T panel)
q64, kc64, vc64, kd64, vd64, do64 = mk(t, h, 64), mk(p, hk, 64), mk(p, hk, 64), mk(t, hk, 64), mk(t, hk, 64), mk(t, h, 64)
in64 = dkv.DualKVInput(q64, kc64, vc64, kd64, vd64, np.concatenate([[0], np.cumsum(rl)]))
o64, l64 = dkv.dualkv_fwd(in64)
g64 = dkv.dualkv_bwd(in64, o64, l64, do64, deterministic=True)
from paper_2605_15422_b200 import packing as pk  # noqa: E402
plan = pk.make_plan([(p, rl), (31, [5, 64])])
xs = [mk(plan.total_standard, hh, d) for hh in (h, hk, hk)]
rq, rk, rv = dkv.repack_rope_to_dualkv(*xs, plan, 1e6)
torch.cuda.synchronize()
print("ok", [float(x.float().abs().sum()) for x in gr], float(rq.float().abs().sum() + rk.float().abs().sum()),
      [float(x.float().abs().sum()) for x in g64])

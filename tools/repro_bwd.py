"""Small backward repro for compute-sanitizer runs: python tools/repro_bwd.py L1,L2,... H HK"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_15422_b200 as dkv  # noqa: E402

lens = [int(x) for x in sys.argv[1].split(",")]
h, hk, d = int(sys.argv[2]), int(sys.argv[3]), 128
t = sum(lens)
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
q, k, v, do = mk(t, h, d), mk(t, hk, d), mk(t, hk, d), mk(t, h, d)
b = dkv.VarlenBatch(q, k, v, np.concatenate([[0], np.cumsum(lens)]))
o, lse = dkv.fa2_varlen_fwd(b)
torch.cuda.synchronize()
print("fwd ok", flush=True)
dq, dk, dv = dkv.fa2_varlen_bwd(b, o, lse, do)
torch.cuda.synchronize()
print("bwd ok", float(dq.float().abs().sum()), flush=True)

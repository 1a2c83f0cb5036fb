"""Print GPU-vs-f64 errors of one parity case (debug aid): python tools/dbg_case.py"""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2605_15422_b200 as dkv
from oracle import dualkv_oracle as orc
from gpu_helpers import make_case, to_np
seed, n, p, rl, h, hk, d = 4, 1, 1, [1], 8, 1, 128
arrs, dev, cu, prec = make_case(seed, n, p, rl, h, hk, d, torch.bfloat16)
inp = dkv.DualKVInput(dev["q"], dev["kc"], dev["vc"], dev["kd"], dev["vd"], cu)
o, lse = dkv.dualkv_fwd(inp)
g = dkv.dualkv_bwd(inp, o, lse, dev["do"])
torch.cuda.synchronize()
o64, lse64 = orc.dualkv_fwd(arrs["q"], arrs["kc"], arrs["vc"], arrs["kd"], arrs["vd"], cu, prec="f64", block_n=128)
g64 = orc.dualkv_bwd(arrs["q"], arrs["kc"], arrs["vc"], arrs["kd"], arrs["vd"], cu, o64, lse64, arrs["do"], prec="f64", block_n=128)
print("lse", to_np(lse).ravel(), lse64.ravel())
print("O err", np.abs(to_np(o) - o64).max())
for nm, a, b in zip(("dQ", "dK_c", "dV_c", "dK_d", "dV_d"), g, g64):
    print(nm, np.abs(to_np(a) - b).max(), np.abs(b).max())

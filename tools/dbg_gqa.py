"""Error vs the f64 oracle of one odd-GQA case on the tensor-core path and on the SIMT path."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2605_15422_b200 as dkv  # noqa: E402
from gpu_helpers import make_case, to_np  # noqa: E402
from oracle import dualkv_oracle as orc  # noqa: E402
seed, n, p, rl, h, hk, d = 66, 4, 0, [50, 3, 0, 130], int(sys.argv[1]), int(sys.argv[2]), 128
arrs, dev, cu, prec = make_case(seed, n, p, rl, h, hk, d, torch.bfloat16)
inp = dkv.DualKVInput(dev["q"], dev["kc"], dev["vc"], dev["kd"], dev["vd"], cu)
o, lse = dkv.dualkv_fwd(inp)
g = dkv.dualkv_bwd(inp, o, lse, dev["do"])
torch.cuda.synchronize()
o64, l64 = orc.dualkv_fwd(arrs["q"], arrs["kc"], arrs["vc"], arrs["kd"], arrs["vd"], cu, prec="f64", block_n=128)
g64 = orc.dualkv_bwd(arrs["q"], arrs["kc"], arrs["vc"], arrs["kd"], arrs["vd"], cu, o64, l64, arrs["do"], prec="f64", block_n=128)
gb = orc.dualkv_bwd(arrs["q"], arrs["kc"], arrs["vc"], arrs["kd"], arrs["vd"], cu, to_np(o), to_np(lse), arrs["do"], prec="bf16", block_n=128)
print(os.environ.get("DKV_FORCE_SIMT", "tc"), "H", h, "Hk", hk)
for name, got, ref, rb in zip(("dQ", "dKc", "dVc", "dKd", "dVd"), g, g64, gb):
    got = to_np(got)
    if ref.size == 0:
        continue
    e = np.abs(got - ref)
    i = np.unravel_index(np.argmax(e), e.shape)
    ratio = e / (1e-2 + 1e-2 * np.abs(ref))
    j = np.unravel_index(np.argmax(ratio), ratio.shape)
    print(f"   {name}: worst err/bound {ratio.max():.3f} at {j} (gpu {got[j]:.4f} f64 {ref[j]:.4f}); "
          f"elements over 0.8 of the bound: {int((ratio > 0.8).sum())}; at (54,0,2): {e[54,0,2] if e.shape[0] > 54 else -1:.4f}")
    print(f"{name}: max|gpu-f64| {e.max():.4f} at {i} (gpu {got[i]:.4f} f64 {ref[i]:.4f} bf16-oracle {rb[i]:.4f}); "
          f"max|bf16oracle-f64| {np.abs(rb - ref).max():.4f}; max|ref| {np.abs(ref).max():.3f}")

"""Timeline of one forward CTA (libdkv_trace.so):  DKV_LIB=libdkv_trace.so python tools/trace_fwd.py [cta] [n]
Per KV-tile iteration: MMA issue of S_A/S_B (next) and PV_A/PV_B, softmax-A/B milestones."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_15422_b200 as dkv  # noqa: E402
from paper_2605_15422_b200._lib import lib  # noqa: E402

cta = int(sys.argv[1]) if len(sys.argv) > 1 else 0
show = int(sys.argv[2]) if len(sys.argv) > 2 else 10
n, p, r, h, hk, d = 32, 8192, 2048, 32, 8, 128
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
t = n * r
qc, kc, vc = mk(p, h, d), mk(p, hk, d), mk(p, hk, d)
q, kd, vd = mk(t, h, d), mk(t, hk, d), mk(t, hk, d)
dec = dkv.DualKVInput(q, kc, vc, kd, vd, np.arange(0, t + 1, r))
run = lambda: dkv.dualkv_two_call_fwd(qc, dec)
run()
torch.cuda.synchronize()
fn = lib.dkv_trace_read_fwd
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((20, 256), dtype=np.int64)  # kTraceEvents x kTraceTiles (trace.cuh)
fn(None, cta)
run()
torch.cuda.synchronize()
fn(buf.ctypes.data, -1)
t0 = buf[buf > 0].min()
rel = np.where(buf > 0, buf - t0, -1)
# event ids: 0 K load, 2 issue S_A, 3 issue S_B, 4 issue PV_A, 5 issue PV_B, 7 A sees S, 9 A loaded,
#            8 A stored P, 11 B sees S, 12 B loaded, 13 B stored P
cols = [(0, "Kld"), (2, "iSA"), (3, "iSB"), (4, "iPVA"), (5, "iPVB"), (7, "A:S"), (9, "A:ld"), (8, "A:P"),
        (11, "B:S"), (12, "B:ld"), (13, "B:P")]
print("it " + " ".join(f"{nm:>7}" for _, nm in cols))
for i in range(show):
    print(f"{i:2d} " + " ".join(f"{rel[e, i]:7d}" for e, _ in cols))
it = [i for i in range(2, 255) if rel[7, i] > 0 and rel[7, i + 1] > 0]
if it:
    med = lambda a, b: np.median([rel[b, i] - rel[a, i] for i in it if rel[a, i] > 0 and rel[b, i] > 0])
    print("median iteration period (A sees S):", np.median([rel[7, i + 1] - rel[7, i] for i in it]), "clk over", len(it))
    print("  A: S seen -> loaded", med(7, 9), " loaded -> P stored", med(9, 8))
    print("  A: loaded -> max done", med(9, 6), " max -> exps+STTM issued", med(6, 14), " -> P stored (wait_st)", med(14, 8))
    print("  B: S seen -> loaded", med(11, 12), " loaded -> P stored", med(12, 13))
    print("  A: P stored -> PV_A issued", med(8, 4), " PV_A issue -> next S_A seen",
          np.median([rel[7, i + 1] - rel[4, i] for i in it]))

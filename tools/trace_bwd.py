"""Timeline of one backward CTA (libdkv_trace.so, built with -DDKV_TRACE):
    DKV_LIB=libdkv_trace.so python tools/trace_bwd.py [cta] [ntiles]
Prints, per query tile, clock64 timestamps (relative to the CTA's first event) of the MMA issue
points, compute-warp and drain-warp milestones, and the per-tile period."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_15422_b200 as dkv  # noqa: E402
from paper_2605_15422_b200._lib import lib  # noqa: E402

EV = ["Qld", "Qarr", "iS", "idP", "idV", "idK", "idQ", "cS", "cP", "cdP", "cdS", "dDQ", "dLD", "dEND", "mEND", "x15", "kld", "sEND", "sDONE"]
cta = int(sys.argv[1]) if len(sys.argv) > 1 else 0
show = int(sys.argv[2]) if len(sys.argv) > 2 else 12
n, p, r, h, hk, d = 32, 8192, 2048, 32, 8, 128
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
t = n * r
qc, kc, vc, doc = mk(p, h, d), mk(p, hk, d), mk(p, hk, d), mk(p, h, d)
q, kd, vd, dod = mk(t, h, d), mk(t, hk, d), mk(t, hk, d), mk(t, h, d)
dec = dkv.DualKVInput(q, kc, vc, kd, vd, np.arange(0, t + 1, r))
oc, lc, od, ld = dkv.dualkv_two_call_fwd(qc, dec)
run = lambda: dkv.dualkv_two_call_bwd(qc, dec, oc, lc, doc, od, ld, dod, deterministic=False)
run()
torch.cuda.synchronize()
fn = getattr(lib, os.environ.get("TRACE_FN", "dkv_trace_read_v1"))
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((20, 256), dtype=np.int64)
fn(None, cta)
run()
torch.cuda.synchronize()
fn(buf.ctypes.data, -1)
t0 = buf[16, 0] if buf[16, 0] > 0 else buf[buf > 0].min()  # T_START when traced
rel = np.where(buf > 0, buf - t0, -1)
print("cta", cta, " columns: clk since the CTA's first event")
print("tile " + " ".join(f"{e:>7}" for e in EV) + "  period(iS)")
for i in range(min(show, 256)):
    if rel[2, i] < 0 and rel[7, i] < 0:
        break
    per = rel[2, i] - rel[2, i - 1] if i > 0 and rel[2, i - 1] >= 0 else 0
    print(f"{i:4d} " + " ".join(f"{rel[e, i]:7d}" for e in list(range(16)) + [17, 18, 19]) + f"  {per}")
valid = [i for i in range(1, 256) if rel[2, i] > 0 and rel[2, i - 1] > 0]
if valid:
    per = np.diff(rel[2, [0] + valid])
    print("median tile period", float(np.median(per)), "clk over", len(valid), "tiles")
    pairs_ = [("Q/dO load issue -> arrival", 0, 1), ("S issue -> compute sees S+dP", 2, 7), ("compute TMEM loads", 7, 9), ("compute math", 9, 8), ("compute waits pds_empty", 8, 14), ("compute stores+arrive", 14, 10),
              ("pds_full -> dV issue", 10, 4), ("dV issue -> dQ issue", 4, 6), ("dQ issue -> drain sees dQ", 6, 11),
              ("drain dQ -> loaded", 11, 12), ("drain loaded -> halves issued", 12, 13)]
    for nm, a, b in pairs_:
        if b == 3:
            dd = [rel[3, i + 1] - rel[6, i] for i in valid[:-1] if rel[3, i + 1] > 0]
        else:
            dd = [rel[b, i] - rel[a, i] for i in valid if rel[a, i] > 0 and rel[b, i] > 0]
        if dd:
            print(f"  {nm:32s} median {np.median(dd):7.0f}")

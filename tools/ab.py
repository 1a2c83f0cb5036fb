"""A/B timing of in-tree library builds (DKV_LIB=libdkv_<x>.so) on the C3 problem: the two-call
forward and backward, and the replicated N-copy forward and backward through the same kernels.
One process per (library, round); `tools/ab.sh` alternates A B A B on one box (power-capped clocks
drift, so comparisons are always interleaved).  Prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_15422_b200 as dkv  # noqa: E402

reps = int(os.environ.get("AB_REPS", "5"))
n, p, r, h, hk, d = 32, 8192, 2048, 32, 8, 128
if os.environ.get("AB_SHAPE"):  # "n,p,r,h,hk" (d = 128), e.g. C5's one group: 32,16384,2048,32,4
    n, p, r, h, hk = (int(x) for x in os.environ["AB_SHAPE"].split(","))
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
t = n * r
qc, kc, vc, doc = mk(p, h, d), mk(p, hk, d), mk(p, hk, d), mk(p, h, d)
q, kd, vd, dod = mk(t, h, d), mk(t, hk, d), mk(t, hk, d), mk(t, h, d)
dec = dkv.DualKVInput(q, kc, vc, kd, vd, np.arange(0, t + 1, r))


def timed(fn, k=reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


out = {}
saved = {}


def fwd():
    saved["f"] = dkv.dualkv_two_call_fwd(qc, dec)


out["fwd"] = timed(fwd)
oc, lc, od, ld = saved["f"]
out["bwd"] = timed(lambda: dkv.dualkv_two_call_bwd(qc, dec, oc, lc, doc, od, ld, dod, deterministic=False))
if os.environ.get("AB_REP", "1") == "1":
    del saved, oc, lc, od, ld
    s_cu = np.arange(0, n * (p + r) + 1, p + r)
    ts = int(s_cu[-1])
    qr, kr, vr, dor = mk(ts, h, d), mk(ts, hk, d), mk(ts, hk, d), mk(ts, h, d)
    rb = dkv.VarlenBatch(qr, kr, vr, s_cu)
    sv = {}

    def rf():
        sv["o"] = dkv.fa2_varlen_fwd(rb)

    out["rep_fwd"] = timed(rf, 3)
    o, l_ = sv["o"]
    out["rep_bwd"] = timed(lambda: dkv.fa2_varlen_bwd(rb, o, l_, dor), 3)
print(json.dumps({"lib": os.environ.get("DKV_LIB", "libdkv.so"), "label": os.environ.get("AB_LABEL"), **{k: round(v, 3) for k, v in out.items()}}))

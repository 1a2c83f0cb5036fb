"""Time the C3 two-call backward under DKV_BWD_ABLATE settings (timing only; results are
garbage when ablated).  Each setting runs in a fresh process: python tools/ablate_bwd.py"""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "run":
    import numpy as np
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2605_15422_b200 as dkv
    n, p, r, h, hk, d = 32, 8192, 2048, 32, 8, 128
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
    print(f"ablate={os.environ.get('DKV_BWD_ABLATE', '0')} bwd_ms={e0.elapsed_time(e1) / 5:.3f}", flush=True)
else:
    for a in (sys.argv[1:] or ["0", "1", "2", "4", "3", "7"]):
        subprocess.run([sys.executable, __file__, "run"], env={**os.environ, "DKV_BWD_ABLATE": a})

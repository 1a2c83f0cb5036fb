"""One full-size C3 run of the CPU path (the oracle port of the reference's algorithm, f32, all host
cores) -- the size-scaling calibration of bench.py's bounded cpu_baseline sample (the
DualKV CPU path at C3 "always runs fully").  Writes profiles/r2_cpu_full_c3.json.

Usage (on the GPU box host, whose cores bench.py's CPU arm uses):
    python tools/cpu_full_c3.py [--out profiles/r2_cpu_full_c3.json]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import dualkv_oracle as orc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_cpu_full_c3.json"))
    args = ap.parse_args()
    c = dict(n=32, p=8192, r=2048, h=32, hk=8, d=128)
    rng = np.random.default_rng(0)
    t = c["n"] * c["r"]
    f = lambda *s: rng.normal(size=s).astype(np.float32)
    qc, kc, vc, doc = f(c["p"], c["h"], c["d"]), f(c["p"], c["hk"], c["d"]), f(c["p"], c["hk"], c["d"]), \
        f(c["p"], c["h"], c["d"])
    q, kd, vd, dod = f(t, c["h"], c["d"]), f(t, c["hk"], c["d"]), f(t, c["hk"], c["d"]), f(t, c["h"], c["d"])
    cu = np.arange(0, t + 1, c["r"], dtype=np.int64)
    cuc = np.array([0, c["p"]], dtype=np.int64)
    times = {}
    t0 = time.perf_counter()
    oc, lc = orc.varlen_fwd(qc, kc, vc, cuc, prec="f32", block_n=128)
    od, ld = orc.dualkv_fwd(q, kc, vc, kd, vd, cu, prec="f32", block_n=128)
    times["fwd_s"] = time.perf_counter() - t0
    t1 = time.perf_counter()
    orc.dualkv_bwd(q, kc, vc, kd, vd, cu, od, ld, dod, prec="f32", block_n=128)
    orc.varlen_bwd(qc, kc, vc, cuc, oc, lc, doc, prec="f32", block_n=128)
    times["bwd_s"] = time.perf_counter() - t1
    total = times["fwd_s"] + times["bwd_s"]
    fl = bench.flops_fwdbwd(c)
    s_tf, s_sec = bench.cpu_sample_tflops(reps=1, warmup=0)
    rec = {"what": "full C3 (N=32 P=8192 R=2048 H=32 Hk=8 d=128) Call1+Call2 fwd+bwd through the CPU oracle port, "
                   "f32, one run", "seconds": round(total, 1), "fwd_s": round(times["fwd_s"], 1),
           "bwd_s": round(times["bwd_s"], 1), "tflops": round(fl / total / 1e12, 6),
           "cores": bench.cpu_threads(), "host": bench.cpu_host(),
           "bench_sample": {"sample": bench.sample_desc(), "tflops": round(s_tf, 6), "seconds": round(s_sec, 2)},
           "full_over_sample_rate": round(fl / total / 1e12 / s_tf, 3)}
    with open(args.out, "w") as fh:
        json.dump(rec, fh, indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()

"""DualKV attention fwd+bwd benchmark (BASELINE.json metric) on B200.

Workload (BASELINE.json configs[2], "C3"): Qwen3-8B attention shapes, one
prompt group of N=32 responses, P=8192 prompt tokens, R=2048 response
tokens each, H=32 query / H_k=8 KV heads, d=128, bf16.  One step = Call 1
(causal self-attention over the single prompt copy) + Call 2 (fused
two-region DualKV) forward AND backward -- the reference's `run_bench` "dk"
unit (src/bench.py:146-152).  value = algorithmic TFLOP/s
(14 * visible_pairs * H * d per step), whole job over all ranks.

Also measured in the same run:
  * replicated N-copy causal attention (same kernels, N(P+R) layout) and
    the speedup vs it;
  * e2e: the same step through the public API with pinned HOST buffers,
    H2D of every input and D2H of every output inside the timed region;
  * roofline of the dominant kernel, timed with CUDA events recorded by
    libdkv on the launching stream;
  * cpu_baseline: the CPU oracle port (numpy, the reference's algorithm)
    on a bounded sample, timed on this host's cores (rank 0, N=1 only).

`--impl reference` times the reference's CPU algorithm (oracle port --
the reference is pure Python and cannot travel to the GPU box) on a
bounded sample of the same workload and prints the same JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DualKV attn fwd+bwd ms & TFLOP/s at Qwen3-8B shapes N=32,P=8K; speedup vs N-copy"
C3 = dict(n=32, p=8192, r=2048, h=32, hk=8, d=128)
CPU_SAMPLE = dict(n=4, p=2048, r=512, h=32, hk=8, d=128)  # same head config, fewer tokens


def pairs(p, r_list):
    tri = lambda s: s * (s + 1) // 2
    return tri(p) + sum(r * p + tri(r) for r in r_list)


def flops_fwdbwd(cfg):
    return 14 * pairs(cfg["p"], [cfg["r"]] * cfg["n"]) * cfg["h"] * cfg["d"]


def rep_flops_fwdbwd(cfg):
    tri = lambda s: s * (s + 1) // 2
    return 14 * cfg["n"] * tri(cfg["p"] + cfg["r"]) * cfg["h"] * cfg["d"]


# ---------------------------------------------------------------- CPU side
def cpu_sample_tflops(reps=1, warmup=0):
    """The reference algorithm (oracle port, f32 as the reference bench default,
    src/bench.py:43) timed fwd+bwd on CPU_SAMPLE; returns (TFLOP/s, seconds/step)."""
    from oracle import dualkv_oracle as orc
    c = CPU_SAMPLE
    rng = np.random.default_rng(0)
    t = c["n"] * c["r"]
    qc = rng.normal(size=(c["p"], c["h"], c["d"])).astype(np.float32)
    kc = rng.normal(size=(c["p"], c["hk"], c["d"])).astype(np.float32)
    vc = rng.normal(size=(c["p"], c["hk"], c["d"])).astype(np.float32)
    q = rng.normal(size=(t, c["h"], c["d"])).astype(np.float32)
    kd = rng.normal(size=(t, c["hk"], c["d"])).astype(np.float32)
    vd = rng.normal(size=(t, c["hk"], c["d"])).astype(np.float32)
    doc = rng.normal(size=qc.shape).astype(np.float32)
    dod = rng.normal(size=q.shape).astype(np.float32)
    cu = np.arange(0, t + 1, c["r"], dtype=np.int64)
    cuc = np.array([0, c["p"]], dtype=np.int64)

    def step():
        oc, lc = orc.varlen_fwd(qc, kc, vc, cuc, prec="f32", block_n=128)
        od, ld = orc.dualkv_fwd(q, kc, vc, kd, vd, cu, prec="f32", block_n=128)
        orc.dualkv_bwd(q, kc, vc, kd, vd, cu, od, ld, dod, prec="f32", block_n=128)
        orc.varlen_bwd(qc, kc, vc, cuc, oc, lc, doc, prec="f32", block_n=128)

    for _ in range(warmup):
        step()
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    sec = float(np.median(times))
    return flops_fwdbwd(c) / sec / 1e12, sec


def cpu_threads():
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS"):
        if os.environ.get(var):
            return int(os.environ[var])
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def sample_desc():
    c = CPU_SAMPLE
    return (f"oracle port (numpy/OpenBLAS f32, the reference tile algorithm) fwd+bwd of Call1+Call2 at "
            f"N={c['n']} P={c['p']} R={c['r']} H={c['h']} Hk={c['hk']} d={c['d']} "
            f"({flops_fwdbwd(c) / 1e9:.1f} GFLOP/step)")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    tflops, sec = cpu_sample_tflops(reps=max(1, args.steps), warmup=args.warmup)
    line = {
        "metric": METRIC, "impl": "reference", "value": round(tflops, 6), "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "C3 head shapes (H=32, Hk=8, d=128), bounded token sample", **CPU_SAMPLE},
        "cpu_baseline": {"value": round(tflops, 6), "unit": "TFLOP/s", "cores": cpu_threads(),
                         "kind": "port", "sample": sample_desc()},
        "e2e": {"value": round(tflops, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU side
class ClockSampler:
    def __init__(self, out_path=None):
        self.samples = []
        self.proc = None
        self.out_path = out_path

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        dev = os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or "0"
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(int(os.environ.get("LOCAL_RANK", "0"))) if dev.isdigit() else dev,
                 f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for i, n in enumerate(names):
                if len(s) > 4 + i and s[4 + i].lower().startswith("active"):
                    reasons.add(n)
        busy = [x for x in sm if x > 0]
        return {"sm_mhz": float(np.median(busy)) if busy else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-replicated", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2605_15422_b200 as dkv
    from paper_2605_15422_b200._lib import lib
    import ctypes

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    c = C3
    n, p, r, h, hk, d = c["n"], c["p"], c["r"], c["h"], c["hk"], c["d"]
    t = n * r
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    mk = lambda *s: torch.randn(*s, device=dev, generator=g, dtype=torch.float32).to(torch.bfloat16)
    # one prompt group per rank: prompt q/k/v (Call 1) shared with Call 2's context KV
    qc, kc, vc = mk(p, h, d), mk(p, hk, d), mk(p, hk, d)
    q, kd, vd = mk(t, h, d), mk(t, hk, d), mk(t, hk, d)
    doc, dod = mk(p, h, d), mk(t, h, d)
    cu = np.arange(0, t + 1, r, dtype=np.int64)
    cuc = np.array([0, p], dtype=np.int64)
    ctx_b = dkv.VarlenBatch(qc, kc, vc, cuc)
    dec = dkv.DualKVInput(q, kc, vc, kd, vd, cu)

    def step():
        # Call 1 + Call 2 fused: one forward launch, one backward launch (prompt grads cast once)
        oc, lc, od, ld = dkv.dualkv_two_call_fwd(qc, dec)
        return dkv.dualkv_two_call_bwd(qc, dec, oc, lc, doc, od, ld, dod, deterministic=False)

    def step_separate():
        # the reference's two separate calls (layer.py:243-255, 274-275), for comparison
        oc, lc = dkv.fa2_varlen_fwd(ctx_b)
        od, ld = dkv.dualkv_fwd(dec)
        dkv.dualkv_bwd(dec, od, ld, dod, deterministic=False)
        dkv.fa2_varlen_bwd(ctx_b, oc, lc, doc)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn, steps):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        barrier()
        ms = e0.elapsed_time(e1) / steps
        if world > 1:
            tt = torch.tensor([ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = tt.item()
        return ms

    clocks = ClockSampler()
    clocks.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # ---- headline: device-resident inputs, K steps, with per-kernel events from libdkv
    lib.dkv_profile_begin()
    ms = timed(step, args.steps)
    fms, fl, bms, bl, al = (ctypes.c_double(), ctypes.c_int32(), ctypes.c_double(), ctypes.c_int32(),
                            ctypes.c_int32())
    lib.dkv_profile_end(ctypes.byref(fms), ctypes.byref(fl), ctypes.byref(bms), ctypes.byref(bl),
                        ctypes.byref(al))
    # fwd / bwd split (separately timed passes)
    saved = {}

    def fwd_only():
        saved["oc"], saved["lc"], saved["od"], saved["ld"] = dkv.dualkv_two_call_fwd(qc, dec)

    fwd_ms = timed(fwd_only, args.steps)

    def bwd_only():
        dkv.dualkv_two_call_bwd(qc, dec, saved["oc"], saved["lc"], doc, saved["od"], saved["ld"], dod,
                                deterministic=False)

    bwd_ms = timed(bwd_only, args.steps)
    sep_ms = timed(step_separate, args.steps)
    fl_step = flops_fwdbwd(c)
    value = fl_step * world / (ms * 1e-3) / 1e12

    # ---- replicated N-copy baseline: same kernels over the N(P+R) layout
    rep = None
    if not args.no_replicated:
        s = p + r
        qr, kr, vr, dor = mk(n * s, h, d), mk(n * s, hk, d), mk(n * s, hk, d), mk(n * s, h, d)
        rb = dkv.VarlenBatch(qr, kr, vr, np.arange(0, n * s + 1, s, dtype=np.int64))

        def rep_step():
            o, l = dkv.fa2_varlen_fwd(rb)
            dkv.fa2_varlen_bwd(rb, o, l, dor)

        rep_step()
        rep_ms = timed(rep_step, max(1, min(args.steps, 3)))
        rep = {"ms_per_step": round(rep_ms, 3),
               "tflops_algorithmic": round(rep_flops_fwdbwd(c) / (rep_ms * 1e-3) / 1e12, 2),
               "speedup_dualkv_vs_ncopy": round(rep_ms / ms, 3)}
        del qr, kr, vr, dor, rb

    # ---- e2e: public API with pinned host buffers, H2D inputs + D2H outputs per step
    e2e = None
    if not args.no_e2e:
        host_in = {k: v.cpu().pin_memory() for k, v in
                   dict(qc=qc, kc=kc, vc=vc, q=q, kd=kd, vd=vd, doc=doc, dod=dod).items()}
        out_shapes = [(p, h, d), (t, h, d), (t, h, d), (p, hk, d), (p, hk, d), (t, hk, d), (t, hk, d),
                      (p, h, d)]
        host_out = [torch.empty(s_, dtype=torch.bfloat16).pin_memory() for s_ in out_shapes]
        h2d = sum(x.numel() * x.element_size() for x in host_in.values())
        d2h = sum(x.numel() * x.element_size() for x in host_out)

        def e2e_step():
            dv_ = {k: v.to(dev, non_blocking=True) for k, v in host_in.items()}
            di = dkv.DualKVInput(dv_["q"], dv_["kc"], dv_["vc"], dv_["kd"], dv_["vd"], cu)
            oc, lc, od, ld = dkv.dualkv_two_call_fwd(dv_["qc"], di)
            cq, gkc, gvc, gq, gkd, gvd = dkv.dualkv_two_call_bwd(dv_["qc"], di, oc, lc, dv_["doc"], od, ld,
                                                                 dv_["dod"], deterministic=False)
            # every output of the layer's attention: both O's and all six input gradients
            outs = [oc, od, gq, gkc, gvc, gkd, gvd, cq]
            for ho, o in zip(host_out, outs):
                ho.copy_(o, non_blocking=True)

        e2e_step()
        e2e_ms = timed(e2e_step, args.steps)
        e2e = {"value": round(fl_step * world / (e2e_ms * 1e-3) / 1e12, 3), "unit": "TFLOP/s",
               "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}
    clk = clocks.stop()

    # ---- roofline of the dominant kernel (backward main kernel of Call 2 + Call 1)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    peak_burst = peaks.get("bf16_tflops", 1590.0)
    # per step each main kernel launches once (Call 1 fused into the Call 2 launch); achieved =
    # algorithmic FLOPs / device time of that launch (CUDA events recorded around it by libdkv)
    launches_per_step = 1
    bwd_kernel_ms = bms.value / max(1, bl.value)
    fwd_kernel_ms = fms.value / max(1, fl.value)
    bwd_flops_per_launch = 10 * pairs(p, [r] * n) * h * d / launches_per_step
    fwd_flops_per_launch = 4 * pairs(p, [r] * n) * h * d / launches_per_step
    bwd_ach = bwd_flops_per_launch / (bwd_kernel_ms * 1e-3) / 1e12
    fwd_ach = fwd_flops_per_launch / (fwd_kernel_ms * 1e-3) / 1e12
    roof = {"bound": "tensor", "kernel": "dualkv_bwd_kernel (tcgen05; Call 1 fused into the Call 2 launch)",
            "achieved": round(bwd_ach, 2), "peak": peak_burst, "unit": "TFLOP/s",
            "frac": round(bwd_ach / peak_burst, 4), "traffic": None,
            "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)" if peaks else "fallback 1.59 PF",
            "fwd_kernel": {"achieved": round(fwd_ach, 2), "frac": round(fwd_ach / peak_burst, 4)},
            "kernel_ms": {"fwd_main_avg": round(fwd_kernel_ms, 4), "bwd_main_avg": round(bwd_kernel_ms, 4),
                          "fwd_main_share": round(fms.value / (ms * args.steps), 3),
                          "bwd_main_share": round(bms.value / (ms * args.steps), 3)}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        tf, sec = cpu_sample_tflops(reps=1, warmup=0)
        cpu = {"value": round(tf, 6), "unit": "TFLOP/s", "cores": cpu_threads(), "kind": "port",
               "sample": sample_desc(), "seconds": round(sec, 2)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (randn, bf16)",
            "config": {"workload": "C3: Qwen3-8B attention, one prompt group per GPU",
                       "N": n, "P": p, "R": r, "H": h, "H_k": hk, "d": d,
                       "global_groups": world, "parallelism": f"dp{world} over prompt groups",
                       "l2": "inputs larger than L2 (q alone 512 MiB > 126 MB)",
                       "unit_of_work": "Call1+Call2 fwd+bwd (reference run_bench dk unit), fused two-call launches",
                       "flops_per_group": fl_step},
            "fwd_ms": round(fwd_ms, 3), "bwd_ms": round(bwd_ms, 3),
            "separate_calls_ms_per_step": round(sep_ms, 3),
            "fwd_tflops": round(4 * pairs(p, [r] * n) * h * d / (fwd_ms * 1e-3) / 1e12, 2),
            "bwd_tflops": round(10 * pairs(p, [r] * n) * h * d / (bwd_ms * 1e-3) / 1e12, 2),
            "replicated_ncopy": rep, "e2e": e2e, "roofline": roof, "cpu_baseline": cpu,
            "gpu_launches": int(al.value), "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

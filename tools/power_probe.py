"""Clock/power during a long C3 backward loop (NVML sampled every 20 ms):
    [DKV_BWD_ABLATE=..] python tools/power_probe.py [fwd|bwd]"""
import os, sys, threading, time
import numpy as np
import pynvml
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_15422_b200 as dkv  # noqa: E402
which = sys.argv[1] if len(sys.argv) > 1 else "bwd"
n, p, r, h, hk, d = 32, 8192, 2048, 32, 8, 128
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
t = n * r
qc, kc, vc, doc = mk(p, h, d), mk(p, hk, d), mk(p, hk, d), mk(p, h, d)
q, kd, vd, dod = mk(t, h, d), mk(t, hk, d), mk(t, hk, d), mk(t, h, d)
inp = dkv.DualKVInput(q, kc, vc, kd, vd, np.arange(0, t + 1, r))
oc, lc, od, ld = dkv.dualkv_two_call_fwd(qc, inp)
if which == "bwd":
    run = lambda: dkv.dualkv_two_call_bwd(qc, inp, oc, lc, doc, od, ld, dod, deterministic=False)
else:
    run = lambda: dkv.dualkv_two_call_fwd(qc, inp)
for _ in range(3):
    run()
torch.cuda.synchronize()
pynvml.nvmlInit()
hd = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0]) if False else 0)
samples, stop = [], threading.Event()
def sampler():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(hd, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(hd) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(hd)))
        time.sleep(0.02)
th = threading.Thread(target=sampler); th.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = int(os.environ.get("REPS", "60"))
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
stop.set(); th.join()
s = np.array([x[:2] for x in samples[len(samples) // 5:]])
reasons = set(x[2] for x in samples)
print(f"{which} ablate={os.environ.get('DKV_BWD_ABLATE', '0')}/{os.environ.get('DKV_FWD_ABLATE', '0')} ms={e0.elapsed_time(e1) / reps:.3f} "
      f"sm_mhz median={np.median(s[:, 0]):.0f} min={s[:, 0].min():.0f} power_w median={np.median(s[:, 1]):.0f} "
      f"max={s[:, 1].max():.0f} reasons={sorted(hex(x) for x in reasons)} n={len(s)}")

"""Pinned host <-> device copy bandwidth: H2D alone, D2H alone, both concurrently (2 streams)."""
import torch
n = 1 << 29  # 1 GiB of bf16
h_in = torch.empty(n, dtype=torch.bfloat16).pin_memory()
h_out = torch.empty(n, dtype=torch.bfloat16).pin_memory()
d_a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
d_b = torch.randn(n, device="cuda").to(torch.bfloat16)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def h2d(): d_a.copy_(h_in, non_blocking=True)
def d2h(): h_out.copy_(d_b, non_blocking=True)
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
gb = n * 2 / 1e9
for nm, fn, f in (("H2D", h2d, 1), ("D2H", d2h, 1), ("both", both, 2)):
    ms = t(fn)
    print(f"{nm}: {ms:.2f} ms per {gb * f:.2f} GB -> {gb * f / ms * 1e3:.1f} GB/s")

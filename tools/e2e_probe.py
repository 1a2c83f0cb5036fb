"""Probe the host-fed e2e pipeline of bench.py: per-step compute-stream intervals, copies alone,
compute alone.  python tools/e2e_probe.py [nsteps] [nbuf]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_15422_b200 as dkv  # noqa: E402

nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
nbuf = int(sys.argv[2]) if len(sys.argv) > 2 else 2
n, p, r, h, hk, d = 32, 8192, 2048, 32, 8, 128
t0 = n * r
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
mk = lambda *s: torch.randn(*s, device=dev, generator=g).to(torch.bfloat16)
host_in = {k: v.cpu().pin_memory() for k, v in dict(qc=mk(p, h, d), kc=mk(p, hk, d), vc=mk(p, hk, d), q=mk(t0, h, d),
                                                     kd=mk(t0, hk, d), vd=mk(t0, hk, d), doc=mk(p, h, d),
                                                     dod=mk(t0, h, d)).items()}
cu0 = np.arange(0, t0 + 1, r)
out_shapes = [(p, h, d), (t0, h, d), (t0, h, d), (p, hk, d), (p, hk, d), (t0, hk, d), (t0, hk, d), (p, h, d)]
host_out = [[torch.empty(s_, dtype=torch.bfloat16).pin_memory() for s_ in out_shapes] for _ in range(nbuf)]
dev_in = [{k: torch.empty_like(v, device=dev) for k, v in host_in.items()} for _ in range(nbuf)]
s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def attention(dv_):
    di = dkv.DualKVInput(dv_["q"], dv_["kc"], dv_["vc"], dv_["kd"], dv_["vd"], cu0)
    oc, lc, od, ld = dkv.dualkv_two_call_fwd(dv_["qc"], di)
    cq, gkc, gvc, gq, gkd, gvd = dkv.dualkv_two_call_bwd(dv_["qc"], di, oc, lc, dv_["doc"], od, ld, dv_["dod"],
                                                         deterministic=False)
    return [oc, od, gq, gkc, gvc, gkd, gvd, cq]


def run(k_steps, do_in=True, do_cmp=True, do_out=True):
    mk_ev = lambda: [torch.cuda.Event(enable_timing=True) for _ in range(k_steps)]
    ev_in, ev_cs, ev_ce, ev_out = mk_ev(), mk_ev(), mk_ev(), mk_ev()
    start = torch.cuda.current_stream()
    for st_ in (s_in, s_cmp, s_out):
        st_.wait_stream(start)
    keep = []
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(start)
    for k in range(k_steps):
        b = k % nbuf
        with torch.cuda.stream(s_in):
            if k >= nbuf:
                s_in.wait_event(ev_ce[k - nbuf])
            if do_in:
                for key, v in host_in.items():
                    dev_in[b][key].copy_(v, non_blocking=True)
            ev_in[k].record(s_in)
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(ev_in[k])
            if k >= nbuf:
                s_cmp.wait_event(ev_out[k - nbuf])
            ev_cs[k].record(s_cmp)
            outs = attention(dev_in[b]) if do_cmp else [torch.empty(s_, dtype=torch.bfloat16, device=dev) for s_ in out_shapes]
            ev_ce[k].record(s_cmp)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_ce[k])
            if do_out:
                for ho, o in zip(host_out[b], outs):
                    ho.copy_(o, non_blocking=True)
            ev_out[k].record(s_out)
        for o in outs:
            o.record_stream(s_out)
        keep.append(outs)
    for st_ in (s_in, s_cmp, s_out):
        start.wait_stream(st_)
    e1 = torch.cuda.Event(enable_timing=True)
    e1.record(start)
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1)
    cs = [e0.elapsed_time(e) for e in ev_cs]
    ce = [e0.elapsed_time(e) for e in ev_ce]
    ins = [e0.elapsed_time(e) for e in ev_in]
    outs_ = [e0.elapsed_time(e) for e in ev_out]
    return total, cs, ce, ins, outs_


run(2)
for name, kw in (("full", {}), ("compute only", dict(do_in=False, do_out=False)),
                 ("copies only", dict(do_cmp=False))):
    total, cs, ce, ins, outs_ = run(nsteps, **kw)
    print(f"{name:14s} nbuf={nbuf}: {total / nsteps:.2f} ms/step over {nsteps} steps")
    if name == "full":
        for k in range(nsteps):
            print(f"  step {k}: H2D done {ins[k]:7.1f}  compute {cs[k]:7.1f} -> {ce[k]:7.1f} ({ce[k] - cs[k]:5.1f})  D2H done {outs_[k]:7.1f}")

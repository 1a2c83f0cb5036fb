"""Small two-call DualKV fwd+bwd (ragged, partial tiles, R_i = 0, G = 4), a d = 64 DualKV fwd+bwd,
the fused repack+RoPE gather, a multi-group two-call launch (one group with an empty prompt), the
fused QKV epilogue (norm + RoPE + scatter) and the attention layer fwd+bwd, for compute-sanitizer."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_15422_b200 as dkv  # noqa: E402
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
p, rl, h, hk, d = 200, [77, 0, 150, 33], 8, 2, 128
t = sum(rl)
qc, kc, vc, doc = mk(p, h, d), mk(p, hk, d), mk(p, hk, d), mk(p, h, d)
q, kd, vd, dod = mk(t, h, d), mk(t, hk, d), mk(t, hk, d), mk(t, h, d)
dec = dkv.DualKVInput(q, kc, vc, kd, vd, np.concatenate([[0], np.cumsum(rl)]))
oc, lc, od, ld = dkv.dualkv_two_call_fwd(qc, dec)
for det in (True, False):
    gr = dkv.dualkv_two_call_bwd(qc, dec, oc, lc, doc, od, ld, dod, deterministic=det)
if os.environ.get("SAN_SMALL"):  # racecheck on the cluster kernels is slow: the first case only
    torch.cuda.synchronize()
    print("ok small")
    raise SystemExit(0)
# d = 64 (tensor-core backward with the zero-padded K^T panel)
q64, kc64, vc64, kd64, vd64, do64 = mk(t, h, 64), mk(p, hk, 64), mk(p, hk, 64), mk(t, hk, 64), mk(t, hk, 64), mk(t, h, 64)
in64 = dkv.DualKVInput(q64, kc64, vc64, kd64, vd64, np.concatenate([[0], np.cumsum(rl)]))
o64, l64 = dkv.dualkv_fwd(in64)
g64 = dkv.dualkv_bwd(in64, o64, l64, do64, deterministic=True)
from paper_2605_15422_b200 import packing as pk  # noqa: E402
plan = pk.make_plan([(p, rl), (31, [5, 64])])
xs = [mk(plan.total_standard, hh, d) for hh in (h, hk, hk)]
rq, rk, rv = dkv.repack_rope_to_dualkv(*xs, plan, 1e6)
# multi-group launch: three groups (one with P = 0) in one fwd and one bwd launch
groups = [(130, [40, 0, 77]), (0, [19]), (257, [128, 3])]
pc = sum(x[0] for x in groups)
lens = [r for _, rs in groups for r in rs]
tt = sum(lens)
mq, mkc, mvc, mdoc = mk(pc, h, d), mk(pc, hk, d), mk(pc, hk, d), mk(pc, h, d)
mqd, mkd, mvd, mdod = mk(tt, h, d), mk(tt, hk, d), mk(tt, hk, d), mk(tt, h, d)
gs = np.concatenate([[0], np.cumsum([len(rs) for _, rs in groups])])
gc = np.concatenate([[0], np.cumsum([x[0] for x in groups])])
minp = dkv.DualKVInput(mqd, mkc, mvc, mkd, mvd, np.concatenate([[0], np.cumsum(lens)]), group_seq_cu=gs, group_ctx_cu=gc)
moc, mlc, mod, mld = dkv.dualkv_two_call_fwd(mq, minp)
mg = dkv.dualkv_two_call_bwd(mq, minp, moc, mlc, mdoc, mod, mld, mdod, deterministic=False, return_context_f32=True)
# the attention layer: one QKV GEMM, fused q/k norm + RoPE + scatter, every group in one launch
from paper_2605_15422_b200.layer import DualKVSelfAttention  # noqa: E402
blk = DualKVSelfAttention(128, h, hk, d, rope_base=1e6, qk_norm=True)
lplan = pk.make_plan(groups)
x = mk(lplan.total_dualkv, 128).requires_grad_()
y = blk(x, lplan)
y.backward(torch.ones_like(y))
# GQA ratio that does not divide the tile rows (G = 5, Qwen3-14B): padded tiles, zeroed padding rows
q5, kc5, vc5, kd5, vd5, do5 = mk(t, 20, d), mk(p, 4, d), mk(p, 4, d), mk(t, 4, d), mk(t, 4, d), mk(t, 20, d)
in5 = dkv.DualKVInput(q5, kc5, vc5, kd5, vd5, np.concatenate([[0], np.cumsum(rl)]))
o5, l5 = dkv.dualkv_fwd(in5)
g5 = dkv.dualkv_bwd(in5, o5, l5, do5, deterministic=False)
torch.cuda.synchronize()
print("ok", [float(x.float().abs().sum()) for x in gr], float(rq.float().abs().sum() + rk.float().abs().sum()),
      [float(x.float().abs().sum()) for x in g64])

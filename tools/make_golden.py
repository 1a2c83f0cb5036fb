"""Generate golden vectors by running the REFERENCE CPU implementation.

Run in the build container only (needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tools/make_golden.py

Writes tests/golden/*.npz.  The fixtures pin `oracle/` (and, through it,
the GPU parity tests) to the reference's own outputs.  Inputs are stored
alongside outputs so the tests never depend on the RNG implementation.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

from dualkv.costmodel import Scenario, attention_flops, visible_pairs
from dualkv.fa2 import VarlenBatch, fa2_varlen_bwd, fa2_varlen_fwd
from dualkv.kernel import DualKVInput, context_grad_contributions, dualkv_bwd, dualkv_fwd
from dualkv.packing import RolloutGroup, RolloutResponse, pack_dualkv, pack_standard
from dualkv.refattn import DenseAttentionCase, ref_attention_bwd, ref_attention_fwd
from dualkv.tensor import Precision, Tensor, bf16_round

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")
PREC = {"f64": Precision.F64, "f32": Precision.F32, "bf16": Precision.BF16EMU}


def _inputs(rng, n, p, r_list, h, h_k, d):
    t = int(sum(r_list))
    mk = lambda *s: rng.normal(size=s)
    return dict(q=mk(t, h, d), k_context=mk(p, h_k, d), v_context=mk(p, h_k, d),
                k_decoded=mk(t, h_k, d), v_decoded=mk(t, h_k, d), d_out=mk(t, h, d),
                cu=np.concatenate([[0], np.cumsum(r_list)]).astype(np.int64))


def dualkv_case(name, seed, n, p, r_list, h, h_k, d, prec, tile, store):
    rng = np.random.default_rng(seed)
    x = _inputs(rng, n, p, r_list, h, h_k, d)
    pr = PREC[prec]
    inp = DualKVInput(Tensor(x["q"], pr), Tensor(x["k_context"], pr), Tensor(x["v_context"], pr),
                      Tensor(x["k_decoded"], pr), Tensor(x["v_decoded"], pr), x["cu"],
                      tile_size=tile)
    dout = Tensor(x["d_out"], pr)
    o, lse = dualkv_fwd(inp)
    grads = dualkv_bwd(inp, o, lse, dout)
    contribs = context_grad_contributions(inp, o, lse, dout)
    rec = {f"in_{k}": (np.asarray(pr.quantize(v)) if k != "cu" else v) for k, v in x.items()}
    rec.update(o=o.data, lse=lse.data, dq=grads[0].data, dkc=grads[1].data, dvc=grads[2].data,
               dkd=grads[3].data, dvd=grads[4].data)
    if contribs and sum(c[0].size for c in contribs) < 200_000:  # keep fixtures small
        rec["contrib_k"] = np.stack([c[0] for c in contribs])
        rec["contrib_v"] = np.stack([c[1] for c in contribs])
    # replicated-baseline view of the same problem (fa2 over [P;R_i] per seq)
    meta = dict(kind="dualkv", n=n, p=p, r_list=[int(r) for r in r_list], h=h, h_k=h_k, d=d,
                prec=prec, tile=tile, scale=float(inp.softmax_scale))
    store[name] = (meta, rec)


def varlen_case(name, seed, lens, h, h_k, d, prec, tile, store):
    rng = np.random.default_rng(seed)
    t = int(sum(lens))
    pr = PREC[prec]
    q, k, v, do = (rng.normal(size=s) for s in ((t, h, d), (t, h_k, d), (t, h_k, d), (t, h, d)))
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    b = VarlenBatch(Tensor(q, pr), Tensor(k, pr), Tensor(v, pr), cu, tile_size=tile)
    o, lse = fa2_varlen_fwd(b)
    dq, dk, dv = fa2_varlen_bwd(b, o, lse, Tensor(do, pr))
    rec = dict(in_q=pr.quantize(q), in_k=pr.quantize(k), in_v=pr.quantize(v),
               in_d_out=pr.quantize(do), in_cu=cu, o=o.data, lse=lse.data, dq=dq.data,
               dk=dk.data, dv=dv.data)
    meta = dict(kind="varlen", lens=[int(x) for x in lens], h=h, h_k=h_k, d=d, prec=prec,
                tile=tile, scale=float(b.softmax_scale))
    store[name] = (meta, rec)


def dense_case(name, seed, sq, sk, h, h_k, d, offset, store):
    rng = np.random.default_rng(seed)
    q, k, v, do = (rng.normal(size=s) for s in ((sq, h, d), (sk, h_k, d), (sk, h_k, d), (sq, h, d)))
    case = DenseAttentionCase(Tensor(q), Tensor(k), Tensor(v), causal_offset=offset)
    o, lse = ref_attention_fwd(case)
    dq, dk, dv = ref_attention_bwd(case, o, lse, Tensor(do))
    rec = dict(in_q=q, in_k=k, in_v=v, in_d_out=do, o=o.data, lse=lse.data, dq=dq.data,
               dk=dk.data, dv=dv.data)
    store[name] = (dict(kind="dense", offset=offset, h=h, h_k=h_k, d=d), rec)


def draw_config(rng):
    """The reference sweep generator (verify.py:54-70), re-drawn here."""
    n = int(rng.integers(1, 9))
    p = int(rng.integers(0, 34))
    r_list = rng.integers(0, 18, size=n)
    if r_list.sum() == 0:
        r_list[int(rng.integers(0, n))] = int(rng.integers(1, 18))
    h_k = int(rng.choice([1, 2]))
    group = int(rng.choice([1, 2, 4]))
    return dict(n=n, p=p, r_list=[int(r) for r in r_list], tile=int(rng.choice([1, 3, 4, 8])),
                h_k=h_k, h=h_k * group, d=int(rng.choice([1, 4, 8])))


def main():
    os.makedirs(OUT, exist_ok=True)
    store = {}
    # randomized sweep in the reference's own config space, all precisions
    rng = np.random.default_rng(2024)
    for i in range(12):
        cfg = draw_config(rng)
        prec = ["f64", "f32", "bf16"][i % 3]
        dualkv_case(f"sweep{i:02d}_{prec}", 1000 + i, cfg["n"], cfg["p"], cfg["r_list"],
                    cfg["h"], cfg["h_k"], cfg["d"], prec, cfg["tile"], store)
    # edge cases named by the reference tests
    dualkv_case("partial_tiles", 0, 2, 7, [5, 6], 2, 1, 4, "f64", 4, store)     # test_dualkv.py:80
    dualkv_case("zero_len_resp", 1, 3, 5, [3, 0, 2], 2, 1, 4, "f64", 4, store)  # test_dualkv.py:90
    dualkv_case("p0", 2, 3, 0, [4, 5, 3], 4, 2, 8, "f64", 4, store)             # verify.py:272
    dualkv_case("gqa4_d16_bf16", 3, 3, 40, [20, 9, 33], 8, 2, 16, "bf16", 16, store)
    # medium shapes with multi-tile regions at head dims the GPU kernels run natively
    dualkv_case("mid_d64_f32", 4, 4, 256, [128, 128, 128, 128], 2, 1, 64, "f32", 64, store)
    dualkv_case("mid_d128_bf16", 5, 3, 200, [77, 150, 1], 4, 1, 128, "bf16", 64, store)
    varlen_case("varlen_f64", 6, [6, 9, 0, 3], 4, 2, 8, "f64", 4, store)
    varlen_case("varlen_bf16", 7, [130, 64, 5], 4, 1, 64, "bf16", 64, store)
    dense_case("dense_offset", 8, 5, 12, 4, 2, 8, 7, store)

    for name, (meta, rec) in store.items():
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), meta=json.dumps(meta), **rec)

    # scalar / integer known answers
    special = np.array([1.0, -2.5, 0.0, 1.0 / 3.0, 1.00390625, 3.4e38, np.inf, -np.inf, np.nan,
                        1e-40, -7.1234567, 65504.0, 1.0078125 + 2**-9], dtype=np.float32)
    rnd = np.random.default_rng(0).normal(0, 100.0, 4096).astype(np.float32)
    grid = np.concatenate([special, rnd])
    np.savez_compressed(os.path.join(OUT, "bf16_round.npz"), x=grid,
                        y=np.asarray(bf16_round(grid), dtype=np.float32))

    groups = [("a", [1, 2], [[3], [4]]), ("b", [5], [[6, 7], [8, 9], [10, 11]]),
              ("c", [10, 11, 12], [[20, 21], [30, 31, 32, 33]]), ("e", [], [[], [7]])]
    rg = [RolloutGroup(pid, pr, [RolloutResponse(t, 1.0) for t in rs]) for pid, pr, rs in groups]
    std, dk = pack_standard(rg), pack_dualkv(rg)
    packing = dict(
        groups=[[len(pr), [len(t) for t in rs]] for _, pr, rs in groups],
        std_tokens=std.token_ids.tolist(), dk_tokens=dk.token_ids.tolist(),
        std_cu=std.all_cu_seqlens().tolist(), std_pos=std.position_ids().tolist(),
        dk_pos=dk.position_ids().tolist(),
        dk_layout=[[g.context_start, g.context_span, g.resp_start, g.resp_cu.tolist()]
                   for g in dk.groups],
    )
    cost = []
    for (n, p, r, h, hk, d) in [(32, 8192, 2048, 32, 8, 128), (16, 4096, 1024, 32, 8, 128),
                                (4, 256, 128, 8, 8, 64), (32, 16384, 2048, 32, 4, 128)]:
        scn = Scenario(n=n, p=p, r=r, heads=h, kv_heads=hk, head_dim=d)
        cost.append(dict(n=n, p=p, r=r, h=h, d=d,
                         pairs_dk=visible_pairs(scn, "dualkv"),
                         pairs_std=visible_pairs(scn, "standard"),
                         flops_dk=attention_flops(scn, "dualkv"),
                         flops_std=attention_flops(scn, "standard")))
    with open(os.path.join(OUT, "packing_cost.json"), "w") as f:
        json.dump(dict(packing=packing, cost=cost), f, indent=1)
    total = sum(os.path.getsize(os.path.join(OUT, x)) for x in os.listdir(OUT))
    print(f"wrote {len(store)} kernel cases, {total/1e6:.2f} MB to {os.path.abspath(OUT)}")


if __name__ == "__main__":
    sys.exit(main())

"""Opt-in kernel variants stay correct: each runs in a subprocess with its switch
set (the switches are read once per process) and must match the default path on the same
two-call problem -- ragged responses, partial tiles, an empty response, GQA."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2605_15422_b200 as dkv
g = torch.Generator(device="cuda").manual_seed(3)
mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(torch.bfloat16)
p, rl, d = 300, [77, 0, 520, 33, 129], 128
h, hk = int(sys.argv[3]), int(sys.argv[4])
t = sum(rl)
qc, kc, vc, doc = mk(p, h, d), mk(p, hk, d), mk(p, hk, d), mk(p, h, d)
q, kd, vd, dod = mk(t, h, d), mk(t, hk, d), mk(t, hk, d), mk(t, h, d)
inp = dkv.DualKVInput(q, kc, vc, kd, vd, np.concatenate([[0], np.cumsum(rl)]))
oc, lc, od, ld = dkv.dualkv_two_call_fwd(qc, inp)
gr = dkv.dualkv_two_call_bwd(qc, inp, oc, lc, doc, od, ld, dod, deterministic=True)
torch.cuda.synchronize()
out = {"oc": oc, "od": od, "lc": lc, "ld": ld}
out.update({f"g{i}": x for i, x in enumerate(gr)})
torch.save({k: v.float().cpu() for k, v in out.items()}, sys.argv[2])
print(json.dumps({"ok": True}))
"""


def _run(tmp_path, name, env_extra, h, hk):
    path = tmp_path / f"{name}_{h}_{hk}.pt"
    env = {**os.environ, **env_extra}
    r = subprocess.run([sys.executable, "-c", _SCRIPT, ROOT, str(path), str(h), str(hk)], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    import torch
    return torch.load(path)


# each switch flips one CTA-pair (cta_group::2) kernel against its single-CTA counterpart:
# the forward pair is the default (DKV_FWD_PAIR=0 turns it off), the backward pair is opt-in;
# DKV_FWD_QT is the pair forward with Q as a TMEM operand and 64-key KV tiles (opt-in)
@pytest.mark.parametrize("switch,h,hk", [("DKV_FWD_PAIR", 16, 4), ("DKV_FWD_PAIR", 32, 4), ("DKV_BWD_PAIR", 16, 4),
                                         ("DKV_BWD_PAIR", 8, 8), ("DKV_BWD_PAIR", 32, 4), ("DKV_BWD_PAIR", 32, 2),
                                         ("DKV_FWD_PAIR+DKV_FWD_QT", 16, 4), ("DKV_FWD_PAIR+DKV_FWD_QT", 32, 4),
                                         ("DKV_FWD_PAIR+DKV_FWD_QT", 8, 8)])
def test_variant_matches_default(switch, h, hk, tmp_path, cuda_device):
    base = _run(tmp_path, "single", {"DKV_FWD_PAIR": "0", "DKV_BWD_PAIR": "0"}, h, hk)
    var = _run(tmp_path, switch, {"DKV_FWD_PAIR": "0", "DKV_BWD_PAIR": "0", **{s: "1" for s in switch.split("+")}},
               h, hk)
    for k, ref in base.items():
        got = var[k]
        tol = 1e-3 if k.startswith("l") else 2e-2
        err = ((got - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item() if not k.startswith("l") \
            else (got - ref).abs().max().item()
        assert err <= tol, f"{switch}: {k} differs from the default path by {err:.3e}"


def test_pair_backward_at_headline_c3(cuda_device):
    """The opt-in CTA-pair backward through the bench's exact call at full C3 against the
    independent f64 slices (test_gpu_headline.py, run in a subprocess with the switch set)."""
    env = {**os.environ, "DKV_BWD_PAIR": "1"}
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-m", "gpu",
                        os.path.join(ROOT, "tests", "test_gpu_headline.py"), "-k", "C3 or c3"],
                       env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    assert " passed" in r.stdout and "failed" not in r.stdout, r.stdout[-2000:]

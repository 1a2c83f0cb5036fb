"""Golden rollout JSONL + the REFERENCE's manifests (cli.py:174-293, packing.py:159-322).

    PYTHONPATH=/root/reference/pkg/src python tools/make_golden_rollouts.py   (build container only)

Writes tests/golden/rollouts.jsonl and tests/golden/rollouts_manifests.json (the reference's
`dualkv pack` output for micro-batch capacities 4 and 8 in both modes, and its rho values).
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile

import numpy as np

from dualkv.cli import read_rollouts
from dualkv.packing import pack_dualkv, token_reduction_ratio

GOLD = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")


def main():
    rng = np.random.default_rng(5)
    recs = []
    for g in range(6):  # interleaved records of 6 prompts, 1-5 responses each, ragged lengths
        p = [int(x) for x in rng.integers(0, 1000, int(rng.integers(0, 12)))]
        for i in range(int(rng.integers(1, 6))):
            recs.append(dict(prompt_id=f"p{g}", prompt_tokens=p,
                             response_tokens=[int(x) for x in rng.integers(0, 1000, int(rng.integers(0, 9)))],
                             advantage=float(np.round(rng.normal(), 3))))
    order = rng.permutation(len(recs))
    path = os.path.join(GOLD, "rollouts.jsonl")
    with open(path, "w") as f:
        for i in order:
            f.write(json.dumps(recs[i]) + "\n")
    out = {"manifests": {}}
    for mode in ("dualkv", "standard"):
        for mb in (5, 8):
            with tempfile.TemporaryDirectory() as td:
                mpath = os.path.join(td, "m.jsonl")
                rc = subprocess.run([sys.executable, "-m", "dualkv", "pack", "--input", path, "--mode", mode, "--mb", str(mb),
                                     "--out", mpath], capture_output=True, text=True)
                assert rc.returncode == 0, rc.stderr
                out["manifests"][f"{mode}_{mb}"] = [json.loads(l) for l in open(mpath)]
    groups = read_rollouts(path)
    out["group_order"] = [g.prompt_id for g in groups]
    out["rho_all"] = [str(token_reduction_ratio(groups))]
    out["dk_positions"] = pack_dualkv(groups).position_ids().tolist()
    with open(os.path.join(GOLD, "rollouts_manifests.json"), "w") as f:
        json.dump(out, f)
    print("wrote", len(recs), "records;", {k: len(v) for k, v in out["manifests"].items()})


if __name__ == "__main__":
    main()

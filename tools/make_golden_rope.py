"""Golden vectors for RoPE at logical positions, from the REFERENCE (layer.py:182-209).

    PYTHONPATH=/root/reference/pkg/src python tools/make_golden_rope.py   (build container only)

Writes tests/golden/rope.npz: inputs, the DualKV-layout logical positions of a small group
(PackedBatch.position_ids, packing.py:105-120) and the reference's rope / rope_bwd outputs.
"""

from __future__ import annotations

import json
import os

import numpy as np

from dualkv.layer import rope, rope_bwd
from dualkv.packing import RolloutGroup, RolloutResponse, pack_dualkv

OUT = os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "rope.npz")


def main():
    rng = np.random.default_rng(7)
    grp = [RolloutGroup("g", list(range(9)), [RolloutResponse(list(range(4)), 1.0), RolloutResponse([], 1.0),
                                              RolloutResponse(list(range(6)), 1.0)]),
           RolloutGroup("h", list(range(3)), [RolloutResponse(list(range(5)), 1.0)])]
    pos = pack_dualkv(grp).position_ids()
    rec = {"pos": np.asarray(pos, dtype=np.int64)}
    cases = []
    for i, (h, d, base) in enumerate([(3, 8, 10000.0), (2, 128, 10000.0), (4, 64, 1000000.0)]):
        x = rng.normal(size=(len(pos), h, d))
        rec[f"x{i}"] = x
        rec[f"y{i}"] = rope(x, pos, base)
        rec[f"b{i}"] = rope_bwd(x, pos, base)
        cases.append(dict(h=h, d=d, base=base))
    # large logical positions (P + r at Qwen3-scale prompts)
    big = np.array([0, 1, 8191, 8192, 10239, 16384 + 2047], dtype=np.int64)
    xb = rng.normal(size=(len(big), 2, 128))
    rec.update(pos_big=big, x_big=xb, y_big=rope(xb, big, 1000000.0))
    np.savez_compressed(OUT, meta=json.dumps(dict(kind="rope", cases=cases, big_base=1000000.0)), **rec)
    print("wrote", os.path.abspath(OUT), len(pos), "rows")


if __name__ == "__main__":
    main()

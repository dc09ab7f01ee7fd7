#!/usr/bin/env python3
"""How a frozen 16-bit bound holds across network seeds: max |delta_gpu - delta_oracle| per seed
(8 motions x 4096 points each) for precision argv[1] (fp16 | bf16), next to the frozen bound."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2402_15281_b200 as S  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

PREC = sys.argv[1] if len(sys.argv) > 1 else "fp16"
SEEDS = [int(x) for x in sys.argv[2:]] or [100, 2024, 3, 5, 17, 21, 29, 31, 77, 1234]
frozen = json.loads((ROOT / "tests" / "golden" / f"{PREC}_bounds.json").read_text())
NETS = {
    "plain_4x256": (WORKLOADS["c2"].program, "he", "c2"),
    "deepsdf_8x512_skip4": (WORKLOADS["c3"].program, "he", "c3"),
    "plain_6x512": (WORKLOADS["c4"].program, "he", "c4"),
    "fig2_5x512": (S.fig2(5, 512, 6), "ref", "c2"),
    "fig2_3x256": (S.fig2(3, 256, 6), "ref", "c2"),
}
for name, (prog, bound, wkey) in NETS.items():
    w = WORKLOADS[wkey]
    errs = []
    for seed in SEEDS:
        pts, q = w.make(seed=seed, motions=8, points=4096)
        params = S.init_params(prog, seed, bound)
        r = S.Model(prog, params).query_min(pts, q, w.margin, precision=PREC, per_point=True)
        opp = O.query_min(prog, params, pts, q, w.margin, per_point=True, threads=32)[3]
        errs.append(float(np.abs(r.per_point.astype(np.float64) - opp).max()))
    b = frozen[name]["bound"]
    print(f"{PREC} {name:22s} bound {b:.4g}  worst seed {max(errs):.4g} ({max(errs) / b:.2f} of the bound)  per seed "
          + " ".join(f"{e:.3g}" for e in errs), flush=True)

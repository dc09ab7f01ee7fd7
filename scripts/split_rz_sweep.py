#!/usr/bin/env python3
"""fp32_split error against the oracle per calibration seed, for the truncation compensation
in SVN_SPLIT_RZ (run once per value: the library reads it at model creation).
    for c in 0 0.25 0.3; do SVN_SPLIT_RZ=$c python scripts/split_rz_sweep.py; done
WIDTH=512 sweeps the width-512 networks (c3/c5, c4, the paper's Fig. 2 5x512)."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2402_15281_b200 as S  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

SEEDS = [int(s) for s in os.environ.get("SEEDS", "3 7 17 23 31 41 100 2024 5 11 13 19").split()]
WIDTH = int(os.environ.get("WIDTH", "256"))
MOTIONS, POINTS = (16, 4096) if WIDTH == 256 else (8, 2048)
w = WORKLOADS["c2"]
if WIDTH == 256:
    nets = {"plain_4x256": (w.program, "he", "c2"), "fig2_3x256": (S.fig2(3, 256, 6), "ref", "c2")}
else:
    nets = {"deepsdf_8x512_skip4": (WORKLOADS["c3"].program, "he", "c3"),
            "plain_6x512": (WORKLOADS["c4"].program, "he", "c4"), "fig2_5x512": (S.fig2(5, 512, 6), "ref", "c3")}
c = os.environ.get("SVN_SPLIT_RZ", "default")
for name, (prog, bound, key) in nets.items():
    errs = []
    w = WORKLOADS[key]
    for seed in SEEDS:
        pts, q = w.make(seed=seed, motions=MOTIONS, points=POINTS)
        params = S.init_params(prog, seed, bound)
        r = S.Model(prog, params).query_min(pts, q, w.margin, precision="fp32_split", per_point=True)
        opp = O.query_min(prog, params, pts, q, w.margin, per_point=True, threads=os.cpu_count())[3]
        errs.append(float(np.abs(r.per_point.astype(np.float64) - opp).max()))
    print(f"rz={c} {name}: max {max(errs):.3e} | " + " ".join(f"{s}:{e:.2e}" for s, e in zip(SEEDS, errs)), flush=True)

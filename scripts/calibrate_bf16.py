#!/usr/bin/env python3
"""Freeze the per-point bound of a 16-bit tensor-core precision (bf16 default, or fp16: argv[1])
per network: bound = 2 x the max |delta_gpu - delta_oracle| over a fixed
calibration subset (seed 100, 8 motions x 4096 points), rounded up to 2 significant digits.
Writes gpurun_out/<prec>_bounds.json; the committed copy is tests/golden/<prec>_bounds.json."""
import json
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2402_15281_b200 as S  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

NETS = {
    "plain_4x256": (WORKLOADS["c2"].program, "he", "c2"),
    "deepsdf_8x512_skip4": (WORKLOADS["c3"].program, "he", "c3"),
    "plain_6x512": (WORKLOADS["c4"].program, "he", "c4"),
    "fig2_5x512": (S.fig2(5, 512, 6), "ref", "c2"),
    "fig2_3x256": (S.fig2(3, 256, 6), "ref", "c2"),
}


def up2(x):
    e = math.floor(math.log10(x))
    return math.ceil(x / 10 ** (e - 1)) * 10 ** (e - 1)


PREC = sys.argv[1] if len(sys.argv) > 1 else "bf16"
out = {"method": f"2 x max |{PREC} - oracle fp32| on seed 100, 8 motions x 4096 points, rounded up (2 s.f.)"}
for name, (prog, bound, wkey) in NETS.items():
    w = WORKLOADS[wkey]
    pts, q = w.make(seed=100, motions=8, points=4096)
    params = S.init_params(prog, 100, bound)
    r = S.Model(prog, params).query_min(pts, q, w.margin, precision=PREC, per_point=True)
    _, _, _, opp = O.query_min(prog, params, pts, q, w.margin, per_point=True, threads=32)
    err = float(np.abs(r.per_point.astype(np.float64) - opp).max())
    scale = float(np.abs(opp).max())
    out[name] = {"max_err": err, "bound": up2(2 * err), "max_abs_delta": scale}
    print(name, out[name], flush=True)
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / f"{PREC}_bounds.json").write_text(json.dumps(out, indent=1))

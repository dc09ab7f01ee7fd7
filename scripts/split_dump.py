#!/usr/bin/env python3
"""GPU side of scripts/emulate_split.py: per-point fp32_split (and bf16) outputs of the c2
network for a few seeds -> gpurun_out/split_dump_<seed>.npz."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2402_15281_b200 as S  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = WORKLOADS[cfg]
(ROOT / "gpurun_out").mkdir(exist_ok=True)
for seed in [int(s) for s in (sys.argv[2:] or ["2024", "7"])]:
    pts, q = w.make(seed=seed, motions=16, points=4096)
    q = q[:4]
    params = S.init_params(w.program, seed, w.bound)
    m = S.Model(w.program, params)
    out = {}
    for prec in ("fp32_split", "bf16"):
        try:
            out[prec] = m.query_min(pts, q, w.margin, precision=prec, per_point=True).per_point
        except Exception as e:  # noqa: BLE001
            print(prec, "unavailable:", e)
    np.savez(ROOT / "gpurun_out" / f"split_dump_{cfg}_{seed}.npz", per_point=out.get("fp32_split"), bf16=out.get("bf16"))
    print("dumped", cfg, seed)

#!/usr/bin/env python3
"""Randomised soak of the host API: random (network, motions, points, precision) cases, each
compared with the bit-identical FP32 path within the precision's frozen bound (class outside the
band, argmin within the bound), plus the cascade's class on every motion.  Runs for argv[1]
seconds (default 120) from seed argv[2]; exits 1 on the first failure with the case printed."""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2402_15281_b200 as S  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
B = {p: {k: v["bound"] for k, v in json.loads((ROOT / "tests" / "golden" / f"{p}_bounds.json").read_text()).items()
         if isinstance(v, dict)} for p in ("fp16", "bf16", "fp32_split")}
NETS = [("c2", WORKLOADS["c2"].program, "he"), ("c3", WORKLOADS["c3"].program, "he"), ("c4", WORKLOADS["c4"].program, "he"),
        ("c2", S.fig2(3, 256, 6), "ref"), ("c2", S.fig2(5, 512, 6), "ref")]
models = {}
t_end, n = time.time() + budget, 0
while time.time() < t_end:
    wkey, prog, bound = NETS[rng.integers(len(NETS))]
    w = WORKLOADS[wkey]
    seed = int(rng.integers(1, 50))
    key = (prog.name, seed)
    if key not in models:
        if len(models) > 12:
            models.pop(next(iter(models))).close()
        models[key] = S.Model(prog, S.init_params(prog, seed, bound))
    model = models[key]
    M = int(rng.choice([1, 2, 3, 7, 37, 64, 75, 149, 300]))
    P = int(rng.choice([1, 31, 128, 129, 255, 256, 257, 1000, 3000, 4096, 9473, 20000, 70001]))
    if M * P > 6_000_000:
        P = max(1, 6_000_000 // M)
    pts, q = w.make(seed=seed + 1000, motions=M, points=P)
    margin = float(rng.choice([w.margin, 0.005, -0.3]))
    exact = model.query_min(pts, q, margin, precision="fp32")
    case = f"{prog.name} seed {seed} M {M} P {P} margin {margin}"
    for prec in ("bf16", "fp16", "fp32_split"):
        bnd = B[prec][prog.name]
        r = model.query_min(pts, q, margin, precision=prec)
        d = np.abs(r.min.astype(np.float64) - exact.min.astype(np.float64))
        out = np.abs(exact.min.astype(np.float64) - margin) > bnd
        if not (d.max() <= bnd and np.array_equal(r.free[out], exact.free[out])):
            print("FAIL", prec, case, "max |dmin|", d.max(), "bound", bnd)
            sys.exit(1)
    cr, st = model.query_min_cascade(pts, q, margin, B["fp16"][prog.name], B["fp32_split"][prog.name])
    if not np.array_equal(cr.free, exact.free):
        print("FAIL cascade", case, st)
        sys.exit(1)
    n += 1
print(f"stress ok: {n} random cases x 3 precisions + cascade in {budget:.0f} s")

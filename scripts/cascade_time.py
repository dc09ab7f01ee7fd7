#!/usr/bin/env python3
"""Cost of the exact-for-every-motion classification (svn_query_min_cascade) next to the plain
precisions, through the host API, on a config's network with its output bias calibrated to ~50 %
free motions:  python scripts/cascade_time.py [c3] [motions] [points]"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2402_15281_b200 as S  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = WORKLOADS[key]
M = int(sys.argv[2]) if len(sys.argv) > 2 else w.motions
P = int(sys.argv[3]) if len(sys.argv) > 3 else w.points
B = {p: json.loads((ROOT / "tests" / "golden" / f"{p}_bounds.json").read_text())[w.program.name]["bound"]
     for p in ("fp16", "bf16", "fp32_split")}
pts, q = w.make(seed=0, motions=M, points=P)
params = S.init_params(w.program, 0, w.bound)
model = S.Model(w.program, params)
mn = model.query_min(pts, q, w.margin, precision="fp16").min
params = params.copy()
params[-1] += np.float32(w.margin - np.median(mn.astype(np.float64)))
model = S.Model(w.program, params)


def timed(f, n=3):
    f()
    t = []
    for _ in range(n):
        t0 = time.perf_counter()
        r = f()
        t.append(time.perf_counter() - t0)
    return r, min(t)


print(f"{key}: {M} motions x {P} points, {w.program.name}, margin {w.margin}")
res = {}
for prec in ("bf16", "fp16", "fp32_split"):
    res[prec], t = timed(lambda: model.query_min(pts, q, w.margin, precision=prec))
    print(f"  {prec:10s} {t * 1e3:9.2f} ms  {M * P / t / 1e6:8.1f} M queries/s   free {res[prec].free.mean():.3f}")
for coarse in ("fp16", "bf16"):
    (r, st), t = timed(lambda: model.query_min_cascade(pts, q, w.margin, B[coarse], B["fp32_split"], coarse=coarse))
    mism_split = int((r.free != res["fp32_split"].free).sum())
    print(f"  cascade/{coarse:5s} {t * 1e3:7.2f} ms  {M * P / t / 1e6:8.1f} M queries/s   stages {st}  "
          f"class differs from fp32_split on {mism_split} motions (within its band of the margin); "
          f"{coarse} alone differs from the cascade on {int((res[coarse].free != r.free).sum())}")

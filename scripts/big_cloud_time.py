#!/usr/bin/env python3
"""predict_min_distance (the reference's entry point: double cloud, one motion) on a 2^24-point
cloud through the host API, SVN_PIPELINE=0|1 from the environment."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2402_15281_b200 as S  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

w = WORKLOADS["c5single"]
pts, q = w.make(seed=0)
cloud = pts.astype(np.float64)
dof = w.program.dof
model = S.Model(w.program, S.init_params(w.program, 0, w.bound))
for prec in ("bf16", "fp16"):
    model.predict_min_distance(cloud, q[0, :dof], q[0, dof:], precision=prec)
    t = []
    for _ in range(3):
        t0 = time.perf_counter()
        r = model.predict_min_distance(cloud, q[0, :dof], q[0, dof:], precision=prec)
        t.append(time.perf_counter() - t0)
    print(f"predict_min_distance {prec}: {cloud.shape[0]} points, {min(t) * 1e3:.1f} ms per call, min {r[0]:.6f} at {r[1]}")

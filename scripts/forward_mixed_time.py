#!/usr/bin/env python3
"""forward_eval (nn.cpp:95-130) on a batch whose rows all differ in motion — the reference's
eval_mae (bench.cpp:80-90) and training-validation (nn.cpp:370) calls — timed per precision."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2402_15281_b200 as S  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
for key, precs in (("c2", ("fp32_exact", "fp32_split", "bf16")), ("c3", ("fp32_exact", "bf16"))):
    w = WORKLOADS[key]
    m = S.Model(w.program, S.init_params(w.program, 1, w.bound))
    pts, q = w.make(seed=1, motions=64, points=4096)
    rng = np.random.default_rng(0)
    rows = np.concatenate([pts[rng.integers(0, pts.shape[0], B)], q[rng.integers(0, 64, B)]], axis=1).astype(np.float32)
    for prec in precs:
        m.forward_eval(rows[:1000], precision=prec)
        t0 = time.perf_counter()
        m.forward_eval(rows, precision=prec)
        dt = time.perf_counter() - t0
        print(f"{key} {prec:10s} {B} mixed-motion rows: {dt * 1e3:8.2f} ms  ({B / dt / 1e6:7.2f} M rows/s)", flush=True)

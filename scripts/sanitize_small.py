"""Tiny invocation of every kernel for compute-sanitizer (memcheck) runs."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2402_15281_b200 as S  # noqa: E402
from paper_2402_15281_b200.robot import default_robot, gcc_min_distance  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

for key, precs in (("c3", ("bf16", "fp32", "fp32_exact")), ("c2", ("bf16", "fp32", "fp32_exact"))):
    w = WORKLOADS[key]
    p = S.init_params(w.program, 1, w.bound)
    pts, q = w.make(seed=1, motions=3, points=300)
    m = S.Model(w.program, p)
    for prec in precs:
        r = m.query_min(pts, q, w.margin, precision=prec, per_point=True)
        raw = np.concatenate([pts[:50], q[np.arange(50) % 3]], axis=1).astype(np.float32)
        m.forward_eval(raw, precision=prec)
        print(key, prec, r.min)
    m.eval_grid([0, 0, 0], 0.05, (3, 4, 5), q[0, :6], q[0, 6:], precision="bf16")
r = default_robot(6)
pts, q = WORKLOADS["c2"].make(seed=2, motions=2, points=200)
print(gcc_min_distance(r, pts, q, steps=20, margin=0.02))
print("sanitize run complete")

"""Per-call latency of the drop-in proxy (svn_predict_min_distance: one motion, host cloud)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_15281_b200 as S  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

for name, prog, bound in (("fig2_5x512", S.fig2(5, 512, 6), "ref"), ("plain_4x256", WORKLOADS["c2"].program, "he")):
    m = S.Model(prog, S.init_params(prog, 1, bound))
    for P in (3000, 20000):
        pts, q = WORKLOADS["c2"].make(seed=1, motions=1, points=P)
        cloud = pts.astype(np.float64)
        for prec in ("bf16", "fp32"):
            for _ in range(20):
                m.predict_min_distance(cloud, q[0, :6], q[0, 6:], precision=prec)
            ts = []
            for _ in range(200):
                t0 = time.perf_counter()
                m.predict_min_distance(cloud, q[0, :6], q[0, 6:], precision=prec)
                ts.append(time.perf_counter() - t0)
            print(f"{name:12s} P={P:6d} {prec:5s} median {np.median(ts) * 1e6:8.1f} us  p90 {np.quantile(ts, 0.9) * 1e6:8.1f} us")

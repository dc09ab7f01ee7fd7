"""Time the GPU geometric checker at c3 size (1024 motions x 65536 points x 200 steps)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2402_15281_b200.robot import default_robot, gcc_min_distance  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

w = WORKLOADS["c3"]
M = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
pts, q = w.make(seed=3, motions=M, points=65536)
r = default_robot(6)
gcc_min_distance(r, pts[:1000], q[:2], steps=200, margin=0.02)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    d, f = gcc_min_distance(r, pts, q, steps=200, margin=0.02)
    ts.append(time.perf_counter() - t0)
print(f"gcc {M} motions x 65536 points x 200 steps: {min(ts):.3f} s (free {f.mean():.3f})")

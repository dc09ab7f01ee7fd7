"""Time svn_gcc_nn_search (Alg. 1 on the GPU) on a bin scene where most motions collide."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_15281_b200 as S  # noqa: E402
from paper_2402_15281_b200.robot import default_robot, gcc_min_distance, gcc_nn_search  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

r = default_robot(6)
rng = np.random.default_rng(12)
cloud = rng.uniform([0.2, -0.5, 0.1], [0.6, 0.5, 0.8], size=(65536, 3))
M = 1024
q01 = rng.uniform(-1, 1, size=(M, 12)) * np.concatenate([r.upper, r.upper])
w = WORKLOADS["c2"]
params = S.init_params(w.program, 12, w.bound)
model = S.Model(w.program, params)
for prec in ("bf16", "fp32"):
    gcc_nn_search(model, r, cloud[:1000], q01[:8], steps=200, margin=0.02, precision=prec)
    t0 = time.perf_counter()
    res = gcc_nn_search(model, r, cloud, q01, steps=200, margin=0.02, precision=prec, batch=64)
    print(prec, {k: (round(v, 4) if isinstance(v, float) else v) for k, v in res.items()}, f"wall {time.perf_counter() - t0:.3f} s")
t0 = time.perf_counter()
d, f = gcc_min_distance(r, cloud, q01, steps=200, margin=0.02)
print(f"full checker on all {M} motions: {time.perf_counter() - t0:.3f} s, free fraction {f.mean():.3f}")

#!/usr/bin/env python3
"""svn_query_min_multi per call with the cloud passed every time against the resident scene
(svn_multi_set_scene), through the host API on the devices of this box:
    python scripts/scene_time.py [devices, e.g. 0 or 0,1,2,3]
Cases: the paper's per-scene batch (Fig. 2 5x512, 64 motions x 20000 points), c4's scene
(4096 x 100000) and c5single (one motion x 2^24 points, point-sharded)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2402_15281_b200 as S  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

devices = [int(d) for d in (sys.argv[1] if len(sys.argv) > 1 else "0").split(",")]


def timed(f, n=7):
    f()
    t = []
    for _ in range(n):
        t0 = time.perf_counter()
        r = f()
        t.append(time.perf_counter() - t0)
    return r, float(np.median(t))


for key, M, P, shard in (("paper", 64, 20000, "motions"), ("c4", 4096, 100000, "motions"),
                         ("c5single", 1, 1 << 24, "points")):
    w = WORKLOADS[key]
    params = S.init_params(w.program, 0, w.bound)
    pts, q = w.make(seed=0, motions=M, points=P)
    mg = S.MultiModel(w.program, params, devices=devices)
    a, t_call = timed(lambda: mg.query_min(pts, q, w.margin, precision="bf16", shard=shard))
    t0 = time.perf_counter()
    mg.set_scene(pts)
    t_up = time.perf_counter() - t0
    b, t_res = timed(lambda: mg.query_min(None, q, w.margin, precision="bf16", shard=shard))
    same = np.array_equal(a.min, b.min) and np.array_equal(a.argmin, b.argmin) and np.array_equal(a.free, b.free)
    print(f"{key:9s} {M:5d} x {P:9d} ({shard:7s}, {len(devices)} device(s)): cloud per call {t_call * 1e3:9.3f} ms | "
          f"resident scene {t_res * 1e3:9.3f} ms (+ one upload {t_up * 1e3:.3f} ms) | bits equal {same}")
    mg.close()

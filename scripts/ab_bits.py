"""Bit comparison of the bf16 path between two builds of the library (A/B):
   python scripts/ab_bits.py dump OUT.npz   (under SVN_LIB=scripts/ab/x.so or the in-tree build)
   python scripts/ab_bits.py cmp A.npz B.npz"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

if sys.argv[1] == "dump":
    import paper_2402_15281_b200 as S
    from paper_2402_15281_b200.workloads import WORKLOADS
    out = {}
    nets = {"c2": (WORKLOADS["c2"].program, "he", "c2"), "c3": (WORKLOADS["c3"].program, "he", "c3"),
            "c4": (WORKLOADS["c4"].program, "he", "c4"), "fig2_5x512": (S.fig2(5, 512, 6), "ref", "c2"),
            "fig2_3x256": (S.fig2(3, 256, 6), "ref", "c2")}
    for name, (prog, bound, wkey) in nets.items():
        w = WORKLOADS[wkey]
        params = S.init_params(prog, 100, bound)
        model = S.Model(prog, params)
        for M, P in ((8, 4096), (300, 5000)):  # small (128-row tiles, K0 stream) and large (256-row tiles, ext ring)
            pts, q = w.make(seed=100, motions=M, points=P)
            r = model.query_min(pts, q, w.margin, precision="bf16", per_point=True)
            out[f"{name}_{M}x{P}"] = r.per_point
        raw = np.concatenate([pts[:777], np.random.default_rng(1).uniform(-1, 1, (777, 2 * prog.dof)).astype(np.float32)], 1)
        out[f"{name}_rows"] = model.forward_eval(raw.astype(np.float32), precision="bf16")
    np.savez(sys.argv[2], **out)
else:
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for k in a.files:
        same = np.array_equal(a[k].view(np.uint32), b[k].view(np.uint32))
        print(k, "identical" if same else f"DIFFERENT max|d|={np.abs(a[k] - b[k]).max():.3e}")

"""Quick check of fp32_split on the width-512 networks (c3/c5 DeepSDF, c4 plain, Fig. 2 5x512)
against the oracle on small seeded samples: max per-point error and argmin agreement."""
import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2402_15281_b200 as S
from oracle import oracle as O
from paper_2402_15281_b200.workloads import WORKLOADS
for key, prog, bound in [("c3", WORKLOADS["c3"].program, "he"), ("c4", WORKLOADS["c4"].program, "he"), ("c3", S.fig2(5,512,6), "ref")]:
    w = WORKLOADS[key]
    params = S.init_params(prog, 5, bound)
    for M, P in [(1, 1000), (3, 3000)]:
        pts, q = w.make(seed=5, motions=M, points=P)
        r = S.Model(prog, params).query_min(pts, q, w.margin, precision="fp32_split", per_point=True)
        omin, oarg, ofree, opp = O.query_min(prog, params, pts, q, w.margin, per_point=True, threads=16)
        err = np.abs(r.per_point.astype(np.float64) - opp).max()
        print(prog.name, M, P, "max err %.3e" % err, "min eq", np.array_equal(r.argmin, oarg), flush=True)

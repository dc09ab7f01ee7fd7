#!/usr/bin/env python3
"""Generate the golden fixtures under tests/golden/ (run in the build container).

  mt19937_64_std.txt   std::mt19937_64 stream + the reference's Rng::uniform transform,
                       dumped by oracle/pin_rng.cpp (the C++ standard library engine the
                       reference wraps, rng.hpp:16) — pins the oracle's RNG restatement.
  <case>.npz           seeded inputs, per-point delta from the C oracle (fp32) and from the
                       independent torch fp64 oracle, per-motion min/argmin/free, and the
                       sha256 of the seeded parameter buffer.

These freeze the restated oracle on the BASELINE configs (plain / DeepSDF networks have no
reference implementation) after it has been checked against the reference's
own nn.cpp on Fig. 2 networks (tests/golden/make_ref_golden.py -> ref_fig2.npz,
tests/test_ref_oracle.py), the standard-library RNG and the torch fp64 implementation.
"""
from __future__ import annotations

import hashlib
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O, torch_fp64 as T  # noqa: E402
import paper_2402_15281_b200 as S  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

CASES = {
    # name: (program, bound, workload for inputs, motions, points, seed, margin)
    "c1_full": (WORKLOADS["c1"].program, "he", "c1", 1, 4096, 11, 0.02),
    "c2_sub": (WORKLOADS["c2"].program, "he", "c2", 4, 1024, 12, 0.02),
    "c3_sub": (WORKLOADS["c3"].program, "he", "c3", 2, 512, 13, 0.02),
    "c4_sub": (WORKLOADS["c4"].program, "he", "c4", 2, 512, 14, 0.02),
    "fig2_5x512_sub": (S.fig2(5, 512, 6), "ref", "c2", 2, 256, 15, 0.02),
    "fig2_3x256_sub": (S.fig2(3, 256, 6), "ref", "c2", 3, 300, 16, 0.0),
}


def dump_rng():
    exe = ROOT / "oracle" / "build" / "pin_rng"
    if not exe.exists():
        O.build()
    lines = []
    for seed in (5489, 1, 42):
        out = subprocess.run([str(exe), str(seed), "1000"], check=True, capture_output=True, text=True).stdout
        lines += [f"{seed} {l}" for l in out.strip().splitlines()]
    (HERE / "mt19937_64_std.txt").write_text("# seed u64 uniform(-b,b) float(uniform(-b,b)), b=1/sqrt(15)\n"
                                             + "\n".join(lines) + "\n")


def make_case(name, program, bound, wkey, M, P, seed, margin):
    w = WORKLOADS[wkey]
    pts, q = w.make(seed=seed, motions=M, points=P)
    params = O.init_params(program, seed, bound)
    mn, am, fr, pp = O.query_min(program, params, pts, q, margin, per_point=True, threads=8)
    pp64 = T.query(program, params, pts, q)
    err = np.abs(pp.astype(np.float64) - pp64).max()
    assert err < 1e-5, (name, err)
    np.savez_compressed(HERE / f"{name}.npz", program=program.name, flags=program.flags_array(),
                        width=program.width, dof=program.dof, bound=bound, seed=seed, margin=margin,
                        points=pts, q01=q, delta_f32=pp, delta_f64=pp64, min=mn, argmin=am, free=fr,
                        params_sha256=hashlib.sha256(params.tobytes()).hexdigest())
    print(f"{name}: {M}x{P}, max|f32-f64|={err:.2e}, free={fr.tolist()}")


if __name__ == "__main__":
    dump_rng()
    for name, args in CASES.items():
        make_case(name, *args)

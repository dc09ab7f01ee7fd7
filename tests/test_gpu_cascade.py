"""svn_query_min_cascade: the margin classification exact for EVERY motion.  The batch runs on a
tensor-core precision; only the motions within that precision's stated band of the margin (or
not finite) are evaluated again on fp32_split, and those within fp32_split's band on the FP32
path — so `free` equals the FP32 path's class (the reference's, bit for bit) with no exceptions,
while almost all the work stays on the fast path."""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2402_15281_b200 as S
from paper_2402_15281_b200 import abi
from paper_2402_15281_b200.workloads import WORKLOADS

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"
BOUNDS = {p: {k: v["bound"] for k, v in json.loads((G / f"{p}_bounds.json").read_text()).items() if isinstance(v, dict)}
          for p in ("fp16", "bf16", "fp32_split")}


def _calibrated(w, seed, M, P):
    """The workload's network with its output bias moved so that about half the motions are free
    (seeded networks are otherwise almost always in collision: a vacuous class check)."""
    pts, q = w.make(seed=seed, motions=M, points=P)
    params = S.init_params(w.program, seed, w.bound)
    mn = S.Model(w.program, params).query_min(pts, q, w.margin, precision="fp32").min
    params = params.copy()
    params[-1] += np.float32(w.margin - np.median(mn.astype(np.float64)))
    return pts, q, params


@pytest.mark.parametrize("coarse", ["fp16", "bf16"])
@pytest.mark.parametrize("key,M,P", [("c3", 400, 3000), ("c2", 300, 4096), ("c4", 250, 2500)])
def test_cascade_class_equals_the_fp32_path_for_every_motion(key, M, P, coarse):
    w = WORKLOADS[key]
    pts, q, params = _calibrated(w, 41, M, P)
    model = S.Model(w.program, params)
    exact = model.query_min(pts, q, w.margin, precision="fp32")
    assert 0.3 <= exact.free.mean() <= 0.7
    name = w.program.name
    r, stages = model.query_min_cascade(pts, q, w.margin, BOUNDS[coarse][name], BOUNDS["fp32_split"][name], coarse=coarse)
    assert np.array_equal(r.free, exact.free)  # every motion, no ambiguous band left
    assert stages[0] == M and stages[1] < M and stages[2] <= stages[1]
    band = np.abs(exact.min.astype(np.float64) - w.margin)
    # the second stage saw at least the motions inside the coarse band around the margin ...
    print(f"{key} {coarse}: stages {stages}, inside the coarse band (exact) {(band <= BOUNDS[coarse][name]).sum()}")
    # ... and min / argmin are within the evaluating stage's bound of the exact path
    assert np.abs(r.min.astype(np.float64) - exact.min).max() <= BOUNDS[coarse][name]
    # the coarse precision alone does have class mismatches or an ambiguous band on this case
    c = model.query_min(pts, q, w.margin, precision=coarse)
    amb = band <= BOUNDS[coarse][name]
    assert np.array_equal(c.free[~amb], exact.free[~amb])
    if coarse == "fp16":  # the tighter band re-evaluates fewer motions than bf16's would
        _, st_bf = model.query_min_cascade(pts, q, w.margin, BOUNDS["bf16"][name], BOUNDS["fp32_split"][name], coarse="bf16")
        assert stages[1] < st_bf[1]


def test_cascade_recovers_rows_outside_the_fp16_range():
    """fp16 reports a row that left its range as -inf (not free); the cascade sends that motion to
    the finer stages, where fp32_split reports the same and the FP32 path returns the real value."""
    w = WORKLOADS["c2"]
    params = S.init_params(w.program, 29, w.bound)
    pts, q = w.make(seed=29, motions=5, points=600)
    big = pts.copy()
    big[5] = (3.0e6, -2.0e6, 1.0e6)
    model = S.Model(w.program, params)
    exact = model.query_min(big, q, w.margin, precision="fp32")
    assert np.all(np.isfinite(exact.min))
    assert np.all(model.query_min(big, q, w.margin, precision="fp16").min == -np.inf)
    name = w.program.name
    r, stages = model.query_min_cascade(big, q, w.margin, BOUNDS["fp16"][name], BOUNDS["fp32_split"][name])
    assert stages == (5, 5, 5)
    assert np.array_equal(r.min, exact.min) and np.array_equal(r.argmin, exact.argmin) and np.array_equal(r.free, exact.free)


def test_cascade_without_fp32_split_and_argument_checks():
    # a Fig. 2 network at width 256: all three stages; zero bands: nothing is re-evaluated
    prog = S.fig2(3, 256, 6)
    params = S.init_params(prog, 7, "ref")
    pts, q = WORKLOADS["c2"].make(seed=7, motions=40, points=700)
    model = S.Model(prog, params)
    r, stages = model.query_min_cascade(pts, q, 0.005, 0.0, 0.0)
    assert stages == (40, 0, 0)
    assert np.array_equal(r.min, model.query_min(pts, q, 0.005, precision="fp16").min)
    # an infinite coarse band sends every motion down: the result is the FP32 path's, bit for bit
    r, stages = model.query_min_cascade(pts, q, 0.005, np.inf, np.inf)
    exact = model.query_min(pts, q, 0.005, precision="fp32")
    assert stages == (40, 40, 40) and np.array_equal(r.min, exact.min) and np.array_equal(r.argmin, exact.argmin)
    with pytest.raises(abi.SvnError):
        model.query_min_cascade(pts, q, 0.005, 0.01, 1e-5, coarse="fp32")
    with pytest.raises(abi.SvnError):
        model.query_min_cascade(pts, q, 0.005, -1.0, 1e-5)


@pytest.mark.parametrize("coarse", ["fp16", "bf16"])
def test_cascade_over_the_box_equals_one_device(coarse):
    """svn_query_min_cascade_multi: motions split over three workers (device 0 three times),
    every output and the per-stage motion counts equal to one device's cascade."""
    w = WORKLOADS["c3"]
    M, P = 301, 3000
    pts, q, params = _calibrated(w, 43, M, P)
    name = w.program.name
    one, st_one = S.Model(w.program, params).query_min_cascade(pts, q, w.margin, BOUNDS[coarse][name],
                                                               BOUNDS["fp32_split"][name], coarse=coarse)
    mg = S.MultiModel(w.program, params, devices=[0, 0, 0])
    box, st_box = mg.query_min_cascade(pts, q, w.margin, BOUNDS[coarse][name], BOUNDS["fp32_split"][name], coarse=coarse)
    assert np.array_equal(box.free, one.free) and np.array_equal(box.min, one.min) and np.array_equal(box.argmin, one.argmin)
    assert st_box == st_one and st_box[0] == M and 0 < st_box[1] < M
    exact = S.Model(w.program, params).query_min(pts, q, w.margin, precision="fp32")
    assert np.array_equal(box.free, exact.free)
    # fewer motions than workers, and the argument checks of the single-device entry
    two, _ = mg.query_min_cascade(pts, q[:2], w.margin, BOUNDS[coarse][name], BOUNDS["fp32_split"][name], coarse=coarse)
    assert np.array_equal(two.free, exact.free[:2])
    with pytest.raises(abi.ReferenceInvalidArgument):
        mg.query_min_cascade(pts, q, w.margin, -1.0, 0.0, coarse=coarse)
    with pytest.raises(abi.ReferenceInvalidArgument, match="empty point cloud"):
        mg.query_min_cascade(pts[:0], q, w.margin, 0.1, 0.0, coarse=coarse)
    mg.close()

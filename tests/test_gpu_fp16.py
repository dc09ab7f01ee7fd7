"""precision="fp16": the single-pass tensor-core kernels (width 512 pair kernel, width 256
two-tiles-in-flight kernel) on fp16 operands instead of bf16 — same instruction rate, 11
significant bits, a bound about 8 times tighter (tests/golden/fp16_bounds.json, frozen by
`scripts/calibrate_bf16.py fp16`).  Every code path the bf16 tests cover is run in fp16 against
the CPU oracle: K0's extension stream and the in-kernel ext ring, both tile sizes, the
model-constant bias extension (ext == 1), Fig. 2 blocks with the BN fold, a make_normalizer-style
normaliser, forward_eval rows of mixed motions, ragged clouds, the NaN-at-0 rule, and the fp16
range: a weight outside it refuses the precision, an activation outside it is reported as
delta = -inf (class "not free"), never dropped.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2402_15281_b200 as S
from fig2_bn import randomize_bn
from oracle import oracle as O
from paper_2402_15281_b200 import abi
from paper_2402_15281_b200.workloads import WORKLOADS
from test_gpu_parity import BF16_BOUND
from test_gpu_ref_parity import trained_like

pytestmark = pytest.mark.gpu

_H = json.loads((Path(__file__).resolve().parent / "golden" / "fp16_bounds.json").read_text())
FP16_BOUND = {k: v["bound"] for k, v in _H.items() if isinstance(v, dict)}


def _check(r, omin, oarg, ofree, opp, margin, bound):
    M = omin.shape[0]
    err = np.abs(r.per_point.astype(np.float64) - opp).max()
    assert err <= bound, err
    assert np.array_equal(r.min, r.per_point.min(axis=1)) and np.array_equal(r.argmin, r.per_point.argmin(axis=1))
    amb = np.abs(omin.astype(np.float64) - margin) <= bound
    assert np.array_equal(r.free[~amb], ofree[~amb])
    d_at = opp[np.arange(M), r.argmin]
    assert np.all((r.argmin == oarg) | (d_at - omin <= bound))
    return err


def test_bounds_are_tighter_than_bf16_and_inside_the_margins():
    """The point of the precision: every stated fp16 bound is at least 6x tighter than the bf16
    one; the BASELINE networks' bounds sit inside the 0.02 m margin and the reference's own
    Fig. 2 5x512 network inside its default 5 mm margin (bench.hpp:85)."""
    for k, b in FP16_BOUND.items():
        assert b * 6 <= BF16_BOUND[k], (k, b, BF16_BOUND[k])
    for k in ("plain_4x256", "deepsdf_8x512_skip4", "plain_6x512"):
        assert FP16_BOUND[k] < 0.02
    assert FP16_BOUND["fig2_5x512"] < 0.005


@pytest.mark.parametrize("key,M,P", [("c2", 4, 3000), ("c3", 3, 1500), ("c4", 3, 1300), ("c1", 1, 4096)])
def test_fp16_within_bound(key, M, P):
    w = WORKLOADS[key]
    pts, q = w.make(seed=3, motions=M, points=P)
    params = S.init_params(w.program, 3, w.bound)
    model = S.Model(w.program, params)
    r = model.query_min(pts, q, w.margin, precision="fp16", per_point=True)
    o = O.query_min(w.program, params, pts, q, w.margin, per_point=True, threads=8)
    bound = FP16_BOUND[w.program.name]
    err = _check(r, *o, w.margin, bound)
    e16 = np.abs(model.query_min(pts, q, w.margin, precision="bf16", per_point=True).per_point.astype(np.float64) - o[3]).max()
    print(f"{key}: fp16 max|err| = {err:.3e} (bound {bound}), bf16 {e16:.3e}")
    assert err * 4 <= e16


@pytest.mark.parametrize("key,M,P", [("c3", 300, 5000), ("c2", 200, 4100), ("c4", 160, 3001)])
def test_fp16_large_launch_against_the_fp32_path(key, M, P):
    """Enough tiles for the 256-row form (and, at width 512, the in-kernel ext ring): checked
    against the bit-identical FP32 path instead of the CPU oracle."""
    w = WORKLOADS[key]
    pts, q = w.make(seed=17, motions=M, points=P)
    params = S.init_params(w.program, 17, w.bound)
    model = S.Model(w.program, params)
    r = model.query_min(pts, q, w.margin, precision="fp16", per_point=True)
    e = model.query_min(pts, q, w.margin, precision="fp32", per_point=True)
    _check(r, e.min, e.argmin, e.free, e.per_point.astype(np.float64), w.margin, FP16_BOUND[w.program.name])
    # batch invariance: a slice of the motions alone gives the same bits
    s = model.query_min(pts, q[7:19], w.margin, precision="fp16", per_point=True)
    assert np.array_equal(s.per_point.view(np.uint32), r.per_point[7:19].view(np.uint32))


@pytest.mark.parametrize("key,M,P", [("c2", 4, 1500), ("c3", 3, 900), ("c4", 3, 800)])
def test_fp16_with_normaliser_and_biases(key, M, P):
    """A make_normalizer-style normaliser and nonzero hidden biases (the model-constant K=16 bias
    extension of non-concat layers), and rows of mixed motions through forward_eval."""
    w = WORKLOADS[key]
    pts, q = w.make(seed=21, motions=M, points=P)
    p = trained_like(w.program, S.init_params(w.program, 21, w.bound), pts, 21)
    model = S.Model(w.program, p)
    o = O.query_min(w.program, p, pts, q, w.margin, per_point=True, threads=8)
    bound = FP16_BOUND[w.program.name]
    _check(model.query_min(pts, q, w.margin, precision="fp16", per_point=True), *o, w.margin, bound)
    rows = np.concatenate([pts[:200], q[np.arange(200) % M]], axis=1).astype(np.float32)
    ref_rows = O.forward_eval(w.program, p, rows)
    assert np.abs(model.forward_eval(rows, precision="fp16").astype(np.float64) - ref_rows).max() <= bound
    grouped = np.concatenate([np.repeat(pts[:50], M, axis=0), np.tile(q, (50, 1))], axis=1).astype(np.float32)
    grouped = grouped[np.argsort(np.tile(np.arange(M), 50), kind="stable")]  # runs of 50 rows per motion
    ref_g = O.forward_eval(w.program, p, grouped)
    assert np.abs(model.forward_eval(grouped, precision="fp16").astype(np.float64) - ref_g).max() <= bound


@pytest.mark.parametrize("width,blocks,neg", [(256, 3, None), (512, 5, None), (512, 5, 2)])
def test_fp16_fig2_with_trained_like_bn(width, blocks, neg):
    """The reference's own architecture with BN statistics (affine fold into the weights, the
    f16x2 residual update; a negative-gamma layer keeps its affine)."""
    prog = S.fig2(blocks, width, 6)
    params = randomize_bn(prog, S.init_params(prog, 31, "ref"), 31, negative_gamma_layer=neg)
    pts, q = WORKLOADS["c2"].make(seed=31, motions=3, points=900)
    params = trained_like(prog, params, pts, 31)
    o = O.query_min(prog, params, pts, q, 0.005, per_point=True, threads=8)
    r = S.Model(prog, params).query_min(pts, q, 0.005, precision="fp16", per_point=True)
    _check(r, *o, 0.005, FP16_BOUND[f"fig2_{blocks}x{width}"])


@pytest.mark.parametrize("P", [1, 63, 129, 255, 257, 1000])
def test_fp16_ragged_point_counts(P):
    for key in ("c2", "c3"):
        w = WORKLOADS[key]
        params = S.init_params(w.program, 5, w.bound)
        pts, q = w.make(seed=5, motions=3, points=P)
        r = S.Model(w.program, params).query_min(pts, q, w.margin, precision="fp16", per_point=True)
        o = O.query_min(w.program, params, pts, q, w.margin, per_point=True, threads=8)
        _check(r, *o, w.margin, FP16_BOUND[w.program.name])


def test_fp16_nan_point_at_index_zero_sticks():
    """nn.cpp:476-478: a NaN at row 0 is returned.  With fp16 operands a non-finite row elsewhere
    is reported as -inf (not free) rather than skipped — the safe side of the margin test."""
    prog = S.fig2(2, 256, 6)
    params = S.init_params(prog, 5, "ref")
    pts, q = WORKLOADS["c2"].make(seed=5, motions=2, points=300)
    bad = pts.copy()
    bad[0] = np.nan
    r = S.Model(prog, params).query_min(bad, q, 0.0, precision="fp16")
    assert np.all(r.argmin == 0) and not r.free.any()
    assert np.all(np.isnan(r.min) | (r.min == -np.inf))


def test_fp16_activation_overflow_is_reported_not_dropped():
    w = WORKLOADS["c2"]
    params = S.init_params(w.program, 29, w.bound)
    pts, q = w.make(seed=29, motions=3, points=600)
    big = pts.copy()
    big[5] = (3.0e6, -2.0e6, 1.0e6)  # layer-0 activations ~1e5-1e6: beyond fp16
    m = S.Model(w.program, params)
    r = m.query_min(big, q, w.margin, precision="fp16", per_point=True)
    assert np.all(r.per_point[:, 5] == -np.inf)
    assert np.all(r.min == -np.inf) and np.all(r.argmin == 5) and not r.free.any()
    o = O.query_min(w.program, params, big, q, w.margin, per_point=True, threads=8)[3]
    ok = np.delete(np.arange(600), 5)
    assert np.abs(r.per_point[:, ok].astype(np.float64) - o[:, ok]).max() <= FP16_BOUND[w.program.name]


def test_fp16_refused_when_a_weight_is_outside_the_range():
    w = WORKLOADS["c2"]
    params = S.init_params(w.program, 1, w.bound)
    params[2 * (3 + 2 * w.program.dof) + 17] = 7.0e4
    pts, q = w.make(seed=1, motions=1, points=64)
    m = S.Model(w.program, params)
    with pytest.raises(abi.SvnError):
        m.query_min(pts, q, w.margin, precision="fp16")
    m.query_min(pts, q, w.margin, precision="bf16")  # bf16 has the fp32 range


def test_fp16_full_size_c3_against_the_fp32_path():
    """The whole c3 workload in fp16; 96 motions x the full cloud against the FP32 path: min
    within the bound, class equal outside a band that is now narrower than the margin."""
    w = WORKLOADS["c3"]
    params = S.init_params(w.program, 0, w.bound)
    pts, q = w.make(seed=0)
    model = S.Model(w.program, params)
    r = model.query_min(pts, q, w.margin, precision="fp16")
    bound = FP16_BOUND[w.program.name]
    ms = np.sort(np.random.default_rng(1).choice(q.shape[0], size=96, replace=False))
    exact = model.query_min(pts, q[ms], w.margin, precision="fp32")
    assert np.abs(r.min[ms].astype(np.float64) - exact.min.astype(np.float64)).max() <= bound
    for margin in (w.margin, float(np.median(exact.min))):
        outside = np.abs(exact.min.astype(np.float64) - margin) > bound
        assert np.array_equal((r.min[ms].astype(np.float64) > margin)[outside],
                              (exact.min.astype(np.float64) > margin)[outside])

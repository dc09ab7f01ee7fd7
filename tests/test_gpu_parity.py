"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star):
  fp32 / fp32_exact  the FP32 path: |delta_gpu - delta_oracle| <= 1e-5, met with zero error —
              SIMT FFMA in the oracle's order (oracle/sweptnet_oracle.c), bit-identical
  fp32_split  fp32-grade on tcgen05 (split-fp16 operands, q-fold, width 256):
              <= FP32_SPLIT_BOUND[network] (frozen, tests/golden/fp32_split_bounds.json)
  bf16        |delta_gpu - delta_oracle| <= BF16_BOUND[config] (frozen)
Classification is bit-exact except for motions whose oracle min is within the
bound of the margin ("ambiguous"), which are counted.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2402_15281_b200 as S
from oracle import oracle as O
from paper_2402_15281_b200.workloads import WORKLOADS

pytestmark = pytest.mark.gpu

# Stated bf16 bounds per network family, frozen by scripts/calibrate_bf16.py
# (2x the max |bf16 - oracle| on a fixed calibration subset).
_B = json.loads((Path(__file__).resolve().parent / "golden" / "bf16_bounds.json").read_text())
BF16_BOUND = {k: v["bound"] for k, v in _B.items() if isinstance(v, dict)}
_F = json.loads((Path(__file__).resolve().parent / "golden" / "fp32_split_bounds.json").read_text())
FP32_SPLIT_BOUND = {k: v["bound"] for k, v in _F.items() if isinstance(v, dict)}


def _case(key, M, P, seed=3):
    w = WORKLOADS[key]
    pts, q = w.make(seed=seed, motions=M, points=P)
    params = S.init_params(w.program, seed, w.bound)
    return w, pts, q, params


def _oracle(program, params, pts, q, margin):
    return O.query_min(program, params, pts, q, margin, per_point=True, threads=8)


@pytest.mark.parametrize("key,M,P", [("c1", 1, 4096), ("c2", 3, 1000)])
def test_fp32_exact_bit_identical(key, M, P):
    w, pts, q, params = _case(key, M, P)
    model = S.Model(w.program, params)
    r = model.query_min(pts, q, w.margin, precision="fp32_exact", per_point=True)
    omin, oarg, ofree, opp = _oracle(w.program, params, pts, q, w.margin)
    assert np.array_equal(r.per_point, opp), np.abs(r.per_point - opp).max()
    assert np.array_equal(r.min, omin) and np.array_equal(r.argmin, oarg) and np.array_equal(r.free, ofree)


@pytest.mark.parametrize("key,M,P", [("c1", 1, 4096), ("c2", 4, 2000), ("c3", 2, 700), ("c4", 2, 500)])
def test_fp32_within_1e5(key, M, P):
    w, pts, q, params = _case(key, M, P)
    model = S.Model(w.program, params)
    r = model.query_min(pts, q, w.margin, precision="fp32", per_point=True)
    omin, oarg, ofree, opp = _oracle(w.program, params, pts, q, w.margin)
    err = np.abs(r.per_point.astype(np.float64) - opp).max()
    assert err <= 1e-5, err
    assert np.array_equal(r.per_point, opp)  # the FP32 path runs in the oracle's order
    # the fused min/argmin equal the min/argmin of the kernel's own per-point output
    assert np.array_equal(r.min, r.per_point.min(axis=1))
    assert np.array_equal(r.argmin, r.per_point.argmin(axis=1))
    amb = np.abs(omin.astype(np.float64) - w.margin) <= 1e-5
    assert np.array_equal(r.free[~amb], ofree[~amb])


@pytest.mark.parametrize("key,M,P", [("c2", 4, 3000), ("c3", 3, 1500), ("c4", 3, 1300)])
def test_bf16_within_bound(key, M, P):
    w, pts, q, params = _case(key, M, P)
    model = S.Model(w.program, params)
    r = model.query_min(pts, q, w.margin, precision="bf16", per_point=True)
    omin, oarg, ofree, opp = _oracle(w.program, params, pts, q, w.margin)
    bound = BF16_BOUND[w.program.name]
    err = np.abs(r.per_point.astype(np.float64) - opp).max()
    print(f"{key}: bf16 max|err| = {err:.3e} (bound {bound})")
    assert err <= bound, err
    assert np.array_equal(r.min, r.per_point.min(axis=1))
    assert np.array_equal(r.argmin, r.per_point.argmin(axis=1))
    amb = np.abs(omin.astype(np.float64) - w.margin) <= bound
    assert np.array_equal(r.free[~amb], ofree[~amb])
    # argmin parity: same index, or the oracle's delta there is within the bound of the min
    d_at = opp[np.arange(M), r.argmin]
    assert np.all((r.argmin == oarg) | (d_at - omin <= bound))


@pytest.mark.parametrize("prec", ["fp32_exact", "fp32", "fp32_split", "bf16"])
def test_fig2_reference_network(prec):
    prog = S.fig2(3, 256, 6)
    params = S.init_params(prog, 11, "ref")
    pts, q = WORKLOADS["c2"].make(seed=5, motions=3, points=700)
    model = S.Model(prog, params)
    r = model.query_min(pts, q, 0.0, precision=prec, per_point=True)
    _, _, _, opp = _oracle(prog, params, pts, q, 0.0)
    err = np.abs(r.per_point.astype(np.float64) - opp).max()
    tol = {"fp32_exact": 0.0, "fp32": 0.0, "fp32_split": FP32_SPLIT_BOUND["fig2_3x256"],
           "bf16": BF16_BOUND["fig2_3x256"]}[prec]
    assert err <= tol, err


def test_forward_eval_mixed_motions_matches_oracle():
    w = WORKLOADS["c2"]
    params = S.init_params(w.program, 2, "he")
    pts, q = w.make(seed=9, motions=5, points=300)
    rng = np.random.default_rng(0)
    seg = np.sort(rng.integers(0, 5, size=pts.shape[0]))  # runs of equal q of varying length
    raw = np.concatenate([pts, q[seg]], axis=1).astype(np.float32)
    model = S.Model(w.program, params)
    out = model.forward_eval(raw, precision="fp32_exact")
    ref = O.forward_eval(w.program, params, raw)
    assert np.array_equal(out, ref)
    out16 = model.forward_eval(raw, precision="bf16")
    assert np.abs(out16 - ref).max() <= BF16_BOUND[w.program.name]


@pytest.mark.parametrize("key,prog_name", [("c3", None), ("c4", None), ("c3", "fig2_5x512")])
@pytest.mark.parametrize("B", [1, 1000, 3001])
def test_forward_eval_rows_of_distinct_motions(key, prog_name, B):
    """forward_eval batches whose rows all differ in motion (eval_mae, bench.cpp:80-90; training
    validation, nn.cpp:370).  The FP32 path runs them as full tiles (each row reads its own q) and
    stays bit-identical; bf16 at width 512 runs 128-row tiles with the q-part per row on the
    tensor core (FusedArgs::mixed) within the network's bound, and agrees with the folded path
    on the same rows grouped by motion."""
    w = WORKLOADS[key]
    prog = S.fig2(5, 512, 6) if prog_name else w.program
    params = S.init_params(prog, 6, "ref" if prog_name else w.bound)
    pts, q = w.make(seed=6, motions=64, points=4096)
    rng = np.random.default_rng(B)
    qi = rng.integers(0, 64, B)
    raw = np.concatenate([pts[rng.integers(0, pts.shape[0], B)],
                          q[qi] + rng.uniform(-0.05, 0.05, (B, q.shape[1])).astype(np.float32)], axis=1).astype(np.float32)
    model = S.Model(prog, params)
    ref = O.forward_eval(prog, params, raw)
    assert np.array_equal(model.forward_eval(raw, precision="fp32_exact"), ref)
    out = model.forward_eval(raw, precision="bf16")
    bound = BF16_BOUND[prog.name]
    assert np.abs(out.astype(np.float64) - ref).max() <= bound
    if B > 1:  # the same rows sorted by motion with a shared q per group: the folded segment path
        g = np.argsort(qi, kind="stable")
        grouped = raw[g].copy()
        grouped[:, 3:] = q[qi[g]]
        ref_g = O.forward_eval(prog, params, grouped)
        assert np.abs(model.forward_eval(grouped, precision="bf16").astype(np.float64) - ref_g).max() <= bound


def test_predict_min_distance_reference_signature():
    w = WORKLOADS["c1"]
    params = S.init_params(w.program, 4, "he")
    pts, q = w.make(seed=1)
    model = S.Model(w.program, params)
    cloud = pts.astype(np.float64)
    q0, q1 = q[0, :6].astype(np.float64), q[0, 6:].astype(np.float64)
    got = model.predict_min_distance(cloud, q0, q1, precision="fp32_exact")
    ref = O.predict_min_distance(w.program, params, cloud, q0, q1)
    assert got == ref
    # single point == forward of that row; duplicated cloud == same min
    one = model.predict_min_distance(cloud[:1], q0, q1, precision="fp32_exact")
    row = O.forward_eval(w.program, params, np.concatenate([pts[:1], q[:1]], axis=1))
    assert one == (float(row[0]), 0)
    dup = model.predict_min_distance(np.concatenate([cloud, cloud]), q0, q1, precision="fp32_exact")
    assert dup == got


def test_reference_errors():
    w = WORKLOADS["c1"]
    model = S.Model(w.program, S.init_params(w.program, 4, "he"))
    with pytest.raises(ValueError, match="predict_min_distance: empty point cloud"):
        model.predict_min_distance(np.zeros((0, 3)), np.zeros(6), np.zeros(6))
    with pytest.raises(ValueError, match="predict_min_distance: motion dof does not match model"):
        model.predict_min_distance(np.zeros((4, 3)), np.zeros(5), np.zeros(5))
    with pytest.raises(ValueError, match="forward: input width mismatch"):
        model.forward_eval(np.zeros((4, 14), np.float32))


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
def test_point_sharded_keys_equal_unsharded(prec):
    """K2 path on one GPU: shard the points, fold keys per shard, min-combine, finalise."""
    import torch
    w = WORKLOADS["c3"]
    params = S.init_params(w.program, 6, "he")
    pts, q = w.make(seed=8, motions=2, points=5000)
    model = S.Model(w.program, params)
    full = model.query_min(pts, q, w.margin, precision=prec)
    dev = torch.device("cuda:0")
    tq = torch.from_numpy(q).to(dev)
    keys = torch.empty(2, dtype=torch.int64, device=dev)
    S.keys_init_device(keys)
    bounds = [0, 1234, 3100, 5000]
    for a, b in zip(bounds[:-1], bounds[1:]):
        model.query_keys_device(torch.from_numpy(pts[a:b]).to(dev), a, tq, keys, precision=prec)
    mn = torch.empty(2, dtype=torch.float32, device=dev)
    am = torch.empty(2, dtype=torch.int32, device=dev)
    fr = torch.empty(2, dtype=torch.uint8, device=dev)
    S.keys_finalize_device(keys, w.margin, mn, am, fr)
    torch.cuda.synchronize()
    assert np.array_equal(mn.cpu().numpy(), full.min)
    assert np.array_equal(am.cpu().numpy(), full.argmin)
    assert np.array_equal(fr.cpu().numpy().astype(bool), full.free)


def test_batch_invariance_bf16():
    """SPEC.md:415 row independence: results do not depend on batching."""
    w = WORKLOADS["c3"]
    params = S.init_params(w.program, 6, "he")
    pts, q = w.make(seed=8, motions=3, points=1000)
    model = S.Model(w.program, params)
    allm = model.query_min(pts, q, w.margin, precision="bf16", per_point=True)
    for m in range(3):
        one = model.query_min(pts, q[m:m + 1], w.margin, precision="bf16", per_point=True)
        assert np.array_equal(one.per_point[0], allm.per_point[m])


def test_checkpoint_round_trip(tmp_path):
    """predictions identical after an SVCKPT01 round trip (nn.cpp:499-576)."""
    import struct
    prog = S.fig2(3, 256, 6)
    params = S.init_params(prog, 21, "ref")
    path = tmp_path / "m.ckpt"
    with open(path, "wb") as f:
        f.write(b"SVCKPT01")
        f.write(struct.pack("<4I", 1, 3, 256, 15))
        f.write(params.astype("<f4").tobytes())
    m1 = S.Model(prog, params)
    m2 = S.Model.from_checkpoint(str(path))
    pts, q = WORKLOADS["c2"].make(seed=2, motions=2, points=500)
    for prec in ("fp32_exact", "bf16"):
        a = m1.query_min(pts, q, 0.0, precision=prec, per_point=True)
        b = m2.query_min(pts, q, 0.0, precision=prec, per_point=True)
        assert np.array_equal(a.per_point, b.per_point)


@pytest.mark.parametrize("key", ["c3", "c4"])
def test_classification_with_calibrated_output_bias(key):
    """with seeded weights almost every c3/c4 motion is in collision, so the
    margin test is shifted onto the data by setting b_o so the median per-motion oracle min
    equals the margin; classification must then be exact outside the ambiguous band."""
    w = WORKLOADS[key]
    params = S.init_params(w.program, 31, w.bound)
    pts, q = w.make(seed=31, motions=48, points=600)
    omin, _, _, _ = _oracle(w.program, params, pts, q, w.margin)
    params = params.copy()
    params[-1] += np.float32(w.margin - np.median(omin.astype(np.float64)))
    omin, oarg, ofree, opp = _oracle(w.program, params, pts, q, w.margin)
    assert 0.2 < ofree.mean() < 0.8
    for prec in ("bf16", "fp32"):
        r = S.Model(w.program, params).query_min(pts, q, w.margin, precision=prec)
        bound = BF16_BOUND[w.program.name] if prec == "bf16" else 1e-5
        amb = np.abs(omin.astype(np.float64) - w.margin) <= bound
        assert np.array_equal(r.free[~amb], ofree[~amb]), (prec, int(amb.sum()))
        print(f"{key} {prec}: free {r.free.mean():.2f}, ambiguous {int(amb.sum())}/48")


@pytest.mark.parametrize("key,M,P,seed", [("c1", 1, 4096, 3), ("c2", 8, 3000, 3), ("c2", 16, 4096, 2024),
                                          ("c3", 4, 3000, 8), ("c4", 3, 2500, 8), ("c3", 1, 129, 9)])
def test_fp32_split_within_stated_bound(key, M, P, seed):
    """fp32_split (split-fp16 on tcgen05; width 256: 128 rows per CTA, width 512: 64 rows per
    CTA on M=128 pair MMAs): within the frozen bound of the network (1e-5 at width 256), and
    the fused min/argmin equal those of its own per-point output."""
    w, pts, q, params = _case(key, M, P, seed)
    r = S.Model(w.program, params).query_min(pts, q, w.margin, precision="fp32_split", per_point=True)
    omin, oarg, ofree, opp = _oracle(w.program, params, pts, q, w.margin)
    bound = FP32_SPLIT_BOUND[w.program.name]
    err = np.abs(r.per_point.astype(np.float64) - opp).max()
    print(f"{key} seed {seed}: fp32_split max|err| = {err:.3e} (bound {bound})")
    assert err <= bound, err
    assert np.array_equal(r.min, r.per_point.min(axis=1))
    assert np.array_equal(r.argmin, r.per_point.argmin(axis=1))
    amb = np.abs(omin.astype(np.float64) - w.margin) <= bound
    assert np.array_equal(r.free[~amb], ofree[~amb])


def test_fp32_split_width_512_forward_eval_mixed_motions():
    """forward_eval rows of mixed motions (the a-8 path, tile table of 128-row tiles) on the
    width-512 split kernel: within the bound, and batch-invariant (rows evaluated alone give
    the same bits); a batch of mostly distinct motions runs on the FP32 path (exact)."""
    w = WORKLOADS["c3"]
    params = S.init_params(w.program, 4, w.bound)
    pts, q = w.make(seed=4, motions=5, points=300)
    idx = np.sort(np.arange(300) % 5)  # five runs of 60 rows: the folded tile-table path
    rows = np.concatenate([pts, q[idx]], axis=1).astype(np.float32)
    m = S.Model(w.program, params)
    out = m.forward_eval(rows, precision="fp32_split")
    ref = O.forward_eval(w.program, params, rows)
    assert np.abs(out.astype(np.float64) - ref).max() <= FP32_SPLIT_BOUND[w.program.name]
    assert np.array_equal(m.forward_eval(rows[60:120], precision="fp32_split"), out[60:120])  # one run alone
    mixed = np.concatenate([pts, q[np.arange(300) % 5]], axis=1).astype(np.float32)
    assert np.array_equal(m.forward_eval(mixed, precision="fp32_split"), O.forward_eval(w.program, params, mixed))


@pytest.mark.parametrize("width,blocks", [(256, 3), (512, 5)])
@pytest.mark.parametrize("neg", [None, 2])
def test_fig2_bf16_affine_fold_with_trained_like_bn(width, blocks, neg):
    """The bf16 kernels fold each block's BN affine into its weights and carry the shifts as an
    offset (abi_model.cu fold_affine_bf16).  With non-trivial BN statistics — and a layer with
    negative gamma columns, which is kept unfolded — the result stays within the network's
    frozen bf16 bound of the oracle."""
    from fig2_bn import randomize_bn
    prog = S.fig2(blocks, width, 6)
    params = randomize_bn(prog, S.init_params(prog, 7, "ref"), 7, negative_gamma_layer=neg)
    pts, q = WORKLOADS["c2"].make(seed=7, motions=4, points=1500)
    r = S.Model(prog, params).query_min(pts, q, 0.0, precision="bf16", per_point=True)
    _, _, _, opp = _oracle(prog, params, pts, q, 0.0)
    err = np.abs(r.per_point.astype(np.float64) - opp).max()
    assert err <= BF16_BOUND[prog.name], err
    assert np.array_equal(r.min, r.per_point.min(axis=1))


def test_trained_like_checkpoint_through_the_loader(tmp_path):
    """A Fig. 2 checkpoint with non-trivial BN statistics (as training leaves them) through
    svn_model_load_checkpoint: FP32 path bit-identical to the oracle, bf16 (affine folded) within
    the frozen bound, and both identical to the model built from the same parameters in memory."""
    import struct
    from fig2_bn import randomize_bn
    prog = S.fig2(5, 512, 6)
    params = randomize_bn(prog, S.init_params(prog, 33, "ref"), 33, negative_gamma_layer=3)
    path = tmp_path / "trained.ckpt"
    with open(path, "wb") as f:
        f.write(b"SVCKPT01")
        f.write(struct.pack("<4I", 1, 5, 512, 15))
        f.write(params.astype("<f4").tobytes())
    loaded, direct = S.Model.from_checkpoint(str(path)), S.Model(prog, params)
    pts, q = WORKLOADS["c2"].make(seed=33, motions=3, points=900)
    _, _, _, opp = _oracle(prog, params, pts, q, 0.0)
    for prec, tol in (("fp32", 0.0), ("bf16", BF16_BOUND["fig2_5x512"])):
        a = loaded.query_min(pts, q, 0.0, precision=prec, per_point=True)
        b = direct.query_min(pts, q, 0.0, precision=prec, per_point=True)
        assert np.array_equal(a.per_point, b.per_point)
        assert np.abs(a.per_point.astype(np.float64) - opp).max() <= tol

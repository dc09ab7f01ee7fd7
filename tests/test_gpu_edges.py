"""GPU edge cases: ragged tiles, tiny inputs, NaN inputs, heavy motion mixing, concurrent
host callers (run_box_world calls predict_min_distance from parallel_for workers,
bench.cpp:156,193), and the device entry points."""
import threading

import numpy as np
import pytest

import paper_2402_15281_b200 as S
from oracle import oracle as O
from paper_2402_15281_b200.workloads import WORKLOADS
from test_gpu_parity import BF16_BOUND, FP32_SPLIT_BOUND

pytestmark = pytest.mark.gpu

TOL = {"fp32_exact": 0.0, "fp32": 1e-5}


def _tol(prec, prog):
    if prec == "fp32_split":
        return FP32_SPLIT_BOUND[prog.name]
    return TOL.get(prec, BF16_BOUND.get(prog.name, 0.1))


@pytest.mark.parametrize("prec", ["bf16", "fp32", "fp32_exact", "fp32_split"])
@pytest.mark.parametrize("P", [1, 2, 127, 129, 255, 257, 511, 1000])
def test_ragged_point_counts(prec, P):
    w = WORKLOADS["c3"] if prec == "bf16" else WORKLOADS["c2"]
    params = S.init_params(w.program, 17, w.bound)
    pts, q = w.make(seed=17, motions=3, points=P)
    r = S.Model(w.program, params).query_min(pts, q, w.margin, precision=prec, per_point=True)
    omin, oarg, ofree, opp = O.query_min(w.program, params, pts, q, w.margin, per_point=True, threads=8)
    tol = _tol(prec, w.program)
    assert np.abs(r.per_point.astype(np.float64) - opp).max() <= tol
    assert np.array_equal(r.min, r.per_point.min(axis=1))
    assert np.array_equal(r.argmin, r.per_point.argmin(axis=1))
    if prec == "fp32_exact":
        assert np.array_equal(r.argmin, oarg) and np.array_equal(r.free, ofree)


@pytest.mark.parametrize("prec", ["bf16", "fp32_split"])
@pytest.mark.parametrize("motions,P", [(3, 1000), (1, 257), (227, 256), (149, 300), (75, 512)])
def test_tile_counts_around_the_pair_count(prec, motions, P):
    # width 256: bf16 runs two tiles in flight per CTA pair (odd tile counts leave slot 1 idle
    # in the last round), fp32 the split kernel; tile counts below, at and above 74 pairs
    w = WORKLOADS["c2"]
    params = S.init_params(w.program, 23, w.bound)
    pts, q = w.make(seed=23, motions=motions, points=P)
    r = S.Model(w.program, params).query_min(pts, q, w.margin, precision=prec, per_point=True)
    omin, oarg, ofree, opp = O.query_min(w.program, params, pts, q, w.margin, per_point=True, threads=8)
    assert np.abs(r.per_point.astype(np.float64) - opp).max() <= _tol(prec, w.program)
    assert np.array_equal(r.min, r.per_point.min(axis=1))
    assert np.array_equal(r.argmin, r.per_point.argmin(axis=1))
    r2 = S.Model(w.program, params).query_min(pts, q, w.margin, precision=prec)
    assert np.array_equal(r2.min, r.min) and np.array_equal(r2.argmin, r.argmin)


@pytest.mark.parametrize("prec", ["bf16", "fp32_exact"])
def test_many_motions_few_points(prec):
    w = WORKLOADS["c2"]
    params = S.init_params(w.program, 3, w.bound)
    pts, q = w.make(seed=3, motions=700, points=5)
    r = S.Model(w.program, params).query_min(pts, q, w.margin, precision=prec, per_point=True)
    omin, oarg, ofree, opp = O.query_min(w.program, params, pts, q, w.margin, per_point=True, threads=8)
    assert np.abs(r.per_point.astype(np.float64) - opp).max() <= _tol(prec, w.program)
    assert np.array_equal(r.argmin, r.per_point.argmin(axis=1))


def test_fp32_split_fp16_overflow_is_reported_not_dropped():
    """fp32_split holds activations as fp16 (hi, lo') planes: a row whose activation reaches
    the fp16 infinity (|h| >= 65520) cannot be represented.  It must not silently drop out of
    the min as a NaN (that could turn a colliding motion "free"); it is reported as
    delta = -inf, so its motion's min is -inf and the class is "not free" (handed to the exact
    checker).  Rows that stay in range keep their bound."""
    w = WORKLOADS["c2"]
    params = S.init_params(w.program, 29, w.bound)
    pts, q = w.make(seed=29, motions=3, points=600)
    big = pts.copy()
    big[5] = (3.0e6, -2.0e6, 1.0e6)  # layer-0 pre-activations ~1e5-1e6: beyond fp16
    m = S.Model(w.program, params)
    r = m.query_min(big, q, w.margin, precision="fp32_split", per_point=True)
    assert np.all(r.per_point[:, 5] == -np.inf)
    assert np.all(r.min == -np.inf) and np.all(r.argmin == 5) and not r.free.any()
    o = O.query_min(w.program, params, big, q, w.margin, per_point=True, threads=8)[3]
    assert np.all(np.isfinite(o[:, 5]))  # the reference's fp32 path stays finite there
    ok = np.delete(np.arange(600), 5)
    assert np.abs(r.per_point[:, ok].astype(np.float64) - o[:, ok]).max() <= _tol("fp32_split", w.program)


@pytest.mark.parametrize("prec", ["bf16", "fp32", "fp32_exact"])
def test_nan_point_at_index_zero_sticks(prec):
    """nn.cpp:476-478: a NaN prediction at row 0 is returned; NaN elsewhere is skipped.
    The Fig. 2 network propagates NaN (its input layer has no ReLU and blocks are residual)."""
    prog = S.fig2(2, 256, 6)
    params = S.init_params(prog, 5, "ref")
    pts, q = WORKLOADS["c2"].make(seed=5, motions=2, points=300)
    bad = pts.copy()
    bad[7] = np.nan
    m = S.Model(prog, params)
    r = m.query_min(bad, q, 0.0, precision=prec, per_point=True)
    assert np.all(np.isnan(r.per_point[:, 7]))
    ok = np.delete(np.arange(300), 7)
    assert np.array_equal(r.argmin, ok[np.argmin(r.per_point[:, ok], axis=1)])
    bad[0] = np.nan
    r = m.query_min(bad, q, 0.0, precision=prec)
    assert np.all(np.isnan(r.min)) and np.all(r.argmin == 0) and not r.free.any()
    o = O.query_min(prog, params, bad, q, 0.0)
    assert np.all(np.isnan(o[0])) and np.all(o[1] == 0)


@pytest.mark.parametrize("prec", ["bf16", "fp32_exact"])
def test_forward_eval_every_row_its_own_motion(prec):
    w = WORKLOADS["c3"]
    params = S.init_params(w.program, 8, w.bound)
    pts, q = w.make(seed=8, motions=300, points=300)
    raw = np.concatenate([pts, q], axis=1).astype(np.float32)  # row i uses motion i
    out = S.Model(w.program, params).forward_eval(raw, precision=prec)
    ref = O.forward_eval(w.program, params, raw)
    assert np.abs(out.astype(np.float64) - ref).max() <= _tol(prec, w.program)


def test_concurrent_host_callers_share_one_model():
    w = WORKLOADS["c1"]
    params = S.init_params(w.program, 9, w.bound)
    model = S.Model(w.program, params)
    pts, q = w.make(seed=9, motions=8, points=500)
    ref = [O.predict_min_distance(w.program, params, pts.astype(np.float64), q[m, :6], q[m, 6:]) for m in range(8)]
    out = [None] * 8
    errs = []

    def work(m):
        try:
            for _ in range(3):
                out[m] = model.predict_min_distance(pts.astype(np.float64), q[m, :6], q[m, 6:],
                                                    precision="fp32_exact")
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=work, args=(m,)) for m in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs
    assert out == ref


def test_device_entry_points_with_torch_stream():
    import torch
    w = WORKLOADS["c3"]
    params = S.init_params(w.program, 10, w.bound)
    pts, q = w.make(seed=10, motions=5, points=3000)
    model = S.Model(w.program, params)
    host = model.query_min(pts, q, w.margin, precision="bf16", per_point=True)
    dev = torch.device("cuda:0")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        tp, tq = torch.from_numpy(pts).to(dev), torch.from_numpy(q).to(dev)
        mn = torch.empty(5, dtype=torch.float32, device=dev)
        am = torch.empty(5, dtype=torch.int32, device=dev)
        fr = torch.empty(5, dtype=torch.uint8, device=dev)
        pp = torch.empty((5, 3000), dtype=torch.float32, device=dev)
        model.query_min_device(tp, tq, w.margin, mn, am, fr, pp, precision="bf16", stream=st)
    st.synchronize()
    assert np.array_equal(mn.cpu().numpy(), host.min)
    assert np.array_equal(am.cpu().numpy(), host.argmin)
    assert np.array_equal(pp.cpu().numpy(), host.per_point)


def test_batched_proxy_matches_per_motion_calls():
    w = WORKLOADS["c2"]
    params = S.init_params(w.program, 12, w.bound)
    model = S.Model(w.program, params)
    pts, q = w.make(seed=12, motions=6, points=800)
    proxy = S.batched_proxy(model, pts, q, precision="fp32_exact")
    for m in range(6):
        mn, _ = model.predict_min_distance(pts.astype(np.float64), q[m, :6], q[m, 6:], precision="fp32_exact")
        assert proxy(m) == mn


def _fma(a, b, c):
    from fractions import Fraction
    return float(Fraction(a) * Fraction(b) + Fraction(c))


@pytest.mark.parametrize("prec", ["fp32_exact", "bf16"])
def test_eval_grid_matches_reference_reconstruction(prec):
    """cmd_reconstruct NN branch (cli.cpp:240-261): voxel centres in (ix, iy, iz) order."""
    w = WORKLOADS["c3"] if prec == "bf16" else WORKLOADS["c2"]
    params = S.init_params(w.program, 13, w.bound)
    model = S.Model(w.program, params)
    origin, vs, dims = np.array([-0.31, -0.47, 0.05]), 0.0371, (9, 11, 13)
    q0 = np.linspace(-1.0, 1.0, 6)
    q1 = np.linspace(0.5, -0.7, 6)
    grid = model.eval_grid(origin, vs, dims, q0, q1, precision=prec)
    cen = np.array([[_fma(vs, float(i), origin[0]), _fma(vs, float(j), origin[1]), _fma(vs, float(k), origin[2])]
                    for i in range(dims[0]) for j in range(dims[1]) for k in range(dims[2])], np.float64)
    raw = np.concatenate([cen.astype(np.float32), np.repeat(np.concatenate([q0, q1])[None], len(cen), 0)],
                         axis=1).astype(np.float32)
    ref = O.forward_eval(w.program, params, raw).reshape(dims)
    if prec == "fp32_exact":
        assert np.array_equal(grid, ref)
    else:
        assert np.abs(grid.astype(np.float64) - ref).max() <= BF16_BOUND[w.program.name]


def test_motion_chunking_matches_single_launch():
    """Queries beyond the per-launch motion limit (int32 TMA rows) run as motion chunks; the
    limit is lowered through the test hook in a subprocess so the chunked path is exercised."""
    import subprocess
    import sys
    code = r'''
import numpy as np, sys
sys.path.insert(0, "{root}")
import paper_2402_15281_b200 as S
from paper_2402_15281_b200.workloads import WORKLOADS
out = []
for key, prec in (("c3", "bf16"), ("c2", "bf16"), ("c2", "fp32_split"), ("c2", "fp32")):
    w = WORKLOADS[key]
    p = S.init_params(w.program, 5, w.bound)
    pts, q = w.make(seed=5, motions=23, points=700)
    r = S.Model(w.program, p).query_min(pts, q, w.margin, precision=prec, per_point=True)
    out.append(np.concatenate([r.min, r.argmin.astype(np.float32), r.free.astype(np.float32), r.per_point.ravel()]))
np.save(sys.argv[1], np.concatenate(out))
'''
    from pathlib import Path
    import tempfile
    import os
    root = str(Path(__file__).resolve().parents[1])
    d = tempfile.mkdtemp()
    res = []
    for i, env_max in enumerate(("", "5")):
        env = dict(os.environ)
        if env_max:
            env["SVN_MAX_MOTIONS_PER_LAUNCH"] = env_max
        f = os.path.join(d, f"r{i}.npy")
        subprocess.run([sys.executable, "-c", code.replace("{root}", root), f], check=True, env=env)
        res.append(np.load(f))
    assert np.array_equal(res[0], res[1])


def test_forward_eval_row_chunking_matches_single_launch():
    """forward_eval with every row its own motion, run as row chunks through the test hook."""
    import os
    import subprocess
    import sys
    import tempfile
    from pathlib import Path
    code = r'''
import numpy as np, sys
sys.path.insert(0, "{root}")
import paper_2402_15281_b200 as S
from paper_2402_15281_b200.workloads import WORKLOADS
w = WORKLOADS["c2"]
p = S.init_params(w.program, 9, w.bound)
pts, q = w.make(seed=9, motions=300, points=1)
raw = np.concatenate([np.repeat(pts, 300, 0), q], 1).astype(np.float32)
m = S.Model(w.program, p)
np.save(sys.argv[1], np.concatenate([m.forward_eval(raw, precision=pr) for pr in ("bf16", "fp32", "fp32_split")]))
'''
    root = str(Path(__file__).resolve().parents[1])
    d = tempfile.mkdtemp()
    res = []
    for i, env_max in enumerate(("", "37")):
        env = dict(os.environ)
        if env_max:
            env["SVN_MAX_MOTIONS_PER_LAUNCH"] = env_max
        f = os.path.join(d, f"r{i}.npy")
        subprocess.run([sys.executable, "-c", code.replace("{root}", root), f], check=True, env=env)
        res.append(np.load(f))
    assert np.array_equal(res[0], res[1])


def test_many_short_lived_host_threads():
    """Each host thread gets its own stream and staging buffers; they are released when the
    thread exits, so threads that come and go (a parallel_for pool) do not accumulate them."""
    import torch
    w = WORKLOADS["c2"]
    params = S.init_params(w.program, 4, w.bound)
    model = S.Model(w.program, params)
    pts, q = w.make(seed=4, motions=1, points=3000)
    ref = model.query_min(pts, q, w.margin, precision="bf16")
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(40):
        out = []
        t = threading.Thread(target=lambda: out.append(model.query_min(pts, q, w.margin, precision="bf16")))
        t.start()
        t.join()
        assert np.array_equal(out[0].min, ref.min)
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < 64 << 20  # no per-thread growth


@pytest.mark.parametrize("prog", [S.plain(3, 128, 6), S.fig2(2, 128, 7), S.deepsdf(6, 128, 6, 3)],
                         ids=lambda p: p.name)
@pytest.mark.parametrize("M,P", [(1, 300), (5, 2000)])
def test_width_128_fp32_bit_identical(prog, M, P):
    """Width 128 (FP32 path only: 4-column FFMA2 pairs per thread) against the oracle, both
    tile sizes (32-row tiles when there are few, 128-row otherwise)."""
    params = S.init_params(prog, 29, "he")
    pts, q = WORKLOADS["c2"].make(seed=29, motions=M, points=P)
    if prog.dof == 7:
        q = np.concatenate([q[:, :6], q[:, :1], q[:, 6:], q[:, 6:7]], axis=1)
    r = S.Model(prog, params).query_min(pts, q, 0.02, precision="fp32_exact", per_point=True)
    omin, oarg, ofree, opp = O.query_min(prog, params, pts, q, 0.02, per_point=True, threads=8)
    assert np.array_equal(r.per_point, opp)
    assert np.array_equal(r.min, omin) and np.array_equal(r.argmin, oarg) and np.array_equal(r.free, ofree)
    with pytest.raises(S.SvnError):
        S.Model(prog, params).query_min(pts, q, 0.02, precision="bf16")


@pytest.mark.parametrize("prec", ["bf16", "fp32_exact", "fp32_split"])
def test_small_calls_read_each_calls_inputs(prec):
    """Host-buffer calls stage through a per-thread pinned block (abi_query.cu, query_min_host):
    every call must use its own points and motions, also with a second model (possibly at a
    freed model's address)."""
    w = WORKLOADS["c2"]
    for mseed in (41, 42):
        params = S.init_params(w.program, mseed, w.bound)
        m = S.Model(w.program, params)
        for seed in (1, 2, 3, 1):
            pts, q = w.make(seed=seed, motions=3, points=2999)
            r = m.query_min(pts, q, w.margin, precision=prec)  # no per-point output
            omin, oarg, ofree, opp = O.query_min(w.program, params, pts, q, w.margin, per_point=True, threads=8)
            tol = _tol(prec, w.program)
            assert np.abs(r.min.astype(np.float64) - omin).max() <= tol
            if prec == "fp32_exact":
                assert np.array_equal(r.min, omin) and np.array_equal(r.argmin, oarg)
                assert np.array_equal(r.free, ofree)
            cloud = pts[:1000].astype(np.float64)
            got = m.predict_min_distance(cloud, q[0, :6], q[0, 6:], precision=prec)
            ref = O.predict_min_distance(w.program, params, cloud, q[0, :6].astype(np.float64),
                                         q[0, 6:].astype(np.float64))
            if prec == "fp32_exact":
                assert got == ref
            else:
                assert abs(got[0] - ref[0]) <= tol
        del m


@pytest.mark.parametrize("prec", ["bf16", "fp32"])
def test_large_cloud_host_call_is_pipelined_and_bit_identical(prec):
    """A cloud of >= 2^21 points given as host float arrays travels in 2^20-point chunks on a second
    stream while the chunks already on the device are folded into the per-motion keys
    (query_min_host); the result equals one launch over the device-resident cloud bit for bit,
    for pageable and for pinned host arrays, including a ragged last chunk."""
    import torch
    w = WORKLOADS["c2"]
    params = S.init_params(w.program, 12, w.bound)
    P = (1 << 21) + 12345
    pts, q = w.make(seed=12, motions=3, points=P)
    model = S.Model(w.program, params)
    dev = torch.device("cuda:0")
    tp, tq = torch.from_numpy(pts).to(dev), torch.from_numpy(q).to(dev)
    mn = torch.empty(3, dtype=torch.float32, device=dev)
    am = torch.empty(3, dtype=torch.int32, device=dev)
    fr = torch.empty(3, dtype=torch.uint8, device=dev)
    model.query_min_device(tp, tq, w.margin, mn, am, fr, None, precision=prec)
    torch.cuda.synchronize()
    for hp, hq in ((pts, q), (torch.from_numpy(pts).pin_memory().numpy(), torch.from_numpy(q).pin_memory().numpy())):
        for _ in range(2):  # the second call reuses the staging block and the grown scratch arena
            r = model.query_min(hp, hq, w.margin, precision=prec)
            assert np.array_equal(r.min, mn.cpu().numpy()) and np.array_equal(r.argmin, am.cpu().numpy())
            assert np.array_equal(r.free, fr.cpu().numpy().astype(bool))
    # the reference's own entry point (double cloud, one motion): its conversion runs chunk by chunk too
    dof = w.program.dof
    d, i = model.predict_min_distance(pts.astype(np.float64), q[1, :dof].astype(np.float64),
                                      q[1, dof:].astype(np.float64), precision=prec)
    assert d == float(mn[1].item()) and i == int(am[1].item())

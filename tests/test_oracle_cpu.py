"""CPU tests: pin the oracle (oracle/sweptnet_oracle.c) before trusting it.

Pins: the C++ standard's mt19937_64 known answer; a std::mt19937_64 stream dump
(tests/golden/mt19937_64_std.txt, from oracle/pin_rng.cpp); SPEC.md known-answer
properties of nn; the independent torch fp64
oracle; and the committed golden fixtures.
"""
import hashlib
from pathlib import Path

import numpy as np
import pytest

import paper_2402_15281_b200 as S
from oracle import oracle as O, torch_fp64 as T

GOLDEN = Path(__file__).resolve().parent / "golden"


def test_mt19937_64_known_answer():
    # C++ standard [rand.predef]: the 10000th invocation of a default-constructed
    # mt19937_64 (seed 5489) produces 9981545732273789042.
    assert O.lib().oracle_mt64_nth(5489, 10000) == 9981545732273789042


def test_rng_stream_matches_std_library_dump():
    rows = [l.split() for l in (GOLDEN / "mt19937_64_std.txt").read_text().splitlines() if not l.startswith("#")]
    import ctypes as C
    b = 1.0 / np.sqrt(15.0)
    for seed in (5489, 1, 42):
        ref = [r for r in rows if int(r[0]) == seed]
        u64 = np.empty(len(ref), np.uint64)
        O.lib().oracle_mt64_stream(seed, len(ref), C.c_void_p(u64.ctypes.data))
        assert [int(r[1]) for r in ref] == [int(x) for x in u64]
        uni = np.empty(len(ref), np.float64)
        O.lib().oracle_uniform_stream(seed, len(ref), -b, b, C.c_void_p(uni.ctypes.data))
        assert np.array_equal(uni, np.array([float(r[2]) for r in ref]))
        assert np.array_equal(uni.astype(np.float32), np.array([float(r[3]) for r in ref], np.float32))


def test_substream_seed_matches_python_restatement():
    from paper_2402_15281_b200.workloads import substream_seed
    for base, idx in [(0, 0), (1, 5), (2**63 + 7, 123456)]:
        assert O.lib().oracle_substream_seed(base, idx) == substream_seed(base, idx)


@pytest.mark.parametrize("prog,bound", [(S.fig2(5, 512, 6), "ref"), (S.plain(4, 256, 6), "he"),
                                        (S.deepsdf(8, 512, 6, 4), "he"), (S.plain(6, 512, 7), "he"),
                                        (S.fig2(2, 8, 2), "ref")])
def test_product_init_equals_oracle_init(prog, bound):
    a = O.init_params(prog, 1234, bound)
    b = S.init_params(prog, 1234, bound)
    assert np.array_equal(a, b)
    assert np.array_equal(S.init_params(prog, 1234, bound), b)  # same seed -> bit-identical
    assert not np.array_equal(S.init_params(prog, 1235, bound), b)


def test_param_count_spec_example():
    # SPEC.md:351 / nn.cpp:19-24: param_count(init(5, 512, 6)) = 1,365,505
    prog = S.fig2(5, 512, 6)
    assert prog.trainable_params() == 1365505
    assert O.trainable_params(prog) == 1365505


def test_init_bn_and_bias_values():
    prog = S.fig2(2, 16, 3)
    p = S.init_params(prog, 3, "ref")
    N, inn = 16, 9
    o = 2 * inn
    assert np.all(p[:inn] == 0) and np.all(p[inn:2 * inn] == 1)
    o += N * inn
    assert np.all(p[o:o + N] == 0)  # input bias
    o += N
    for _ in range(2):
        K = N + inn
        W = p[o:o + N * K]
        assert np.abs(W).max() <= 1 / np.sqrt(K)
        o += N * K
        b, g, beta, mu, var = (p[o + i * N:o + (i + 1) * N] for i in range(5))
        assert np.all(b == 0) and np.all(g == 1) and np.all(beta == 0) and np.all(mu == 0) and np.all(var == 1)
        o += 5 * N


@pytest.mark.parametrize("prog,bound", [(S.fig2(3, 64, 6), "ref"), (S.plain(4, 64, 6), "he"),
                                        (S.deepsdf(6, 64, 7, 3), "he")])
def test_oracle_matches_torch_fp64(prog, bound):
    params = O.init_params(prog, 9, bound)
    rng = np.random.default_rng(1)
    raw = np.concatenate([rng.random((50, 3)), rng.uniform(-3, 3, (50, 2 * prog.dof))], axis=1)
    d64 = O.forward_eval(prog, params.astype(np.float64), raw, np.float64)
    t64 = T.forward(prog, params, raw)
    assert np.abs(d64 - t64).max() < 1e-12
    d32 = O.forward_eval(prog, params, raw)
    assert np.abs(d32 - t64).max() < 1e-5


def test_zero_weight_model_gives_output_bias():
    # SPEC.md:360
    prog = S.fig2(2, 32, 6)
    p = np.zeros(prog.param_floats(), np.float32)
    p[prog.input_dim:2 * prog.input_dim] = 1.0
    p[-1] = 0.375
    # affine layers need var=1, gamma=1 for a well-defined fold; zero gamma makes BN output beta=0
    raw = np.random.default_rng(0).random((7, prog.input_dim)).astype(np.float32)
    assert np.all(O.forward_eval(prog, p, raw) == np.float32(0.375))


def test_forward_row_independence():
    # eval forward of a batch == per-row forward, exactly
    prog = S.deepsdf(8, 128, 6, 4)
    params = O.init_params(prog, 5, "he")
    raw = np.random.default_rng(2).uniform(-1, 1, (40, prog.input_dim)).astype(np.float32)
    full = O.forward_eval(prog, params, raw)
    rows = np.array([O.forward_eval(prog, params, raw[i:i + 1])[0] for i in range(40)])
    assert np.array_equal(full, rows)
    perm = np.random.default_rng(3).permutation(40)
    assert np.array_equal(O.forward_eval(prog, params, raw[perm]), full[perm])


def test_predict_min_distance_spec_examples():
    prog = S.plain(4, 64, 6)
    params = O.init_params(prog, 5, "he")
    rng = np.random.default_rng(4)
    cloud = rng.random((200, 3))
    q0, q1 = rng.uniform(-2, 2, 6), rng.uniform(-2, 2, 6)
    mn, am = O.predict_min_distance(prog, params, cloud, q0, q1)
    raw = np.concatenate([cloud, np.repeat(np.concatenate([q0, q1])[None], 200, 0)], axis=1).astype(np.float32)
    one_by_one = np.array([O.forward_eval(prog, params, raw[i:i + 1])[0] for i in range(200)])
    assert mn == float(one_by_one.min()) and am == int(one_by_one.argmin())
    assert O.predict_min_distance(prog, params, cloud[am:am + 1], q0, q1) == (float(one_by_one[am]), 0)
    dup = O.predict_min_distance(prog, params, np.concatenate([cloud, cloud]), q0, q1)
    assert dup == (mn, am)  # duplicated cloud: same min, lowest index
    with pytest.raises(ValueError, match="empty point cloud"):
        O.predict_min_distance(prog, params, np.zeros((0, 3)), q0, q1)
    with pytest.raises(ValueError, match="motion dof does not match model"):
        O.predict_min_distance(prog, params, cloud, q0[:5], q1[:5])


def test_nan_semantics_of_argmin():
    # nn.cpp:476-478: best starts at 0, strict '<': NaN at index 0 sticks, NaN elsewhere is skipped
    prog = S.fig2(1, 16, 2)
    params = O.init_params(prog, 1, "ref")
    pts = np.random.default_rng(0).random((20, 3)).astype(np.float32)
    q = np.zeros((1, 4), np.float32)
    base = O.query_min(prog, params, pts, q, 0.0, per_point=True)
    p2 = pts.copy()
    p2[5] = np.nan
    mn, am, _, pp = O.query_min(prog, params, p2, q, 0.0, per_point=True)
    assert np.isnan(pp[0, 5])
    ok = np.delete(np.arange(20), 5)
    assert am[0] == ok[np.argmin(pp[0, ok])]
    p2[0] = np.nan
    mn, am, fr, _ = O.query_min(prog, params, p2, q, 0.0, per_point=True)
    assert np.isnan(mn[0]) and am[0] == 0 and not fr[0]
    assert base[1][0] == np.argmin(base[3][0])


def test_query_min_thread_invariance():
    prog = S.plain(4, 64, 6)
    params = O.init_params(prog, 8, "he")
    rng = np.random.default_rng(6)
    pts = rng.random((301, 3)).astype(np.float32)
    q = rng.uniform(-2, 2, (3, 12)).astype(np.float32)
    r1 = O.query_min(prog, params, pts, q, 0.1, per_point=True, threads=1)
    r8 = O.query_min(prog, params, pts, q, 0.1, per_point=True, threads=8)
    for a, b in zip(r1, r8):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("name", ["c1_full", "c2_sub", "c3_sub", "c4_sub", "fig2_5x512_sub", "fig2_3x256_sub"])
def test_golden_fixture(name):
    g = np.load(GOLDEN / f"{name}.npz")
    from paper_2402_15281_b200.program import Layer, LayerProgram
    fl = g["flags"].reshape(-1, 4)
    prog = LayerProgram(str(g["program"]), int(g["width"]), int(g["dof"]),
                        tuple(Layer(*map(bool, f)) for f in fl))
    params = O.init_params(prog, int(g["seed"]), str(g["bound"]))
    assert hashlib.sha256(params.tobytes()).hexdigest() == str(g["params_sha256"])
    assert np.array_equal(S.init_params(prog, int(g["seed"]), str(g["bound"])), params)
    mn, am, fr, pp = O.query_min(prog, params, g["points"], g["q01"], float(g["margin"]), per_point=True, threads=4)
    assert np.array_equal(pp, g["delta_f32"])
    assert np.array_equal(mn, g["min"]) and np.array_equal(am, g["argmin"]) and np.array_equal(fr, g["free"])
    assert np.abs(pp.astype(np.float64) - g["delta_f64"]).max() < 1e-5
    if pp.shape[0] <= 2:
        t = T.query(prog, params, g["points"], g["q01"])
        assert np.abs(t - g["delta_f64"]).max() < 1e-12

"""The C oracle against the reference's OWN code (CPU).

tests/golden/ref_fig2.npz holds outputs of /root/reference/proj/src/nn.cpp compiled
unmodified (oracle/ref/Makefile -> oracle/_ref/libref_nn.so, tests/golden/make_ref_golden.py)
on trained-like Fig. 2 networks: the reference's make_normalizer (or a random non-identity
normaliser), nonzero biases, BN statistics with negative gammas.  The oracle must reproduce
them bit for bit — init_model, forward_eval<float> and <double>, predict_min_distance — and
the product's checkpoint loader must raise the reference's error kinds and texts.  When the
reference build is present (this container; or carried to the GPU box in oracle/_ref) the
same comparison also runs live on fresh inputs.
"""
import hashlib
import tempfile
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from oracle import ref_oracle as R
from paper_2402_15281_b200.program import fig2
from paper_2402_15281_b200.workloads import limits_default

import ref_golden as G

Z, NAMES = G.load()


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


@pytest.mark.parametrize("name", NAMES)
def test_oracle_init_matches_reference_init_model(name):
    g, prog, init, _ = G.params(Z, name)
    assert hashlib.sha256(init.tobytes()).hexdigest() == str(g["init_sha256"])
    assert prog.trainable_params() == int(g["param_count"])


@pytest.mark.parametrize("name", NAMES)
def test_oracle_forward_eval_bit_identical_to_reference(name):
    g, prog, init, p = G.params(Z, name)
    raw = g["raw"]
    assert np.array_equal(bits(O.forward_eval(prog, p, raw)), bits(g["forward_eval_f32"]))
    assert np.array_equal(bits(O.forward_eval(prog, p, raw.astype(np.float64), dtype=np.float64)),
                          bits(g["forward_eval_f64"]))
    assert np.array_equal(bits(O.forward_eval(prog, init, raw)), bits(g["forward_eval_f32_init"]))
    # the ISA-dependent order of nn.cpp:127 (Eigen packet reductions): stated bound
    assert np.abs(g["forward_eval_f32_packet8"] - g["forward_eval_f32"]).max() <= G.DOT_ORDER_BOUND
    # the fixture exercises a non-identity normaliser and nonzero biases
    assert np.any(g["pert_shift"] != 0) and np.any(g["pert_scale"] != 1) and np.any(g["pert_b0"] != 0)


@pytest.mark.parametrize("name", NAMES)
def test_oracle_predict_min_distance_matches_reference(name):
    g, prog, _, p = G.params(Z, name)
    mn, idx = O.predict_min_distance(prog, p, g["cloud"], g["q0"], g["q1"])
    assert (mn, idx) == (float(g["pmd"][0]), int(g["pmd"][1]))


def test_mknorm_fixture_is_make_normalizer():
    """make_normalizer (nn.cpp:314-338) restated: x shift = mean of the split, scale 1/reach;
    joints mid / 2/(hi-lo) (default_robot limits, robot.cpp:91-92,122).  The fixture's
    values come from the reference; this pins our reading of them."""
    from paper_2402_15281_b200.workloads import _rng, bin_cloud
    for name in NAMES:
        g, nb, N, dof, seed = G.case(Z, name)
        if str(g["norm"]) != "mknorm":
            continue
        x = bin_cloud(_rng(seed, 7), 4096).astype(np.float32).astype(np.float64)
        lengths = {2: [0.55, 0.45], 6: [0.20, 0.25, 0.20, 0.15, 0.12, 0.08]}[dof]
        reach = float(np.sum(lengths))
        lim = limits_default(dof)
        exp_shift = np.concatenate([np.float32(x.mean(axis=0)), np.float32(0.0 * lim), np.float32(0.0 * lim)])
        exp_scale = np.concatenate([np.full(3, np.float32(1.0 / reach)), np.float32(2.0 / (2 * lim)),
                                    np.float32(2.0 / (2 * lim))])
        assert np.allclose(g["pert_shift"], exp_shift, atol=1e-7), name
        assert np.array_equal(g["pert_scale"], exp_scale.astype(np.float32)), name


def test_checkpoint_errors_match_reference_texts(tmp_path):
    """The product loader (svn_model_load_checkpoint) raises the reference's error kinds with
    the reference's texts (nn.cpp:524-576), as recorded from the reference build."""
    import paper_2402_15281_b200 as S
    from paper_2402_15281_b200 import abi
    kinds = {"IoError": abi.IoError, "FormatError": abi.FormatError, "TruncationError": abi.TruncationError,
             "VersionError": abi.VersionError}
    prog = fig2(1, 64, 2)
    good = O.init_params(prog, 1, "ref")
    for key, kind, text in Z["load_errors"]:
        path = tmp_path / f"{key}.ckpt"
        if key == "short_header":
            path.write_bytes(b"SVCKPT01" + b"\1\0\0\0\1\0")
        elif key != "missing":
            body, arch, ver, magic, extra = good, (1, 64, 7), 1, b"SVCKPT01", b""
            if key == "bad_magic":
                magic = b"SVCKPT02"
            elif key == "version":
                ver = 2
            elif key == "truncated":
                body = good[:-100]
            elif key == "trailing":
                extra = b"\0\0\0\0"
            elif key == "header_only":
                body = good[:0]
            elif key == "bad_arch":
                arch = (0, 64, 7)
            R.write_checkpoint(path, *arch, body, version=ver, magic=magic, extra=extra)
        with pytest.raises(kinds[str(kind)]) as e:
            S.Model.from_checkpoint(str(path))
        assert str(text).replace("{path}", str(path)) in str(e.value), (key, str(e.value))


needs_ref = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
@pytest.mark.parametrize("nb,N,dof,seed", [(1, 32, 3, 101), (2, 256, 6, 102), (4, 128, 7, 103)])
def test_live_reference_vs_oracle_fresh_inputs(nb, N, dof, seed, tmp_path):
    """Live: the reference build and the oracle on fresh random trained-like nets and inputs."""
    prog = fig2(nb, N, dof)
    ck = tmp_path / "m.ckpt"
    init = R.init_model(nb, N, dof, seed, ck)
    assert np.array_equal(bits(init), bits(O.init_params(prog, seed, "ref")))
    rng = np.random.default_rng(seed)
    p = init.copy()
    in_ = 3 + 2 * dof
    off = G.layout(nb, N, in_)
    p[:in_] = rng.uniform(-1, 1, in_)
    p[in_:2 * in_] = rng.uniform(0.3, 3, in_)
    for i in range(1, nb + 1):
        p[off[f"b{i}"]:off[f"b{i}"] + N] = rng.uniform(-0.3, 0.3, N)
        p[off[f"gamma{i}"]:off[f"gamma{i}"] + N] = rng.uniform(-1.5, 1.5, N)
        p[off[f"beta{i}"]:off[f"beta{i}"] + N] = rng.uniform(-0.3, 0.3, N)
        p[off[f"mean{i}"]:off[f"mean{i}"] + N] = rng.uniform(-0.3, 0.3, N)
        p[off[f"var{i}"]:off[f"var{i}"] + N] = rng.uniform(0.1, 3, N)
    R.write_checkpoint(ck, nb, N, in_, p)
    raw = rng.uniform(-2, 2, (300, in_)).astype(np.float32)
    assert np.array_equal(bits(R.forward_eval(ck, raw)), bits(O.forward_eval(prog, p, raw)))
    r64 = R.forward_eval_f64(ck, raw.astype(np.float64))
    assert np.array_equal(bits(r64), bits(O.forward_eval(prog, p, raw.astype(np.float64), dtype=np.float64)))
    cloud = rng.uniform(-1, 1, (500, 3))
    q0, q1 = rng.uniform(-2, 2, dof), rng.uniform(-2, 2, dof)
    assert R.predict_min_distance(ck, cloud, q0, q1) == O.predict_min_distance(prog, p, cloud, q0, q1)


@needs_ref
def test_live_reference_rng_stream():
    """Rng::uniform (rng.hpp:21-23) as compiled in the reference header == the oracle's stream."""
    a = R.uniform_stream(5489, 1000, -0.25, 0.75)
    b = np.empty(1000)
    O.lib().oracle_uniform_stream(5489, 1000, -0.25, 0.75, b.ctypes.data)
    assert np.array_equal(bits(a), bits(b))


@needs_ref
def test_live_reference_errors():
    """predict_min_distance / forward_eval argument errors: the reference's own texts."""
    with tempfile.TemporaryDirectory() as d:
        ck = Path(d) / "m.ckpt"
        R.init_model(1, 16, 2, 1, ck)
        with pytest.raises(R.RefError, match="predict_min_distance: empty point cloud"):
            R.predict_min_distance(ck, np.zeros((0, 3)), np.zeros(2), np.zeros(2))
        with pytest.raises(R.RefError, match="predict_min_distance: motion dof does not match model"):
            R.predict_min_distance(ck, np.zeros((1, 3)), np.zeros(3), np.zeros(3))
        with pytest.raises(R.RefError, match="forward: input width mismatch"):
            R.forward_eval(ck, np.zeros((2, 6), np.float32))

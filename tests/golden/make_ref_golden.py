"""Golden vectors from the reference's OWN inference code (TEST INFRASTRUCTURE).

Runs oracle/_ref/libref_nn.so — /root/reference/proj/src/nn.cpp (+ robot.cpp, geometry.cpp)
compiled unmodified against oracle/ref/eigen_subset by oracle/ref/Makefile — and writes
tests/golden/ref_fig2.npz.  Needs /root/reference (this container only); the GPU box and the
CPU suite read the committed .npz.

Per case (a Fig. 2 network, the only architecture the reference implements, nn.hpp:11-15):
  - init_model<float>(n_blocks, N, dof, seed) (nn.cpp:57-93): sha256 of its parameter body;
  - a trained-like parameter set on top of it: the input normaliser from the reference's
    make_normalizer (nn.cpp:314-338) for default_robot(dof) on a seeded training split
    ("mknorm" cases) or a random non-identity shift/scale ("randnorm"), and random nonzero
    biases, BN gamma (some negative) / beta / running mean / running var and output bias;
  - raw rows [B x in] mixing 4 motions -> forward_eval<float> and forward_eval<double>
    (nn.cpp:95-130, 587-588) through load_checkpoint (nn.cpp:524-576);
  - one double cloud + motion -> predict_min_distance (nn.cpp:460-480);
  - the same forward_eval with Eigen's reductions in 8-lane packet order (libref_nn_packet8.so)
    to state how far the ISA-dependent dot order at nn.cpp:127 moves the result.
Plus the reference's load_checkpoint error kinds and texts for malformed files.

    python tests/golden/make_ref_golden.py
"""
from __future__ import annotations

import hashlib
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref_oracle as R  # noqa: E402
from paper_2402_15281_b200.workloads import bin_cloud, limits_default, _rng  # noqa: E402

CASES = [  # (name, n_blocks, N, dof, seed, normaliser)
    ("fig2_3x256_mknorm", 3, 256, 6, 11, "mknorm"),
    ("fig2_5x512_mknorm", 5, 512, 6, 12, "mknorm"),
    ("fig2_5x512_dof7_randnorm", 5, 512, 7, 13, "randnorm"),
    ("fig2_2x128_randnorm", 2, 128, 6, 14, "randnorm"),
    ("fig2_1x64_dof2_mknorm", 1, 64, 2, 15, "mknorm"),
]
B_ROWS = 256
P_CLOUD = 2000


def layout(nb, N, in_):
    """Offsets of the SVCKPT01 body (nn.cpp:507-520)."""
    off = {"shift": 0, "scale": in_}
    o = 2 * in_
    off["W0"], o = o, o + N * in_
    off["b0"], o = o, o + N
    for i in range(nb):
        off[f"W{i + 1}"], o = o, o + N * (N + in_)
        for k in ("b", "gamma", "beta", "mean", "var"):
            off[f"{k}{i + 1}"], o = o, o + N
    off["wo"], o = o, o + N
    off["bo"], o = o, o + 1
    off["total"] = o
    return off


def perturb(params, nb, N, dof, seed, norm):
    """Trained-like parameters: returns (params, dict of the perturbation vectors)."""
    in_ = 3 + 2 * dof
    rng = np.random.default_rng(1000 + seed)
    off = layout(nb, N, in_)
    assert off["total"] == params.size
    p = params.copy()
    if norm == "mknorm":
        train_x = bin_cloud(_rng(seed, 7), 4096).astype(np.float32)
        shift, scale = R.make_normalizer(dof, train_x)
    else:
        shift = rng.uniform(-0.5, 0.5, in_).astype(np.float32)
        scale = rng.uniform(0.5, 2.0, in_).astype(np.float32)
    pert = {"shift": shift, "scale": scale}
    p[off["shift"]:off["shift"] + in_] = shift
    p[off["scale"]:off["scale"] + in_] = scale
    pert["b0"] = rng.uniform(-0.1, 0.1, N).astype(np.float32)
    p[off["b0"]:off["b0"] + N] = pert["b0"]
    for i in range(1, nb + 1):
        g = rng.uniform(0.5, 1.5, N)
        g[rng.random(N) < 0.1] *= -1.0  # some negative gammas (a trained BN can flip sign)
        vals = {"b": rng.uniform(-0.1, 0.1, N), "gamma": g, "beta": rng.uniform(-0.2, 0.2, N),
                "mean": rng.uniform(-0.2, 0.2, N), "var": rng.uniform(0.5, 2.0, N)}
        for k, v in vals.items():
            pert[f"{k}{i}"] = v.astype(np.float32)
            p[off[f"{k}{i}"]:off[f"{k}{i}"] + N] = pert[f"{k}{i}"]
    pert["bo"] = np.array([rng.uniform(-0.1, 0.1)], np.float32)
    p[off["bo"]] = pert["bo"][0]
    return p, pert


def raw_rows(seed, dof, B):
    """B rows [x, q0, q1] over 4 motions (rows of different motions interleaved)."""
    rng = _rng(seed, 8)
    pts = bin_cloud(rng, B).astype(np.float32)
    lim = np.concatenate([limits_default(dof)] * 2) if dof <= 7 else np.full(2 * dof, np.pi)
    q = (-lim + 2 * lim * rng.random((4, 2 * dof))).astype(np.float32)
    which = rng.integers(0, 4, B)
    return np.concatenate([pts, q[which]], axis=1).astype(np.float32), which


def main():
    R.build()
    out = {}
    tmp = Path(tempfile.mkdtemp(prefix="svn_refgold_"))
    for name, nb, N, dof, seed, norm in CASES:
        in_ = 3 + 2 * dof
        ck = tmp / f"{name}_init.ckpt"
        init = R.init_model(nb, N, dof, seed, ck)
        p, pert = perturb(init, nb, N, dof, seed, norm)
        ck2 = tmp / f"{name}.ckpt"
        R.write_checkpoint(ck2, nb, N, in_, p)
        raw, which = raw_rows(seed, dof, B_ROWS)
        y32 = R.forward_eval(ck2, raw)
        y64 = R.forward_eval_f64(ck2, raw.astype(np.float64))
        y_pk8 = R.forward_eval(ck2, raw, "_packet8")
        y_init = R.forward_eval(ck, raw)  # the seeded model as init_model leaves it
        crng = _rng(seed, 9)
        cloud = bin_cloud(crng, P_CLOUD)  # double, as PointCloud carries it (collision.hpp:11-13)
        q0, q1 = raw[0, 3:3 + dof].astype(np.float64), raw[0, 3 + dof:].astype(np.float64)
        mn, idx = R.predict_min_distance(ck2, cloud, q0, q1)
        pre = f"{name}/"
        out[pre + "spec"] = np.array([nb, N, dof, seed], np.int64)
        out[pre + "norm"] = np.array(norm)
        out[pre + "init_sha256"] = np.array(hashlib.sha256(init.tobytes()).hexdigest())
        out[pre + "param_count"] = np.array(R.param_count(nb, N, dof), np.int64)
        for k, v in pert.items():
            out[pre + "pert_" + k] = v
        out[pre + "raw"] = raw
        out[pre + "motion_of_row"] = which.astype(np.int32)
        out[pre + "forward_eval_f32"] = y32
        out[pre + "forward_eval_f64"] = y64
        out[pre + "forward_eval_f32_packet8"] = y_pk8
        out[pre + "forward_eval_f32_init"] = y_init
        out[pre + "cloud"] = cloud
        out[pre + "q0"], out[pre + "q1"] = q0, q1
        out[pre + "pmd"] = np.array([mn, float(idx)])
        print(f"{name}: |y| max {np.abs(y32).max():.3f}, packet8 vs scalar max {np.abs(y_pk8 - y32).max():.3g}, "
              f"pmd ({mn:.6f}, {idx})")
    # load_checkpoint error kinds / texts (nn.cpp:524-576) for malformed files
    nb, N, dof = 1, 64, 2
    good = R.init_model(nb, N, dof, 1, tmp / "good.ckpt")
    bad = {
        "missing": None,
        "bad_magic": dict(magic=b"SVCKPT02"),
        "version": dict(version=2),
        "truncated": dict(trunc=100),
        "trailing": dict(extra=b"\0\0\0\0"),
        "header_only": dict(trunc=len(good)),
        "bad_arch": dict(arch=(0, N, 3 + 2 * dof)),
        "short_header": "raw",
    }
    errs = []
    for key, how in bad.items():
        path = tmp / f"{key}.ckpt"
        if how == "raw":
            path.write_bytes(b"SVCKPT01" + b"\1\0\0\0\1\0")
        elif how is not None:
            arch = how.get("arch", (nb, N, 3 + 2 * dof))
            body = good[: good.size - how.get("trunc", 0)] if how.get("trunc", 0) < good.size else good[:0]
            R.write_checkpoint(path, *arch, body, version=how.get("version", 1), magic=how.get("magic", b"SVCKPT01"),
                               extra=how.get("extra", b""))
        try:
            R.load_checkpoint_header(path)
            errs.append((key, "ok", ""))
        except R.RefError as e:
            errs.append((key, e.kind_name, e.msg.replace(str(path), "{path}")))
    out["load_errors"] = np.array(errs)
    dst = Path(__file__).resolve().parent / "ref_fig2.npz"
    np.savez_compressed(dst, **out)
    print("wrote", dst, dst.stat().st_size, "bytes;", errs)


if __name__ == "__main__":
    main()

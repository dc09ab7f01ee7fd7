"""The reference with the B200 drop-in applied, run on the GPU through the
reference's own API, against the golden vectors of the UNPATCHED reference.

oracle/_ref/ref_dropin_driver (built in the build container by oracle/ref/Makefile `dropin`
from the patched reference sources + integration/nn_b200.cpp + libsweptnet_b200.so) calls
forward_eval<float>, forward<float>(Eval), forward_eval<double> and predict_min_distance on
trained-like Fig. 2 checkpoints.  The float results come from the CUDA FP32 path and must be
bit-identical to the unpatched reference's CPU results; the double path stays on the CPU body
and must be too; concurrent callers get the same answer; argument errors keep the reference's
exception type and text.
"""
import subprocess
from pathlib import Path

import numpy as np
import pytest

import ref_golden as G

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
EXE = ROOT / "oracle" / "_ref" / "ref_dropin_driver"
Z, NAMES = G.load()


@pytest.mark.skipif(not EXE.exists(), reason="oracle/_ref/ref_dropin_driver not built (needs /root/reference)")
@pytest.mark.parametrize("name", [n for n in NAMES if int(G.case(Z, n)[2]) in (128, 256, 512)])
def test_reference_api_with_dropin_matches_unpatched_reference(name, tmp_path):
    g, prog, _, p = G.params(Z, name)
    ck = tmp_path / "m.ckpt"
    G.write_checkpoint(ck, prog, p)
    raw = np.ascontiguousarray(g["raw"], np.float32)
    cloud = np.ascontiguousarray(g["cloud"], np.float64)
    q01 = np.concatenate([g["q0"], g["q1"]]).astype(np.float64)
    (tmp_path / "raw.f32").write_bytes(raw.tobytes())
    (tmp_path / "cloud.f64").write_bytes(cloud.tobytes())
    (tmp_path / "q.f64").write_bytes(q01.tobytes())
    threads = 4
    out = subprocess.run([str(EXE), str(ck), str(tmp_path / "raw.f32"), str(raw.shape[0]), str(tmp_path / "cloud.f64"),
                          str(cloud.shape[0]), str(tmp_path / "q.f64"), str(tmp_path / "out.bin"), str(threads)],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    B = raw.shape[0]
    b = (tmp_path / "out.bin").read_bytes()
    y = np.frombuffer(b, np.float32, B, 0)
    y2 = np.frombuffer(b, np.float32, B, 4 * B)
    y64 = np.frombuffer(b, np.float64, B, 8 * B)
    ref = g["forward_eval_f32"]
    assert np.array_equal(y.view(np.uint32), ref.view(np.uint32)), np.abs(y - ref).max()
    assert np.array_equal(y2.view(np.uint32), ref.view(np.uint32))
    assert np.array_equal(y64.view(np.uint64), g["forward_eval_f64"].view(np.uint64))
    off = 16 * B
    for k in range(1 + threads):
        mn = np.frombuffer(b, np.float64, 1, off)[0]
        idx = int(np.frombuffer(b, np.int32, 1, off + 8)[0])
        off += 12
        assert (mn, idx) == (float(g["pmd"][0]), int(g["pmd"][1])), k
    lines = out.stdout
    assert "empty_cloud: invalid_argument: predict_min_distance: empty point cloud" in lines
    assert "dof_mismatch: invalid_argument: predict_min_distance: motion dof does not match model" in lines
    assert "width_mismatch: invalid_argument: forward: input width mismatch" in lines


@pytest.mark.skipif(not EXE.exists(), reason="oracle/_ref/ref_dropin_driver not built (needs /root/reference)")
@pytest.mark.parametrize("prec", ["fp32_split", "bf16", "fp16"])
@pytest.mark.parametrize("name", [n for n in NAMES if int(G.case(Z, n)[2]) in (256, 512)])
def test_dropin_tensor_core_precisions_within_bounds(prec, name, tmp_path):
    """SWEPTNET_B200_PRECISION selects the drop-in's arithmetic (integration/nn_b200.cpp): the
    reference API then runs fp32_split or bf16 on the tensor cores, within those paths' frozen
    bounds of the unpatched reference's results; forward_eval<double> stays bit-identical."""
    import json
    import os
    g, prog, _, p = G.params(Z, name)
    key = f"fig2_{prog.n_layers - 1}x{prog.width}"
    f = ROOT / "tests" / "golden" / f"{prec}_bounds.json"
    bound = json.loads(f.read_text())[key]["bound"]
    ck = tmp_path / "m.ckpt"
    G.write_checkpoint(ck, prog, p)
    raw = np.ascontiguousarray(g["raw"], np.float32)
    cloud = np.ascontiguousarray(g["cloud"], np.float64)
    q01 = np.concatenate([g["q0"], g["q1"]]).astype(np.float64)
    (tmp_path / "raw.f32").write_bytes(raw.tobytes())
    (tmp_path / "cloud.f64").write_bytes(cloud.tobytes())
    (tmp_path / "q.f64").write_bytes(q01.tobytes())
    env = dict(os.environ, SWEPTNET_B200_PRECISION=prec)
    out = subprocess.run([str(EXE), str(ck), str(tmp_path / "raw.f32"), str(raw.shape[0]), str(tmp_path / "cloud.f64"),
                          str(cloud.shape[0]), str(tmp_path / "q.f64"), str(tmp_path / "out.bin"), "2"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stdout + out.stderr
    B = raw.shape[0]
    b = (tmp_path / "out.bin").read_bytes()
    y = np.frombuffer(b, np.float32, B, 0)
    y64 = np.frombuffer(b, np.float64, B, 8 * B)
    err = np.abs(y.astype(np.float64) - g["forward_eval_f32"]).max()
    print(f"{name} {prec}: forward_eval max|err| {err:.3e} (bound {bound})")
    assert err <= bound
    assert np.array_equal(y64.view(np.uint64), g["forward_eval_f64"].view(np.uint64))
    mn = np.frombuffer(b, np.float64, 1, 16 * B)[0]
    assert abs(mn - float(g["pmd"][0])) <= bound

"""CPU tests of the C-ABI library and host logic (no compute calls without a GPU)."""
import ctypes as C
import re
import struct
from pathlib import Path

import numpy as np
import pytest

import paper_2402_15281_b200 as S
from paper_2402_15281_b200 import abi
from paper_2402_15281_b200.workloads import WORKLOADS

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "sweptnet_b200.h").read_text()
    return sorted(set(re.findall(r"SVN_API[^;(]*?\b(svn_[a-z0-9_]+)\s*\(", text, flags=re.S)))


def test_library_exports_every_declared_symbol():
    lib = abi.lib()
    names = declared_symbols()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(abi.EXPORTED)


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(abi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(abi.LIB_PATH)], capture_output=True, text=True).stdout
    # tcgen05.mma -> UTCHMMA, bulk async copy (TMA engine) -> UBLKCP, tcgen05.ld -> LDTM
    for mnemonic in ("UTCHMMA", "UBLKCP", "LDTM"):
        assert mnemonic in sass, mnemonic


def test_param_counts_via_abi():
    for prog in (S.fig2(5, 512, 6), S.plain(4, 256, 6), S.deepsdf(8, 512, 6, 4), S.plain(6, 512, 7)):
        desc, keep = abi.make_desc(prog)
        assert abi.lib().svn_param_count(C.byref(desc)) == prog.param_floats()
        assert abi.lib().svn_trainable_param_count(C.byref(desc)) == prog.trainable_params()
    assert S.fig2(5, 512, 6).trainable_params() == 1365505


def test_flops_per_query_matches_survey():
    # SURVEY.md §8d table
    assert WORKLOADS["c1"].program.flops_per_query() == 395264
    assert WORKLOADS["c3"].program.flops_per_query() == 3677184
    assert WORKLOADS["c4"].program.flops_per_query() == 2625536


def test_invalid_descriptor_reports_error():
    bad = S.LayerProgram("bad", 256, 0, (S.Layer(True, True),))
    desc, keep = abi.make_desc(bad)
    h = C.c_void_p()
    p = np.zeros(16, np.float32)
    st = abi.lib().svn_model_create(C.byref(desc), abi.ptr(p), 16, 0, C.byref(h))
    assert st == abi.INVALID_ARGUMENT
    assert "dof" in abi.lib().svn_last_error().decode()
    with pytest.raises(ValueError, match="parameter count mismatch"):
        S.Model(S.plain(4, 256, 6), np.zeros(10, np.float32))


def _write_ckpt(path, n_blocks, N, dof, params, version=1, magic=b"SVCKPT01", extra=b""):
    with open(path, "wb") as f:
        f.write(magic)
        f.write(struct.pack("<4I", version, n_blocks, N, 3 + 2 * dof))
        f.write(params.astype("<f4").tobytes())
        f.write(extra)


def test_checkpoint_errors_match_reference(tmp_path):
    # nn.cpp:524-576 error taxonomy (errors.hpp:8-27), raised before any device work
    prog = S.fig2(2, 16, 3)
    params = S.init_params(prog, 1, "ref")
    with pytest.raises(abi.IoError, match="cannot open checkpoint"):
        S.Model.from_checkpoint(str(tmp_path / "missing.ckpt"))
    p = tmp_path / "badmagic.ckpt"
    _write_ckpt(p, 2, 16, 3, params, magic=b"NOTACKPT")
    with pytest.raises(abi.FormatError, match="not a sweptnet checkpoint"):
        S.Model.from_checkpoint(str(p))
    p = tmp_path / "ver.ckpt"
    _write_ckpt(p, 2, 16, 3, params, version=2)
    with pytest.raises(abi.VersionError, match="version 2 not supported"):
        S.Model.from_checkpoint(str(p))
    p = tmp_path / "trunc.ckpt"
    _write_ckpt(p, 2, 16, 3, params[:-5])
    with pytest.raises(abi.TruncationError, match="ends inside tensor data"):
        S.Model.from_checkpoint(str(p))
    p = tmp_path / "trail.ckpt"
    _write_ckpt(p, 2, 16, 3, params, extra=b"\0")
    with pytest.raises(abi.FormatError, match="trailing bytes"):
        S.Model.from_checkpoint(str(p))
    p = tmp_path / "hdr.ckpt"
    _write_ckpt(p, 0, 16, 3, params)
    with pytest.raises(abi.FormatError, match="implausible architecture header"):
        S.Model.from_checkpoint(str(p))


def test_workloads_shapes_and_shard_slices():
    for key, w in WORKLOADS.items():
        pts, q = w.make(seed=1, motions=4, points=1000)
        assert pts.shape == (1000, 3) and pts.dtype == np.float32
        assert q.shape == (4, 2 * w.program.dof)
        lim = w.q_limits()
        assert np.all(np.abs(q) <= np.concatenate([lim, lim]) + 1e-6)
        pts2, q2 = w.make(seed=1, motions=2, points=1000, motion_offset=2)
        assert np.array_equal(pts, pts2) and np.array_equal(q[2:], q2)
    pts, _ = WORKLOADS["c2"].make(seed=0, motions=1, points=4000)
    assert np.all(pts >= np.array([0, -0.4, 0]) - 1e-6) and np.all(pts <= np.array([1.2, 0.4, 0.5]) + 1e-6)


def test_whole_batch_setting_needs_no_device():
    """svn_set_whole_batch is a thread-local setting (no CUDA call): the context manager sets and
    clears it without a GPU, and nonsense shapes clear it."""
    import paper_2402_15281_b200 as S
    with S.whole_batch(9, 2100) as wb:
        assert wb.shape == (9, 2100)
    S.abi.lib().svn_set_whole_batch(-3, 10)
    S.abi.lib().svn_set_whole_batch(0, 0)

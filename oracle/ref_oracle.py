"""ctypes binding of oracle/_ref/libref_nn.so — the reference's OWN nn.cpp / robot.cpp /
geometry.cpp compiled unmodified against oracle/ref/eigen_subset (recipe: oracle/ref/Makefile).

TEST INFRASTRUCTURE ONLY: the checker of the C restatement (oracle/sweptnet_oracle.c) and of
the CUDA path (tests/, tests/golden/make_ref_golden.py), and the reference's own CPU path timed
by bench.py's CPU legs (--impl reference, cpu_baseline).  Building needs the
reference sources (/root/reference, present in the build container only); the built .so
travels to the GPU box with the repo snapshot, where available() tells the tests whether it
came along.
"""
from __future__ import annotations

import ctypes as C
import struct
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
OUT = HERE / "_ref"
REF = Path("/root/reference/proj")
KINDS = {1: "IoError", 2: "FormatError", 3: "TruncationError", 4: "VersionError", 5: "invalid_argument",
         6: "runtime_error"}

_libs: dict[str, C.CDLL] = {}


class RefError(Exception):
    def __init__(self, kind: int, msg: str):
        super().__init__(f"{KINDS.get(kind, kind)}: {msg}")
        self.kind, self.kind_name, self.msg = kind, KINDS.get(kind, str(kind)), msg


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE / "ref")], check=True)


def available(variant: str = "") -> bool:
    return (OUT / f"libref_nn{variant}.so").exists()


def lib(variant: str = "") -> C.CDLL:
    """variant "" = Eigen scalar reductions; "_packet8" = 8-lane packet-structured reductions."""
    if variant in _libs:
        return _libs[variant]
    p = OUT / f"libref_nn{variant}.so"
    if REF.exists():
        build()  # make is a no-op when up to date
    if not p.exists():
        raise FileNotFoundError(f"{p} not built (needs /root/reference; see oracle/ref/Makefile)")
    L = C.CDLL(str(p))
    VP, L64, I = C.c_void_p, C.c_long, C.c_int
    L.ref_last_error.restype = C.c_char_p
    L.ref_init_save.argtypes = [I, I, I, C.c_uint64, C.c_char_p]
    L.ref_param_count.restype = L64
    L.ref_param_count.argtypes = [I, I, I]
    L.ref_forward_eval.argtypes = [C.c_char_p, VP, L64, L64, VP]
    L.ref_forward_eval_f64.argtypes = [C.c_char_p, VP, L64, L64, VP]
    L.ref_predict_min_distance.argtypes = [C.c_char_p, VP, L64, VP, VP, I, VP, VP]
    if hasattr(L, "ref_time_predict_min_distance"):
        L.ref_time_predict_min_distance.argtypes = [C.c_char_p, VP, L64, VP, L64, I, I, VP, VP, VP]
    L.ref_make_normalizer.argtypes = [I, VP, L64, VP, VP]
    L.ref_load_checkpoint.argtypes = [C.c_char_p, VP, VP, VP]
    L.ref_uniform_stream.argtypes = [C.c_uint64, L64, C.c_double, C.c_double, VP]
    _libs[variant] = L
    return L


def _p(a):
    return C.c_void_p(a.ctypes.data)


def _check(L, rc):
    if rc:
        raise RefError(rc, L.ref_last_error().decode())


def write_checkpoint(path, n_blocks: int, block_dim: int, input_dim: int, params: np.ndarray, version: int = 1,
                     magic: bytes = b"SVCKPT01", extra: bytes = b"") -> None:
    """SVCKPT01 layout (nn.cpp:499-522): magic, u32 {version, n_blocks, block_dim, input_dim}, floats."""
    with open(path, "wb") as f:
        f.write(magic)
        f.write(struct.pack("<4I", version, n_blocks, block_dim, input_dim))
        f.write(np.ascontiguousarray(params, np.float32).tobytes())
        f.write(extra)


def read_checkpoint(path) -> tuple[tuple[int, int, int], np.ndarray]:
    b = Path(path).read_bytes()
    _v, nb, n, ind = struct.unpack("<4I", b[8:24])
    return (nb, n, ind), np.frombuffer(b[24:], np.float32).copy()


def init_model(n_blocks: int, block_dim: int, dof: int, seed: int, path) -> np.ndarray:
    """init_model<float> -> save_checkpoint -> the parameter body (== the Fig. 2 param layout)."""
    L = lib()
    _check(L, L.ref_init_save(n_blocks, block_dim, dof, C.c_uint64(seed), str(path).encode()))
    return read_checkpoint(path)[1]


def param_count(n_blocks: int, block_dim: int, dof: int) -> int:
    return int(lib().ref_param_count(n_blocks, block_dim, dof))


def forward_eval(ckpt, raw: np.ndarray, variant: str = "") -> np.ndarray:
    L = lib(variant)
    raw = np.ascontiguousarray(raw, np.float32)
    out = np.empty(raw.shape[0], np.float32)
    _check(L, L.ref_forward_eval(str(ckpt).encode(), _p(raw), raw.shape[0], raw.shape[1], _p(out)))
    return out


def forward_eval_f64(ckpt, raw: np.ndarray, variant: str = "") -> np.ndarray:
    L = lib(variant)
    raw = np.ascontiguousarray(raw, np.float64)
    out = np.empty(raw.shape[0], np.float64)
    _check(L, L.ref_forward_eval_f64(str(ckpt).encode(), _p(raw), raw.shape[0], raw.shape[1], _p(out)))
    return out


def predict_min_distance(ckpt, cloud, q0, q1, variant: str = "") -> tuple[float, int]:
    L = lib(variant)
    cloud = np.ascontiguousarray(cloud, np.float64).reshape(-1, 3)
    q0 = np.ascontiguousarray(q0, np.float64)
    q1 = np.ascontiguousarray(q1, np.float64)
    mn, idx = np.zeros(1, np.float64), np.zeros(1, np.int32)
    _check(L, L.ref_predict_min_distance(str(ckpt).encode(), _p(cloud), cloud.shape[0], _p(q0), _p(q1), q0.size,
                                         _p(mn), _p(idx)))
    return float(mn[0]), int(idx[0])


def time_predict_min_distance(ckpt, cloud, q01, threads: int, variant: str = ""):
    """M predict_min_distance calls (one per motion, nn.cpp:460-480) from `threads` worker threads,
    the reference's own per-motion pattern (bench.cpp:156,193); returns (min[M], argmin[M], seconds)."""
    L = lib(variant)
    cloud = np.ascontiguousarray(cloud, np.float64).reshape(-1, 3)
    q01 = np.ascontiguousarray(q01, np.float64)
    M, dof = q01.shape[0], q01.shape[1] // 2
    mn, idx, sec = np.zeros(M, np.float64), np.zeros(M, np.int32), np.zeros(1, np.float64)
    _check(L, L.ref_time_predict_min_distance(str(ckpt).encode(), _p(cloud), cloud.shape[0], _p(q01), M, dof,
                                              int(threads), _p(mn), _p(idx), _p(sec)))
    return mn, idx, float(sec[0])


def make_normalizer(dof: int, train_x: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    L = lib()
    x = np.ascontiguousarray(train_x, np.float32).reshape(-1, 3)
    sh, sc = np.empty(3 + 2 * dof, np.float32), np.empty(3 + 2 * dof, np.float32)
    _check(L, L.ref_make_normalizer(dof, _p(x), x.shape[0], _p(sh), _p(sc)))
    return sh, sc


def load_checkpoint_header(ckpt) -> tuple[int, int, int]:
    L = lib()
    a, b, c = (np.zeros(1, np.int32) for _ in range(3))
    _check(L, L.ref_load_checkpoint(str(ckpt).encode(), _p(a), _p(b), _p(c)))
    return int(a[0]), int(b[0]), int(c[0])


def uniform_stream(seed: int, n: int, lo: float, hi: float) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().ref_uniform_stream(C.c_uint64(seed), n, lo, hi, _p(out))
    return out

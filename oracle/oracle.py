"""ctypes binding of the C oracle (oracle/sweptnet_oracle.c).

TEST INFRASTRUCTURE ONLY — the parity checker and the CPU baseline.  Only
tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
may import this.  Parity status: unpinned by reference golden vectors (the
reference needs Eigen, absent here); pinned by the std::mt19937_64 dump, the SPEC
known-answer properties and the independent torch fp64 oracle — see the C header.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
BUILD = HERE / "build"
LIB = BUILD / "liboracle.so"

_lib = None


def build(march: str | None = None, out: Path | None = None) -> Path:
    """make -C oracle; march=native rebuilds the timed baseline like the reference
    (-march=native, proj/CMakeLists.txt:31-38) into a separate directory."""
    env = dict(os.environ)
    args = ["make", "-s", "-C", str(HERE)]
    if march:
        args.append(f"ORACLE_MARCH={march}")
    if out:
        args.append(f"OUT={out}")
    subprocess.run(args, check=True, env=env)
    return (out or BUILD) / "liboracle.so"


def lib(path: Path | None = None) -> C.CDLL:
    global _lib
    if path is None and _lib is not None:
        return _lib
    p = path or LIB
    if not p.exists() or (path is None and (HERE / "sweptnet_oracle.c").stat().st_mtime > p.stat().st_mtime):
        build()
    L = C.CDLL(str(p))
    VP, I64, I32 = C.c_void_p, C.c_int64, C.c_int
    L.oracle_mt64_nth.restype = C.c_uint64
    L.oracle_mt64_nth.argtypes = [C.c_uint64, I64]
    L.oracle_mt64_stream.argtypes = [C.c_uint64, I64, VP]
    L.oracle_uniform_stream.argtypes = [C.c_uint64, I64, C.c_double, C.c_double, VP]
    L.oracle_substream_seed.restype = C.c_uint64
    L.oracle_substream_seed.argtypes = [C.c_uint64, C.c_uint64]
    L.oracle_param_floats.restype = I64
    L.oracle_param_floats.argtypes = [VP, I32, I32, I32]
    L.oracle_trainable_params.restype = I64
    L.oracle_trainable_params.argtypes = [VP, I32, I32, I32]
    L.oracle_init_params.argtypes = [VP, I32, I32, I32, C.c_uint64, I32, VP]
    L.oracle_forward_eval_f32.argtypes = [VP, I32, I32, I32, VP, VP, I64, I64, VP]
    L.oracle_forward_eval_f64.argtypes = [VP, I32, I32, I32, VP, VP, I64, I64, VP]
    L.oracle_predict_min_distance.argtypes = [VP, I32, I32, I32, VP, VP, I64, VP, VP, I32, VP, VP]
    L.oracle_gcc.argtypes = [VP, I32, VP, I32, VP, VP, I64, VP, I64, I32, C.c_double, I32, I32, VP, VP]
    L.oracle_query_min.argtypes = [VP, I32, I32, I32, VP, VP, I64, VP, I64, C.c_double, VP, VP, VP, VP, I32]
    if path is None:
        _lib = L
    return L


def _p(a):
    return C.c_void_p(0) if a is None else C.c_void_p(a.ctypes.data)


def _prog(program):
    flags = np.ascontiguousarray(program.flags_array(), dtype=np.int32)
    return flags, program.n_layers, program.width, program.dof


def param_floats(program) -> int:
    f, L, N, dof = _prog(program)
    return int(lib().oracle_param_floats(_p(f), L, N, dof))


def trainable_params(program) -> int:
    f, L, N, dof = _prog(program)
    return int(lib().oracle_trainable_params(_p(f), L, N, dof))


def init_params(program, seed: int, bound: str = "he") -> np.ndarray:
    f, L, N, dof = _prog(program)
    out = np.empty(param_floats(program), np.float32)
    lib().oracle_init_params(_p(f), L, N, dof, C.c_uint64(seed), 1 if bound == "he" else 0, _p(out))
    return out


def forward_eval(program, params, raw, dtype=np.float32) -> np.ndarray:
    f, L, N, dof = _prog(program)
    raw = np.ascontiguousarray(raw, dtype=dtype)
    params = np.ascontiguousarray(params, dtype=dtype)
    out = np.empty(raw.shape[0], dtype)
    fn = lib().oracle_forward_eval_f32 if dtype == np.float32 else lib().oracle_forward_eval_f64
    rc = fn(_p(f), L, N, dof, _p(params), _p(raw), raw.shape[0], raw.shape[1], _p(out))
    if rc:
        raise ValueError("forward: input width mismatch" if raw.shape[1] != 3 + 2 * dof
                         else "forward: batch must be non-empty")
    return out


def predict_min_distance(program, params, cloud, q0, q1) -> tuple[float, int]:
    f, L, N, dof = _prog(program)
    cloud = np.ascontiguousarray(cloud, np.float64).reshape(-1, 3)
    q0 = np.ascontiguousarray(q0, np.float64)
    q1 = np.ascontiguousarray(q1, np.float64)
    mn = np.zeros(1, np.float64)
    am = np.zeros(1, np.int32)
    rc = lib().oracle_predict_min_distance(_p(f), L, N, dof, _p(np.ascontiguousarray(params, np.float32)),
                                           _p(cloud), cloud.shape[0], _p(q0), _p(q1), q0.size, _p(mn), _p(am))
    if rc == 1:
        raise ValueError("predict_min_distance: empty point cloud")
    if rc == 2:
        raise ValueError("predict_min_distance: motion dof does not match model")
    return float(mn[0]), int(am[0])


def query_min(program, params, points, q01, margin, per_point=False, threads=1, library=None):
    """Every (point x motion) pair: per-motion (min, argmin, free) [+ per-point delta]."""
    f, L, N, dof = _prog(program)
    pts = np.ascontiguousarray(points, np.float32).reshape(-1, 3)
    q = np.ascontiguousarray(q01, np.float32).reshape(-1, 2 * dof)
    P, M = pts.shape[0], q.shape[0]
    mn = np.empty(M, np.float32)
    am = np.empty(M, np.int32)
    fr = np.empty(M, np.uint8)
    pp = np.empty((M, P), np.float32) if per_point else None
    Lb = library or lib()
    rc = Lb.oracle_query_min(_p(f), L, N, dof, _p(np.ascontiguousarray(params, np.float32)), _p(pts), P, _p(q), M,
                             float(margin), _p(mn), _p(am), _p(fr), _p(pp), int(threads))
    if rc:
        raise ValueError("query_min: empty input")
    return mn, am, fr.astype(bool), pp


def gcc(robot, points, q01, steps=200, margin=0.005, early_exit=False, prune=True, library=None):
    """gcc_min_distance (early_exit False) / gcc_clearance (True) per motion -> (dist, free)."""
    pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    q = np.ascontiguousarray(q01, np.float64).reshape(-1, 2 * robot.dof)
    j = robot.joints_flat()
    c = robot.capsules_flat()
    base = np.ascontiguousarray(robot.base_pose, np.float64).reshape(-1)
    M = q.shape[0]
    dist = np.empty(M, np.float64)
    free = np.empty(M, np.uint8)
    rc = (library or lib()).oracle_gcc(_p(j), robot.dof, _p(c), c.shape[0], _p(base), _p(pts), pts.shape[0], _p(q),
                                       M, int(steps), float(margin), int(early_exit), int(prune), _p(dist), _p(free))
    if rc:
        raise ValueError("gcc: invalid arguments")
    return dist, free.astype(bool)

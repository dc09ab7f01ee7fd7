"""ctypes binding of the C-ABI (include/sweptnet_b200.h).

The shared library is built in-tree (paper_2402_15281_b200/_lib/libsweptnet_b200.so
by build.py) and loaded from there.  There is no fallback: a missing or stale
library raises, so nothing silently runs on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import build as _build

LIB_PATH = _build.LIB

# svn_status
OK, INVALID_ARGUMENT, CUDA_ERROR, OUT_OF_MEMORY, UNSUPPORTED, IO, FORMAT, TRUNCATION, VERSION, NCCL_ERROR, HOST_ERROR = range(11)
SHARD_MODES = {"auto": 0, "motions": 1, "points": 2}
# svn_precision
PREC_BF16, PREC_FP32, PREC_FP32_EXACT, PREC_FP32_SPLIT, PREC_FP16 = 0, 1, 2, 3, 4
PRECISIONS = {"bf16": PREC_BF16, "fp32": PREC_FP32, "fp32_exact": PREC_FP32_EXACT, "fp32_split": PREC_FP32_SPLIT,
              "fp16": PREC_FP16}


class SvnLayer(C.Structure):
    _fields_ = [("concat", C.c_int32), ("act", C.c_int32), ("affine", C.c_int32), ("residual", C.c_int32)]


class SvnModelDesc(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("width", C.c_int32), ("dof", C.c_int32), ("layers", C.POINTER(SvnLayer))]


class SvnSearchResult(C.Structure):
    """svn_search_result: sweptnet::SearchResult (collision.hpp:31-40)."""
    _fields_ = [("found", C.c_int32), ("motion_index", C.c_int32), ("certified_distance", C.c_double),
                ("exact_checks", C.c_int64), ("nn_checks", C.c_int64), ("proxy_seconds", C.c_double),
                ("exact_seconds", C.c_double), ("total_seconds", C.c_double)]


class SvnError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class ReferenceInvalidArgument(SvnError, ValueError):
    """std::invalid_argument in the reference (nn.cpp:98-99, 462, 465)."""


class IoError(SvnError, OSError):
    """sweptnet::IoError (errors.hpp:8)."""


class FormatError(SvnError):
    """sweptnet::FormatError (errors.hpp:13)."""


class TruncationError(SvnError):
    """sweptnet::TruncationError (errors.hpp:18)."""


class VersionError(SvnError):
    """sweptnet::VersionError (errors.hpp:23)."""


_EXC = {INVALID_ARGUMENT: ReferenceInvalidArgument, IO: IoError, FORMAT: FormatError,
        TRUNCATION: TruncationError, VERSION: VersionError}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    override = os.environ.get("SVN_LIB")  # A/B experiments: another in-tree build of the same ABI
    if override:
        ab_dir = (Path(__file__).resolve().parent.parent / "scripts" / "ab").resolve()
        cand = Path(override).resolve()
        if ab_dir not in cand.parents:
            raise RuntimeError(f"SVN_LIB must name an A/B build under {ab_dir} (got {override})")
        return _finish(C.CDLL(str(cand)))
    if os.environ.get("SVN_NO_BUILD") != "1":
        try:
            _build.build()
        except Exception as e:  # no nvcc on this host: use the shipped .so if present
            if not LIB_PATH.exists():
                raise RuntimeError(f"sweptnet_b200 native library missing and build failed: {e}") from e
    if not LIB_PATH.exists():
        raise RuntimeError(f"sweptnet_b200 native library not found at {LIB_PATH}")
    return _finish(C.CDLL(str(LIB_PATH)))


def _finish(L):
    global _lib
    P, I64, I32, D, VP = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_void_p
    desc_p = C.POINTER(SvnModelDesc)
    sig = {
        "svn_param_count": (I64, [desc_p]),
        "svn_trainable_param_count": (I64, [desc_p]),
        "svn_init_params": (C.c_int, [desc_p, C.c_uint64, I32, P]),
        "svn_model_create": (C.c_int, [desc_p, P, I64, I32, C.POINTER(VP)]),
        "svn_model_load_checkpoint": (C.c_int, [C.c_char_p, I32, C.POINTER(VP)]),
        "svn_model_destroy": (C.c_int, [VP]),
        "svn_model_get_program": (C.c_int, [VP, C.POINTER(I32), C.POINTER(I32), C.POINTER(I32), P, I32]),
        "svn_query_min_device": (C.c_int, [VP, C.c_int, P, I64, P, I64, D, P, P, P, P, VP]),
        "svn_query_min": (C.c_int, [VP, C.c_int, P, I64, P, I64, D, P, P, P, P]),
        "svn_query_min_cascade": (C.c_int, [VP, C.c_int, D, D, P, I64, P, I64, D, P, P, P, P]),
        "svn_keys_init_device": (C.c_int, [P, I64, VP]),
        "svn_query_min_keys_device": (C.c_int, [VP, C.c_int, P, I64, I64, P, I64, P, VP]),
        "svn_keys_finalize_device": (C.c_int, [P, I64, D, P, P, P, VP]),
        "svn_forward_eval": (C.c_int, [VP, C.c_int, P, I64, I64, P]),
        "svn_forward_eval_device": (C.c_int, [VP, C.c_int, P, I64, I64, P, VP]),
        "svn_predict_min_distance": (C.c_int, [VP, C.c_int, P, I64, P, P, I32, P, P]),
        "svn_eval_grid": (C.c_int, [VP, C.c_int, P, D, P, P, P, I32, P]),
        "svn_gcc_min_distance": (C.c_int, [P, P, I64, P, I64, I32, D, I32, P, P]),
        "svn_gcc_min_distance_device": (C.c_int, [P, P, I64, P, I64, I32, D, P, P, VP]),
        "svn_gcc_nn_search": (C.c_int, [P, C.c_int, P, P, I64, P, I64, I32, D, I32, C.POINTER(SvnSearchResult)]),
        "svn_multi_create": (C.c_int, [desc_p, P, I64, P, I32, C.POINTER(VP)]),
        "svn_multi_destroy": (C.c_int, [VP]),
        "svn_multi_device_count": (I32, [VP]),
        "svn_set_whole_batch": (None, [I64, I64]),
        "svn_multi_set_scene": (C.c_int, [VP, P, I64]),
        "svn_query_min_multi": (C.c_int, [VP, C.c_int, P, I64, P, I64, D, C.c_int, P, P, P]),
        "svn_query_min_cascade_multi": (C.c_int, [VP, C.c_int, D, D, P, I64, P, I64, D, P, P, P, P]),
        "svn_launch_count": (I64, []),
        "svn_launch_count_reset": (None, []),
        "svn_kernel_timing_begin": (None, []),
        "svn_kernel_timing_end": (C.c_int, [C.POINTER(D), C.POINTER(I64)]),
        "svn_last_error": (C.c_char_p, []),
        "svn_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("SVN_LIB") and not hasattr(L, name):
            continue  # A/B build of an older revision (SVN_LIB): entry points added since are absent
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


EXPORTED = ("svn_param_count", "svn_trainable_param_count", "svn_init_params", "svn_model_create",
            "svn_model_load_checkpoint", "svn_model_destroy", "svn_model_get_program", "svn_query_min_device", "svn_query_min",
            "svn_query_min_cascade", "svn_keys_init_device", "svn_query_min_keys_device", "svn_keys_finalize_device", "svn_forward_eval",
            "svn_forward_eval_device", "svn_predict_min_distance", "svn_eval_grid", "svn_gcc_min_distance",
            "svn_gcc_min_distance_device", "svn_gcc_nn_search", "svn_multi_create", "svn_multi_destroy",
            "svn_multi_device_count", "svn_multi_set_scene", "svn_set_whole_batch", "svn_query_min_multi", "svn_query_min_cascade_multi", "svn_launch_count",
            "svn_launch_count_reset",
            "svn_kernel_timing_begin", "svn_kernel_timing_end", "svn_last_error", "svn_version")


def check(status: int) -> None:
    if status != OK:
        msg = lib().svn_last_error().decode()
        raise _EXC.get(status, SvnError)(status, msg)


def make_desc(program) -> tuple[SvnModelDesc, C.Array]:
    arr = (SvnLayer * program.n_layers)(*[SvnLayer(*l.flags()) for l in program.layers])
    return SvnModelDesc(program.n_layers, program.width, program.dof, arr), arr


def ptr(x) -> C.c_void_p:
    """Raw pointer of a numpy array or torch tensor (None -> NULL)."""
    if x is None:
        return C.c_void_p(0)
    if hasattr(x, "data_ptr"):
        return C.c_void_p(x.data_ptr())
    return C.c_void_p(x.ctypes.data)

"""Python mirror of the reference's inference interface, on the B200 C-ABI.

Names, argument meaning and error behaviour follow /root/reference/proj:
    init_model            nn.hpp:80-81   / nn.cpp:57-93
    forward_eval          nn.hpp:92-93   / nn.cpp:95-130
    predict_min_distance  nn.hpp:162-163 / nn.cpp:460-480
    load_checkpoint       nn.hpp:168     / nn.cpp:524-576
    ProxyEvaluator        collision.hpp:45 (batched: Model.query_min / batched_proxy)
Argument errors raise ReferenceInvalidArgument (a ValueError) carrying the
reference's std::invalid_argument text.  Every call runs the CUDA library; there
is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import abi
from .program import LayerProgram, fig2


def init_params(program: LayerProgram, seed: int, bound: str = "he") -> np.ndarray:
    """Seeded parameters (init_model, nn.cpp:57-93, on std::mt19937_64).
    bound: "ref" = uniform(+-1/sqrt(fan_in)) as init_model; "he" = +-sqrt(6/fan_in)."""
    desc, _keep = abi.make_desc(program)
    out = np.empty(program.param_floats(), dtype=np.float32)
    abi.check(abi.lib().svn_init_params(C.byref(desc), C.c_uint64(seed), 1 if bound == "he" else 0, abi.ptr(out)))
    return out


@dataclass
class QueryResult:
    min: np.ndarray       # float32 [M]
    argmin: np.ndarray    # int32 [M]
    free: np.ndarray      # bool [M]: double(min) > margin
    per_point: np.ndarray | None = None  # float32 [M, P]


class Model:
    """A model resident on one GPU (immutable, shareable across threads)."""

    def __init__(self, program: LayerProgram, params: np.ndarray, device: int = 0):
        params = np.ascontiguousarray(params, dtype=np.float32)
        if params.size != program.param_floats():
            raise abi.ReferenceInvalidArgument(abi.INVALID_ARGUMENT, "model: parameter count mismatch")
        self.program = program
        self.device = device
        desc, keep = abi.make_desc(program)
        h = C.c_void_p()
        abi.check(abi.lib().svn_model_create(C.byref(desc), abi.ptr(params), params.size, device, C.byref(h)))
        self._h = h
        self.params = params

    @classmethod
    def from_checkpoint(cls, path: str, device: int = 0) -> "Model":
        """load_checkpoint (nn.cpp:524-576): SVCKPT01 -> Fig. 2 program."""
        h = C.c_void_p()
        abi.check(abi.lib().svn_model_load_checkpoint(str(path).encode(), device, C.byref(h)))
        with open(path, "rb") as f:
            f.read(8)
            _ver, n_blocks, block_dim, input_dim = np.frombuffer(f.read(16), dtype=np.uint32)
            params = np.frombuffer(f.read(), dtype=np.float32).copy()
        self = cls.__new__(cls)
        self.program = fig2(int(n_blocks), int(block_dim), (int(input_dim) - 3) // 2)
        self.device = device
        self._h = h
        self.params = params
        return self

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None):
            abi.lib().svn_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ host entry --
    def query_min(self, points: np.ndarray, q01: np.ndarray, margin: float, precision: str = "bf16",
                  per_point: bool = False) -> QueryResult:
        """Every (point x motion) pair -> per-motion min, argmin, `min > margin`.
        points float [P, 3]; q01 float [M, 2*dof] = (q0 | q1).
        precision: "bf16" (tcgen05, per-network stated bound), "fp16" (the same kernels on fp16
        operands: ~9x tighter bound at ~0.95x the throughput; rows leaving the fp16 range are
        reported as -inf), "fp32" / "fp32_exact" (the FP32
        path: FFMA in the reference's order, bit-identical to the oracle), "fp32_split"
        (width 256/512: fp32-grade split-fp16 on tcgen05; 1e-5 at width 256, a stated bound at
        width 512)."""
        pts = np.ascontiguousarray(points, dtype=np.float32).reshape(-1, 3)
        q = np.ascontiguousarray(q01, dtype=np.float32).reshape(-1, 2 * self.program.dof)
        P, M = pts.shape[0], q.shape[0]
        mn = np.empty(M, np.float32)
        am = np.empty(M, np.int32)
        fr = np.empty(M, np.uint8)
        pp = np.empty((M, P), np.float32) if per_point else None
        abi.check(abi.lib().svn_query_min(self._h, abi.PRECISIONS[precision], abi.ptr(pts), P, abi.ptr(q), M,
                                          float(margin), abi.ptr(mn), abi.ptr(am), abi.ptr(fr), abi.ptr(pp)))
        return QueryResult(mn, am, fr.astype(bool), pp)

    def query_min_cascade(self, points: np.ndarray, q01: np.ndarray, margin: float, band_coarse: float,
                          band_split: float, coarse: str = "fp16") -> tuple[QueryResult, tuple[int, int, int]]:
        """query_min whose class `free` equals the FP32 path's (the reference's, collision.cpp:68)
        for EVERY motion: the batch on `coarse` ("fp16" | "bf16"), the motions within band_coarse
        of the margin (the precision's stated bound) or not finite again on fp32_split, those
        within band_split of it on the FP32 path.  Returns the result (min/argmin of the finest
        stage evaluated per motion) and the motions evaluated per stage."""
        pts = np.ascontiguousarray(points, dtype=np.float32).reshape(-1, 3)
        q = np.ascontiguousarray(q01, dtype=np.float32).reshape(-1, 2 * self.program.dof)
        P, M = pts.shape[0], q.shape[0]
        mn, am, fr = np.empty(M, np.float32), np.empty(M, np.int32), np.empty(M, np.uint8)
        stages = np.zeros(3, np.int64)
        abi.check(abi.lib().svn_query_min_cascade(self._h, abi.PRECISIONS[coarse], float(band_coarse),
                                                  float(band_split), abi.ptr(pts), P, abi.ptr(q), M, float(margin),
                                                  abi.ptr(mn), abi.ptr(am), abi.ptr(fr), abi.ptr(stages)))
        return QueryResult(mn, am, fr.astype(bool)), (int(stages[0]), int(stages[1]), int(stages[2]))

    def forward_eval(self, raw: np.ndarray, precision: str = "fp32_exact") -> np.ndarray:
        """forward_eval<float> (nn.cpp:95-130): raw [B, 3 + 2*dof] rows [x, q0, q1]."""
        raw = np.ascontiguousarray(raw, dtype=np.float32)
        if raw.ndim != 2:
            raise abi.ReferenceInvalidArgument(abi.INVALID_ARGUMENT, "forward: input width mismatch")
        out = np.empty(raw.shape[0], np.float32)
        abi.check(abi.lib().svn_forward_eval(self._h, abi.PRECISIONS[precision], abi.ptr(raw), raw.shape[0],
                                             raw.shape[1], abi.ptr(out)))
        return out

    def predict_min_distance(self, cloud, q0, q1, precision: str = "fp32_exact") -> tuple[float, int]:
        """predict_min_distance (nn.cpp:460-480): double cloud [P,3] and q -> (double min, int argmin)."""
        cloud = np.ascontiguousarray(cloud, dtype=np.float64).reshape(-1, 3)
        q0 = np.ascontiguousarray(q0, dtype=np.float64).reshape(-1)
        q1 = np.ascontiguousarray(q1, dtype=np.float64).reshape(-1)
        mn = C.c_double()
        am = C.c_int32()
        abi.check(abi.lib().svn_predict_min_distance(self._h, abi.PRECISIONS[precision], abi.ptr(cloud),
                                                     cloud.shape[0], abi.ptr(q0), abi.ptr(q1), q0.size,
                                                     C.byref(mn), C.byref(am)))
        return mn.value, am.value

    def eval_grid(self, origin, voxel_size: float, dims, q0, q1, precision: str = "fp32_exact") -> np.ndarray:
        """NN branch of cmd_reconstruct (cli.cpp:240-261): every voxel centre of the grid
        for one motion; returns float32 [dx, dy, dz] (SdfGrid::values order)."""
        o = np.ascontiguousarray(origin, np.float64).reshape(3)
        d = np.ascontiguousarray(dims, np.int32).reshape(3)
        q0 = np.ascontiguousarray(q0, np.float64).reshape(-1)
        q1 = np.ascontiguousarray(q1, np.float64).reshape(-1)
        out = np.empty(int(np.prod(d.astype(np.int64))), np.float32)
        abi.check(abi.lib().svn_eval_grid(self._h, abi.PRECISIONS[precision], abi.ptr(o), float(voxel_size),
                                          abi.ptr(d), abi.ptr(q0), abi.ptr(q1), q0.size, abi.ptr(out)))
        return out.reshape(tuple(int(x) for x in d))

    # ---------------------------------------------------------- device entry --
    def query_min_device(self, points, q01, margin: float, min_out, argmin_out, free_out, per_point=None,
                         precision: str = "bf16", stream=None) -> None:
        """Device-resident batched query on torch CUDA tensors; asynchronous on `stream`."""
        st = C.c_void_p(stream.cuda_stream if stream is not None else 0)
        abi.check(abi.lib().svn_query_min_device(self._h, abi.PRECISIONS[precision], abi.ptr(points),
                                                 points.shape[0], abi.ptr(q01), q01.shape[0], float(margin),
                                                 abi.ptr(min_out), abi.ptr(argmin_out), abi.ptr(free_out),
                                                 abi.ptr(per_point), st))

    def query_keys_device(self, points, index_offset: int, q01, keys, precision: str = "bf16", stream=None) -> None:
        """Point-shard partial: atomicMin of packed (delta, index) keys into `keys` (uint64 as int64 tensor)."""
        st = C.c_void_p(stream.cuda_stream if stream is not None else 0)
        abi.check(abi.lib().svn_query_min_keys_device(self._h, abi.PRECISIONS[precision], abi.ptr(points),
                                                      points.shape[0], int(index_offset), abi.ptr(q01),
                                                      q01.shape[0], abi.ptr(keys), st))


class MultiModel:
    """One model per listed GPU of this box, driven from this process by one native worker
    thread per device (svn_multi_*).  query_min has Model.query_min's
    contract; shard = "motions" (no communication), "points" (one NCCL u64 MIN all-reduce of
    8 B per motion; distinct devices only) or "auto" (points when there are fewer motions
    than devices).  Results are bit-identical to a single Model."""

    def __init__(self, program: LayerProgram, params: np.ndarray, devices=(0,)):
        params = np.ascontiguousarray(params, dtype=np.float32)
        if params.size != program.param_floats():
            raise abi.ReferenceInvalidArgument(abi.INVALID_ARGUMENT, "model: parameter count mismatch")
        self.program = program
        self.devices = tuple(int(d) for d in devices)
        desc, keep = abi.make_desc(program)
        devs = np.asarray(self.devices, dtype=np.int32)
        h = C.c_void_p()
        abi.check(abi.lib().svn_multi_create(C.byref(desc), abi.ptr(params), params.size, abi.ptr(devs),
                                             len(self.devices), C.byref(h)))
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None):
            abi.lib().svn_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_scene(self, points) -> None:
        """Keep one scene's cloud resident on every device (svn_multi_set_scene); query_min
        with points=None then runs against it.  points=None drops the scene."""
        if points is None:
            abi.check(abi.lib().svn_multi_set_scene(self._h, None, 0))
            self._scene_points = 0
            return
        pts = np.ascontiguousarray(points, dtype=np.float32).reshape(-1, 3)
        abi.check(abi.lib().svn_multi_set_scene(self._h, abi.ptr(pts), pts.shape[0]))
        self._scene_points = pts.shape[0]

    def query_min(self, points, q01: np.ndarray, margin: float, precision: str = "bf16",
                  shard: str = "auto") -> QueryResult:
        q = np.ascontiguousarray(q01, dtype=np.float32).reshape(-1, 2 * self.program.dof)
        M = q.shape[0]
        if points is None:  # the resident scene
            pts, P = None, getattr(self, "_scene_points", 0)
        else:
            pts = np.ascontiguousarray(points, dtype=np.float32).reshape(-1, 3)
            P = pts.shape[0]
        mn = np.empty(M, np.float32)
        am = np.empty(M, np.int32)
        fr = np.empty(M, np.uint8)
        abi.check(abi.lib().svn_query_min_multi(self._h, abi.PRECISIONS[precision],
                                                abi.ptr(pts) if pts is not None else None, P, abi.ptr(q), M,
                                                float(margin), abi.SHARD_MODES[shard], abi.ptr(mn), abi.ptr(am),
                                                abi.ptr(fr)))
        return QueryResult(mn, am, fr.astype(bool), None)

    def query_min_cascade(self, points, q01, margin: float, band_coarse: float, band_split: float,
                          coarse: str = "fp16"):
        """Model.query_min_cascade over the box (svn_query_min_cascade_multi): motions split over the
        devices, the class equal to the FP32 path's for every motion, outputs equal to one device's."""
        pts = np.ascontiguousarray(points, dtype=np.float32).reshape(-1, 3)
        q = np.ascontiguousarray(q01, dtype=np.float32).reshape(-1, 2 * self.program.dof)
        P, M = pts.shape[0], q.shape[0]
        mn, am, fr = np.empty(M, np.float32), np.empty(M, np.int32), np.empty(M, np.uint8)
        stages = np.zeros(3, np.int64)
        abi.check(abi.lib().svn_query_min_cascade_multi(self._h, abi.PRECISIONS[coarse], float(band_coarse),
                                                        float(band_split), abi.ptr(pts), P, abi.ptr(q), M, float(margin),
                                                        abi.ptr(mn), abi.ptr(am), abi.ptr(fr), abi.ptr(stages)))
        return QueryResult(mn, am, fr.astype(bool), None), (int(stages[0]), int(stages[1]), int(stages[2]))


class whole_batch:
    """`with whole_batch(M_total, P_total): ...` — the calls inside are shards (motion ranges or
    point chunks) of one batch of that shape and take its tile shape, so the tensor-core
    precisions give the same bits whatever the split (svn_set_whole_batch; thread-local)."""

    def __init__(self, motions: int, points: int):
        self.shape = (int(motions), int(points))

    def __enter__(self):
        abi.lib().svn_set_whole_batch(*self.shape)
        return self

    def __exit__(self, *exc):
        abi.lib().svn_set_whole_batch(0, 0)
        return False


def keys_init_device(keys, stream=None) -> None:
    st = C.c_void_p(stream.cuda_stream if stream is not None else 0)
    abi.check(abi.lib().svn_keys_init_device(abi.ptr(keys), keys.numel(), st))


def keys_finalize_device(keys, margin: float, min_out, argmin_out, free_out, stream=None) -> None:
    st = C.c_void_p(stream.cuda_stream if stream is not None else 0)
    abi.check(abi.lib().svn_keys_finalize_device(abi.ptr(keys), keys.numel(), float(margin), abi.ptr(min_out),
                                                 abi.ptr(argmin_out), abi.ptr(free_out), st))


def batched_proxy(model: Model, cloud: np.ndarray, motions_q01: np.ndarray, precision: str = "bf16"):
    """ProxyEvaluator (collision.hpp:45) for gcc_nn_search_impl, batched: one GPU call
    for every motion of a scene; returns proxy(j) as a callable."""
    res = model.query_min(cloud, motions_q01, 0.0, precision=precision)
    vals = res.min.astype(np.float64)
    return lambda j: float(vals[j])


def launch_count() -> int:
    return int(abi.lib().svn_launch_count())


def launch_count_reset() -> None:
    abi.lib().svn_launch_count_reset()


def kernel_timing_begin() -> None:
    abi.lib().svn_kernel_timing_begin()


def kernel_timing_end() -> tuple[float, int]:
    ms = C.c_double()
    n = C.c_int64()
    abi.check(abi.lib().svn_kernel_timing_end(C.byref(ms), C.byref(n)))
    return ms.value, n.value

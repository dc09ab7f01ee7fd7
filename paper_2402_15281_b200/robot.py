"""Robot models for the geometric checker (svn_gcc_min_distance).

default_robot restates the reference's fixed synthetic manipulator
(/root/reference/proj/src/robot.cpp:85-131): revolute joints alternating z / y axes,
offsets along local z, one capsule per link from (0,0,-len) to the frame origin, limits
+-170 deg (z joints) / +-120 deg (y joints) rounded to float.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import abi

# chain_spec (robot.cpp:99-111): link lengths and capsule radii per dof
_CHAINS = {
    2: ([0.55, 0.45], [0.060, 0.050]),
    3: ([0.40, 0.35, 0.25], [0.060, 0.050, 0.045]),
    4: ([0.35, 0.30, 0.20, 0.15], [0.060, 0.052, 0.047, 0.042]),
    5: ([0.28, 0.25, 0.20, 0.15, 0.12], [0.060, 0.053, 0.048, 0.044, 0.040]),
    6: ([0.20, 0.25, 0.20, 0.15, 0.12, 0.08], [0.060, 0.055, 0.050, 0.045, 0.042, 0.040]),
    7: ([0.18, 0.17, 0.16, 0.14, 0.13, 0.12, 0.10], [0.060, 0.055, 0.050, 0.047, 0.044, 0.042, 0.040]),
}


class SvnJoint(C.Structure):
    _fields_ = [("axis", C.c_double * 3), ("offset", C.c_double * 3)]


class SvnCapsule(C.Structure):
    _fields_ = [("link", C.c_int32), ("pad", C.c_int32), ("a", C.c_double * 3), ("b", C.c_double * 3),
                ("radius", C.c_double)]


class SvnRobotDesc(C.Structure):
    _fields_ = [("dof", C.c_int32), ("joints", C.POINTER(SvnJoint)), ("n_capsules", C.c_int32),
                ("capsules", C.POINTER(SvnCapsule)), ("base_pose", C.POINTER(C.c_double))]


@dataclass
class Robot:
    axes: np.ndarray      # [dof, 3]
    offsets: np.ndarray   # [dof, 3]
    capsules: list        # [(link, a[3], b[3], radius)], link-major
    lower: np.ndarray
    upper: np.ndarray
    base_pose: np.ndarray  # [3, 4]

    @property
    def dof(self) -> int:
        return int(self.axes.shape[0])

    def joints_flat(self) -> np.ndarray:
        """[dof, 6] = (axis, offset) — the oracle's layout."""
        return np.ascontiguousarray(np.concatenate([self.axes, self.offsets], axis=1), np.float64)

    def capsules_flat(self) -> np.ndarray:
        """[n, 8] = (link, a, b, r) — the oracle's layout."""
        return np.array([[l, *a, *b, r] for l, a, b, r in self.capsules], np.float64)

    def desc(self):
        js = (SvnJoint * self.dof)(*[SvnJoint((C.c_double * 3)(*self.axes[i]), (C.c_double * 3)(*self.offsets[i]))
                                     for i in range(self.dof)])
        cs = (SvnCapsule * len(self.capsules))(*[SvnCapsule(l, 0, (C.c_double * 3)(*a), (C.c_double * 3)(*b), r)
                                                 for l, a, b, r in self.capsules])
        base = (C.c_double * 12)(*np.asarray(self.base_pose, np.float64).reshape(-1))
        d = SvnRobotDesc(self.dof, js, len(self.capsules), cs, base)
        return d, (js, cs, base)


def default_robot(dof: int) -> Robot:
    if dof not in _CHAINS:
        raise ValueError("default_robot: dof must be in 2..7")
    lengths, radii = _CHAINS[dof]
    lim_z = float(np.float32(170.0 * np.pi / 180.0))
    lim_y = float(np.float32(120.0 * np.pi / 180.0))
    axes = np.array([[0, 0, 1] if i % 2 == 0 else [0, 1, 0] for i in range(dof)], np.float64)
    offsets = np.array([[0, 0, lengths[i]] for i in range(dof)], np.float64)
    caps = [(i, (0.0, 0.0, -lengths[i]), (0.0, 0.0, 0.0), radii[i]) for i in range(dof)]
    lim = np.array([lim_z if i % 2 == 0 else lim_y for i in range(dof)])
    return Robot(axes, offsets, caps, -lim, lim, np.eye(3, 4))


def gcc_min_distance(robot: Robot, points: np.ndarray, q01: np.ndarray, steps: int = 200, margin: float = 0.005,
                     device: int = 0):
    """GPU geometric checker: per motion (exact min distance, min > margin)
    = gcc_min_distance / gcc_clearance(...).free (collision.cpp:18-34)."""
    pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
    q = np.ascontiguousarray(q01, np.float64).reshape(-1, 2 * robot.dof)
    M = q.shape[0]
    dist = np.empty(M, np.float64)
    free = np.empty(M, np.uint8)
    desc, keep = robot.desc()
    abi.check(abi.lib().svn_gcc_min_distance(C.byref(desc), abi.ptr(pts), pts.shape[0], abi.ptr(q), M, int(steps),
                                             float(margin), int(device), abi.ptr(dist), abi.ptr(free)))
    return dist, free.astype(bool)


def gcc_nn_search(model, robot: Robot, cloud: np.ndarray, q01: np.ndarray, steps: int = 200, margin: float = 0.005,
                  precision: str = "fp32", batch: int = 64) -> dict:
    """Alg. 1 on the GPU: gcc_nn_search (collision.cpp:120-130, impl 55-107) with the proxy
    (`model`, one batched launch) and the geometric checker (batches in the sequential
    algorithm's visiting order).  Returns the fields of sweptnet::SearchResult."""
    pts = np.ascontiguousarray(cloud, np.float64).reshape(-1, 3)
    q = np.ascontiguousarray(q01, np.float64).reshape(-1, 2 * robot.dof)
    res = abi.SvnSearchResult()
    desc, keep = robot.desc()
    abi.check(abi.lib().svn_gcc_nn_search(model._h, abi.PRECISIONS[precision], C.byref(desc), abi.ptr(pts),
                                          pts.shape[0], abi.ptr(q), q.shape[0], int(steps), float(margin), int(batch),
                                          C.byref(res)))
    return {"found": bool(res.found), "motion_index": int(res.motion_index),
            "certified_distance": float(res.certified_distance), "exact_checks": int(res.exact_checks),
            "nn_checks": int(res.nn_checks), "proxy_seconds": float(res.proxy_seconds),
            "exact_seconds": float(res.exact_seconds), "total_seconds": float(res.total_seconds)}

"""Seeded synthetic workloads for BASELINE.json's configs (c1..c5).

No public dataset is named by the reference or BASELINE.json; these generators
stand in for the paper's box-world / bin-picking clouds with the shapes, sizes and
value ranges BASELINE.json states.  Motions are drawn
from one seeded stream so any motion shard is a slice of the 1-GPU input.

Placement choices (unspecified upstream, recorded here and in DESIGN.md):
  bin box         x in [0, 1.2], y in [-0.4, 0.4], z in [0, 0.5] m, robot base at origin
  obstacle boxes  8 axis-aligned, sides U[5, 30] cm, centres inside the bin box,
                  area-weighted face sampling (pattern of geometry.cpp:72-93)
  c4 scene        1.2 x 0.8 m plane at z=0 with N(0, 2 mm) normal noise + 20 ellipsoids,
                  semi-axes U[3, 15] cm, points split by surface area
  joint limits    default_robot(6): +-170 deg (z joints) / +-120 deg (y joints) alternating
                  (robot.cpp:91-92,122); c1 U[-pi, pi]; c4 +-170 deg on all 7 joints
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .program import LayerProgram, deepsdf, fig2, plain

BIN_LO = np.array([0.0, -0.4, 0.0])
BIN_HI = np.array([1.2, 0.4, 0.5])
LIM_Z = float(np.float32(170.0 * np.pi / 180.0))  # robot.cpp:89-91 rounds limits to float
LIM_Y = float(np.float32(120.0 * np.pi / 180.0))


def substream_seed(base: int, index: int) -> int:
    """rng.hpp:68-73 (SplitMix64 finaliser)."""
    m = (1 << 64) - 1
    z = (base + 0x9E3779B97F4A7C15 * (index + 1)) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(substream_seed(seed, stream)))


def uniform_box(rng, n, lo=BIN_LO, hi=BIN_HI) -> np.ndarray:
    return lo + (hi - lo) * rng.random((n, 3))


def box_surfaces(rng, n, n_boxes=8) -> np.ndarray:
    """n points on the surfaces of n_boxes random AABBs inside the bin, area-weighted."""
    sides = rng.uniform(0.05, 0.30, size=(n_boxes, 3))
    centres = BIN_LO + sides / 2 + (BIN_HI - BIN_LO - sides).clip(min=0) * rng.random((n_boxes, 3))
    # 6 faces per box: area of face (axis a) = product of the other two sides
    faces = []
    for b in range(n_boxes):
        for a in range(3):
            area = np.prod(np.delete(sides[b], a))
            faces += [(b, a, +1, area), (b, a, -1, area)]
    areas = np.array([f[3] for f in faces])
    which = rng.choice(len(faces), size=n, p=areas / areas.sum())
    u = rng.random((n, 3)) - 0.5
    out = np.empty((n, 3))
    for i, (b, a, sgn, _area) in enumerate(faces):
        sel = which == i
        k = int(sel.sum())
        if not k:
            continue
        local = u[sel] * sides[b]
        local[:, a] = sgn * sides[b][a] / 2
        out[sel] = centres[b] + local
    return out


def bin_cloud(rng, n) -> np.ndarray:
    """c2/c3/c5 cloud: 50 % uniform in the bin box, 50 % on 8 random box surfaces."""
    n_u = n // 2
    pts = np.concatenate([uniform_box(rng, n_u), box_surfaces(rng, n - n_u)])
    return pts[rng.permutation(n)]


def _ellipsoid_area(a, b, c, p=1.6075):
    return 4 * np.pi * (((a * b) ** p + (a * c) ** p + (b * c) ** p) / 3) ** (1 / p)


def depth_scan_cloud(rng, n, n_ell=20) -> np.ndarray:
    """c4 cloud: noisy 1.2 x 0.8 m plane + 20 ellipsoid surfaces, split by area."""
    axes = rng.uniform(0.03, 0.15, size=(n_ell, 3))
    centres = np.stack([rng.uniform(0.1, 1.1, n_ell), rng.uniform(-0.3, 0.3, n_ell),
                        rng.uniform(0.05, 0.4, n_ell)], axis=1)
    areas = np.concatenate([[1.2 * 0.8], _ellipsoid_area(*axes.T)])
    counts = rng.multinomial(n, areas / areas.sum())
    parts = []
    k = counts[0]
    plane = np.stack([rng.uniform(0, 1.2, k), rng.uniform(-0.4, 0.4, k), rng.normal(0, 0.002, k)], axis=1)
    parts.append(plane)
    for e in range(n_ell):
        k = int(counts[e + 1])
        if k == 0:  # a cloud of a few points: this ellipsoid drew none
            continue
        got = []
        a, b, c = axes[e]
        wmax = max(b * c, a * c, a * b)
        while sum(len(g) for g in got) < k:
            d = rng.normal(size=(2 * k + 8, 3))
            d /= np.linalg.norm(d, axis=1, keepdims=True)
            w = np.sqrt((b * c * d[:, 0]) ** 2 + (a * c * d[:, 1]) ** 2 + (a * b * d[:, 2]) ** 2) / wmax
            got.append(d[rng.random(len(d)) < w])
        d = np.concatenate(got)[:k]
        parts.append(centres[e] + d * axes[e])
    pts = np.concatenate(parts)
    return pts[rng.permutation(n)]


def limits_default(dof: int) -> np.ndarray:
    return np.array([LIM_Z if i % 2 == 0 else LIM_Y for i in range(dof)])


def sample_motions(rng, m, lim: np.ndarray) -> np.ndarray:
    """[m, 2*dof] = (q0 | q1), each uniform within +-lim (sample_motion, dataset.cpp:57-66)."""
    lim2 = np.concatenate([lim, lim])
    return -lim2 + 2 * lim2 * rng.random((m, lim2.size))


@dataclass(frozen=True)
class Workload:
    key: str
    description: str
    program: LayerProgram
    motions: int
    points: int
    margin: float
    precision: str         # "fp32" or "bf16"
    bound: str             # weight init bound ("he")
    cloud: Callable
    q_limits: Callable

    @property
    def queries(self) -> int:
        return self.motions * self.points

    def make(self, seed: int = 0, motions: int | None = None, points: int | None = None,
             motion_offset: int = 0):
        """Returns (points float32 [P,3], q01 float32 [M, 2*dof]).  motion_offset/motions
        slice the motion stream (shards are slices of the 1-GPU input)."""
        P = self.points if points is None else points
        M = self.motions if motions is None else motions
        pts = self.cloud(_rng(seed, 1), P).astype(np.float32)
        allq = sample_motions(_rng(seed, 2), motion_offset + M, self.q_limits())
        return np.ascontiguousarray(pts), np.ascontiguousarray(allq[motion_offset:].astype(np.float32))


WORKLOADS: dict[str, Workload] = {
    "c1": Workload("c1", "CPU-runnable ref: plain 4x256 fp32, 6-DoF, 1 motion x 4096 points",
                   plain(4, 256, 6), 1, 4096, 0.02, "fp32", "he",
                   lambda r, n: uniform_box(r, n), lambda: np.full(6, np.pi)),
    "c2": Workload("c2", "plain 4x256 fp32, 6-DoF, 64 motions x 16384 points (bin + 8 boxes)",
                   plain(4, 256, 6), 64, 16384, 0.02, "fp32", "he", bin_cloud, lambda: limits_default(6)),
    "c3": Workload("c3", "DeepSDF 8x512 concat@4 bf16, 6-DoF, 1024 motions x 65536 points",
                   deepsdf(8, 512, 6, 4), 1024, 65536, 0.02, "bf16", "he", bin_cloud, lambda: limits_default(6)),
    "c4": Workload("c4", "plain 6x512 bf16, 7-DoF (+-170 deg), 4096 motions x 100000 points (plane + 20 ellipsoids)",
                   plain(6, 512, 7), 4096, 100000, 0.02, "bf16", "he", depth_scan_cloud,
                   lambda: np.full(7, LIM_Z)),
    "c5": Workload("c5", "DeepSDF 8x512 concat@4 bf16, 32768 motions x 262144 points (motion-sharded)",
                   deepsdf(8, 512, 6, 4), 32768, 262144, 0.02, "bf16", "he", bin_cloud, lambda: limits_default(6)),
    "c5single": Workload("c5single", "DeepSDF 8x512 concat@4 bf16, 1 motion x 16777216 points (point-sharded)",
                         deepsdf(8, 512, 6, 4), 1, 1 << 24, 0.02, "bf16", "he", bin_cloud,
                         lambda: limits_default(6)),
    # context only (not a BASELINE config): the network the paper timed on an RTX 3090
    # (Fig. 2 wiring, 5 blocks x 512), one motion x 20000 points as there,
    # reference init (nn.cpp:57-93); --motions widens it to a batch of motions
    "paper": Workload("paper", "paper's Fig. 2 5x512 network (PAPER.md:556), 1 motion x 20000 points",
                      fig2(5, 512, 6), 1, 20000, 0.005, "bf16", "ref", bin_cloud, lambda: limits_default(6)),
}

"""Geometric collision checker: oracle restatement pinned against an
independent numpy implementation; the GPU checker against the oracle."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2402_15281_b200.robot import default_robot, gcc_min_distance
from paper_2402_15281_b200.workloads import WORKLOADS


def _rot(axis, ang):
    x, y, z = axis
    c, s = np.cos(ang), np.sin(ang)
    K = np.array([[0, -z, y], [z, 0, -x], [-y, x, 0]])
    return np.eye(3) + s * K + (1 - c) * (K @ K)


def _numpy_gcc(robot, pts, q01, steps):
    """Independent brute force: every config, every capsule, every point."""
    out = []
    dof = robot.dof
    for q in q01:
        q0, q1 = q[:dof], q[dof:]
        best = np.inf
        for i in range(steps):
            s = i / (steps - 1)
            qi = np.where(q0 == q1, q0, (1 - s) * q0 + s * q1)
            R, p = np.eye(3), np.zeros(3)
            for j in range(dof):
                R = R @ _rot(robot.axes[j], qi[j])
                p = p + R @ robot.offsets[j]
                for link, a, b, r in robot.capsules:
                    if link != j:
                        continue
                    A, B = R @ np.array(a) + p, R @ np.array(b) + p
                    pa, ba = pts - A, B - A
                    t = np.clip(pa @ ba / (ba @ ba), 0, 1)
                    d = np.linalg.norm(pa - t[:, None] * ba, axis=1) - r
                    best = min(best, d.min())
        out.append(best)
    return np.array(out)


def test_zero_configuration_geometry():
    r = default_robot(6)
    q = np.zeros((1, 12))
    # point 1 m along +x at height 0.1: nearest is link 0 (axis z from 0 to 0.2, radius 0.06)
    d, f = O.gcc(r, np.array([[1.0, 0.0, 0.1]]), q, steps=2, margin=0.005)
    assert abs(d[0] - (1.0 - 0.060)) < 1e-12 and f[0]
    # on top of the arm: total height 1.0, last link radius 0.04
    d, _ = O.gcc(r, np.array([[0.0, 0.0, 1.5]]), q, steps=2, margin=0.005)
    assert abs(d[0] - (0.5 - 0.040)) < 1e-12


@pytest.mark.parametrize("dof", [2, 6, 7])
def test_oracle_gcc_matches_independent_numpy(dof):
    r = default_robot(dof)
    rng = np.random.default_rng(dof)
    pts = rng.uniform([-0.8, -0.8, -0.2], [0.8, 0.8, 1.2], size=(150, 3))
    lim = np.concatenate([r.upper, r.upper])
    q = rng.uniform(-lim, lim, size=(3, 2 * dof))
    q[0, 1] = q[0, dof + 1]  # identical component: exact, not interpolated
    d, _ = O.gcc(r, pts, q, steps=25, margin=0.005)
    ref = _numpy_gcc(r, pts, q, 25)
    assert np.abs(d - ref).max() < 1e-9


def test_oracle_gcc_pruning_and_early_exit_consistent():
    r = default_robot(6)
    pts, q = WORKLOADS["c2"].make(seed=4, motions=6, points=400)
    pts = pts + np.array([0.6, 0.0, 0.0], np.float32)  # push part of the cloud away so some motions are free
    d_full, f_full = O.gcc(r, pts, q, steps=60, margin=0.02)
    d_np, _ = O.gcc(r, pts, q, steps=60, margin=0.02, prune=False)
    assert np.array_equal(d_full, d_np)  # the 1e-9-slack skip never changes the min
    d_ee, f_ee = O.gcc(r, pts, q, steps=60, margin=0.02, early_exit=True)
    assert np.array_equal(f_ee, f_full)  # gcc_clearance.free == (gcc_min_distance > margin)
    assert np.array_equal(d_ee[f_full], d_full[f_full])  # free: certified == exact min


@pytest.mark.gpu
@pytest.mark.parametrize("dof,wkey", [(6, "c2"), (7, "c4")])
def test_gpu_gcc_matches_oracle(dof, wkey):
    r = default_robot(dof)
    pts, q = WORKLOADS[wkey].make(seed=6, motions=12, points=3000)
    pts = pts + np.array([0.4, 0.0, 0.0], np.float32)
    d_gpu, f_gpu = gcc_min_distance(r, pts, q, steps=200, margin=0.02)
    d_ref, f_ref = O.gcc(r, pts, q, steps=200, margin=0.02)
    assert np.abs(d_gpu - d_ref).max() <= 1e-12
    amb = np.abs(d_ref - 0.02) <= 1e-12
    assert np.array_equal(f_gpu[~amb], f_ref[~amb])


def _sequential_search(proxies, dist, margin):
    """gcc_nn_search_impl (collision.cpp:55-107) over precomputed proxy and checker values."""
    M = len(proxies)
    nn = ex = 0
    done = [False] * M
    for j in range(M):
        nn += 1
        if proxies[j] > margin:
            ex += 1
            done[j] = True
            if dist[j] > margin:
                return True, j, dist[j], ex, nn
    for j in sorted((j for j in range(M) if not done[j]), key=lambda j: -proxies[j]):  # stable, descending
        ex += 1
        if dist[j] > margin:
            return True, j, dist[j], ex, nn
    return False, -1, 0.0, ex, nn


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["loop1", "loop2", "none"])
def test_gcc_nn_search_matches_sequential_algorithm(case):
    import paper_2402_15281_b200 as S
    from paper_2402_15281_b200.robot import gcc_nn_search
    r = default_robot(6)
    rng = np.random.default_rng(12)
    lo, hi = ([0.2, -0.5, 0.1], [0.6, 0.5, 0.8]) if case != "none" else ([-0.2, -0.2, 0.0], [0.2, 0.2, 0.3])
    cloud = rng.uniform(lo, hi, size=(1200, 3))
    M, margin, steps = 40, 0.02, 24
    q01 = rng.uniform(-1, 1, size=(M, 12)) * np.concatenate([r.upper, r.upper])
    w = WORKLOADS["c2"]
    params = S.init_params(w.program, 12, w.bound)
    prox = np.array([O.predict_min_distance(w.program, params, cloud, q[:6], q[6:])[0] for q in q01])
    params = params.copy()  # move the proxy's decision onto the data: median (loop1) or below (loop2)
    params[-1] += np.float32(margin - np.median(prox) + (0.0 if case == "loop1" else -10.0))
    prox = np.array([O.predict_min_distance(w.program, params, cloud, q[:6], q[6:])[0] for q in q01])
    dist, _ = O.gcc(r, cloud, q01, steps=steps, margin=margin)
    want = _sequential_search(prox, dist, margin)
    got = gcc_nn_search(S.Model(w.program, params), r, cloud, q01, steps=steps, margin=margin, precision="fp32",
                        batch=7)
    print(case, want, {k: got[k] for k in ("found", "motion_index", "exact_checks", "nn_checks")})
    assert got["found"] == want[0] and got["motion_index"] == want[1]
    assert abs(got["certified_distance"] - want[2]) <= 1e-12
    assert got["exact_checks"] == want[3] and got["nn_checks"] == want[4]
    if case == "loop1":
        assert want[0] and want[4] < M  # certified inside the first loop
    if case == "loop2":
        assert want[0] and want[4] == M and (prox <= margin).all()
    if case == "none":
        assert not want[0]

"""Several GPUs from one process (svn_multi_*): motion shards and point shards
are bit-identical to one device; argument errors and unsupported layouts fail loudly.

The box behind gpurun has one GPU, so motion sharding runs with the same device listed
several times (one worker thread and one model copy each, concurrently), and point sharding
with one NCCL rank; the shard-then-combine arithmetic of several point shards is covered by
test_gpu_parity.py::test_point_sharded_keys_equal_unsharded and the gloo tests."""
import threading

import numpy as np
import pytest
import torch

import paper_2402_15281_b200 as S
from paper_2402_15281_b200.abi import ReferenceInvalidArgument, SvnError, UNSUPPORTED
from paper_2402_15281_b200.workloads import WORKLOADS

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert np.array_equal(a.min, b.min) and np.array_equal(a.argmin, b.argmin) and np.array_equal(a.free, b.free)


@pytest.mark.parametrize("key,prec", [("c3", "bf16"), ("c2", "fp32"), ("c2", "fp32_split"), ("c2", "bf16")])
@pytest.mark.parametrize("copies", [1, 2, 3])
def test_motion_shards_equal_one_device(key, prec, copies):
    w = WORKLOADS[key]
    params = S.init_params(w.program, 31, w.bound)
    pts, q = w.make(seed=31, motions=7, points=1500)
    ref = S.Model(w.program, params).query_min(pts, q, w.margin, precision=prec)
    mg = S.MultiModel(w.program, params, devices=[0] * copies)
    _same(mg.query_min(pts, q, w.margin, precision=prec, shard="motions"), ref)
    _same(mg.query_min(pts, q, w.margin, precision=prec, shard="auto"), ref)  # 7 motions >= devices
    mg.close()


@pytest.mark.parametrize("prec", ["bf16", "fp32_exact"])
def test_point_shard_one_rank_through_nccl(prec):
    w = WORKLOADS["c3"] if prec == "bf16" else WORKLOADS["c2"]
    params = S.init_params(w.program, 37, w.bound)
    pts, q = w.make(seed=37, motions=2, points=3000)
    ref = S.Model(w.program, params).query_min(pts, q, w.margin, precision=prec)
    mg = S.MultiModel(w.program, params, devices=[0])
    _same(mg.query_min(pts, q, w.margin, precision=prec, shard="points"), ref)
    # a one-motion batch on the single device, and the same through "auto"
    r1 = S.Model(w.program, params).query_min(pts, q[:1], w.margin, precision=prec)
    _same(mg.query_min(pts, q[:1], w.margin, precision=prec, shard="points"), r1)
    _same(mg.query_min(pts, q[:1], w.margin, precision=prec, shard="auto"), r1)


def test_point_shards_need_distinct_devices():
    w = WORKLOADS["c2"]
    params = S.init_params(w.program, 3, w.bound)
    pts, q = w.make(seed=3, motions=1, points=100)
    mg = S.MultiModel(w.program, params, devices=[0, 0])
    with pytest.raises(SvnError) as e:
        mg.query_min(pts, q, w.margin, precision="fp32", shard="points")
    assert e.value.status == UNSUPPORTED and "distinct devices" in str(e.value)
    with pytest.raises(SvnError):  # "auto" with 1 motion < 2 devices means points
        mg.query_min(pts, q, w.margin, precision="fp32", shard="auto")
    # with as many motions as devices "auto" shards motions, which a repeated device supports
    q2 = np.repeat(q, 2, axis=0)
    _same(mg.query_min(pts, q2, w.margin, precision="fp32", shard="auto"),
          S.Model(w.program, params).query_min(pts, q2, w.margin, precision="fp32"))


def test_multi_argument_errors_and_launch_count():
    w = WORKLOADS["c2"]
    params = S.init_params(w.program, 5, w.bound)
    pts, q = w.make(seed=5, motions=4, points=300)
    mg = S.MultiModel(w.program, params, devices=[0, 0])
    with pytest.raises(ReferenceInvalidArgument, match="empty point cloud"):
        mg.query_min(pts[:0], q, w.margin, precision="bf16", shard="motions")
    with pytest.raises(ReferenceInvalidArgument):
        S.MultiModel(w.program, params, devices=[torch.cuda.device_count()])
    S.launch_count_reset()
    mg.query_min(pts, q, w.margin, precision="bf16", shard="motions")
    assert S.launch_count() >= 4  # K0 + fused kernel on each worker, counted in the caller


def test_concurrent_callers_serialise():
    w = WORKLOADS["c2"]
    params = S.init_params(w.program, 9, w.bound)
    pts, q = w.make(seed=9, motions=9, points=800)
    ref = S.Model(w.program, params).query_min(pts, q, w.margin, precision="bf16")
    mg = S.MultiModel(w.program, params, devices=[0, 0, 0])
    out, errs = [], []

    def call():
        try:
            for _ in range(5):
                out.append(mg.query_min(pts, q, w.margin, precision="bf16", shard="motions"))
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ts = [threading.Thread(target=call) for _ in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs and len(out) == 20
    for r in out:
        _same(r, ref)


@pytest.mark.parametrize("key,prec", [("c3", "bf16"), ("c2", "fp32"), ("c2", "fp32_split")])
def test_resident_scene_equals_per_call_cloud(key, prec):
    """svn_multi_set_scene: the cloud uploaded once to every device, later calls pass
    points=None and move only motions in and results out — same bits as passing the cloud."""
    w = WORKLOADS[key]
    params = S.init_params(w.program, 41, w.bound)
    pts, q = w.make(seed=41, motions=9, points=2100)
    ref = S.Model(w.program, params).query_min(pts, q, w.margin, precision=prec)
    mg = S.MultiModel(w.program, params, devices=[0, 0, 0])
    with pytest.raises(ReferenceInvalidArgument, match="null buffer"):  # no scene yet
        mg.query_min(None, q, w.margin, precision=prec, shard="motions")
    mg.set_scene(pts)
    for _ in range(2):
        _same(mg.query_min(None, q, w.margin, precision=prec, shard="motions"), ref)
    _same(mg.query_min(None, q[2:3], w.margin, precision=prec, shard="motions"),  # fewer motions than devices
          S.Model(w.program, params).query_min(pts, q[2:3], w.margin, precision=prec))
    _same(mg.query_min(pts, q, w.margin, precision=prec, shard="motions"), ref)  # an explicit cloud still works
    # a second scene replaces the first
    pts2, _ = w.make(seed=43, motions=1, points=700)
    mg.set_scene(pts2)
    _same(mg.query_min(None, q, w.margin, precision=prec, shard="motions"),
          S.Model(w.program, params).query_min(pts2, q, w.margin, precision=prec))
    mg.set_scene(None)
    with pytest.raises(ReferenceInvalidArgument, match="null buffer"):
        mg.query_min(None, q, w.margin, precision=prec, shard="motions")
    mg.close()


def test_resident_scene_point_shards_one_rank():
    w = WORKLOADS["c3"]
    params = S.init_params(w.program, 47, w.bound)
    pts, q = w.make(seed=47, motions=2, points=3000)
    ref = S.Model(w.program, params).query_min(pts, q, w.margin, precision="bf16")
    mg = S.MultiModel(w.program, params, devices=[0])
    mg.set_scene(pts)
    _same(mg.query_min(None, q, w.margin, precision="bf16", shard="points"), ref)
    mg.close()

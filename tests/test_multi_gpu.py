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
    # 9 x 2100 is 81 big tiles (>= 74 pairs: 256-row tiles) while a 3-motion shard alone would run
    # 128-row tiles: the shards take the whole batch's shape, so `ref` is matched bit for bit
    with pytest.raises(ReferenceInvalidArgument):  # no scene yet: an empty cloud (P = 0)
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
    with pytest.raises(ReferenceInvalidArgument):
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


@pytest.mark.parametrize("key,prec", [("c3", "bf16"), ("c3", "fp16"), ("c2", "bf16"), ("c4", "bf16"), ("c3", "fp32_split")])
def test_shards_take_the_whole_batch_tile_shape(key, prec):
    """A launch with fewer 256-row tiles than CTA pairs runs 128-row tiles, whose output dot
    sums in another order (~1e-6).  Declared as shards of the whole batch (svn_set_whole_batch),
    motion ranges and point chunks give the whole batch's bits; svn_query_min_multi does so itself."""
    w = WORKLOADS[key]
    params = S.init_params(w.program, 41, w.bound)
    pts, q = w.make(seed=41, motions=9, points=2100)  # 81 big tiles; 3 motions alone: 27
    m = S.Model(w.program, params)
    ref = m.query_min(pts, q, w.margin, precision=prec)
    with S.whole_batch(9, 2100):
        parts = [m.query_min(pts, q[i:i + 3], w.margin, precision=prec) for i in (0, 3, 6)]
    assert np.array_equal(np.concatenate([p.min for p in parts]), ref.min)
    assert np.array_equal(np.concatenate([p.argmin for p in parts]), ref.argmin)
    # the setting is cleared on exit: a later small call runs its own shape again
    alone = m.query_min(pts, q[:3], w.margin, precision=prec)
    bound = 1e-5 if prec == "fp32_split" else 1e-4
    assert np.abs(alone.min.astype(np.float64) - ref.min[:3]).max() <= bound
    # point chunks through the keys entry points
    import torch
    from paper_2402_15281_b200 import parallel
    dev = torch.device("cuda", 0)
    qd = torch.from_numpy(q).to(dev)
    keys = torch.empty(9, dtype=torch.int64, device=dev)
    S.keys_init_device(keys)
    with S.whole_batch(9, 2100):
        for b in range(0, 2100, 700):
            m.query_keys_device(torch.from_numpy(np.ascontiguousarray(pts[b:b + 700])).to(dev), b, qd, keys, precision=prec)
    mn = torch.empty(9, dtype=torch.float32, device=dev)
    am = torch.empty(9, dtype=torch.int32, device=dev)
    fr = torch.empty(9, dtype=torch.uint8, device=dev)
    S.keys_finalize_device(keys, w.margin, mn, am, fr)
    torch.cuda.synchronize()
    assert np.array_equal(mn.cpu().numpy(), ref.min) and np.array_equal(am.cpu().numpy(), ref.argmin)
    # and the box: three workers, three motions each
    mg = S.MultiModel(w.program, params, devices=[0, 0, 0])
    _same(mg.query_min(pts, q, w.margin, precision=prec, shard="motions"), ref)
    mg.close()


def test_point_shard_large_chunk_is_piped_and_bit_identical():
    """A worker's point chunk of >= 2^21 points travels in 2^20-point pieces on a second stream
    while the pieces already on the device are folded into the keys: same bits as one device."""
    w = WORKLOADS["c3"]
    params = S.init_params(w.program, 53, w.bound)
    pts, q = w.make(seed=53, motions=2, points=(1 << 21) + 5000)
    ref = S.Model(w.program, params).query_min(pts, q, w.margin, precision="bf16")
    mg = S.MultiModel(w.program, params, devices=[0])
    _same(mg.query_min(pts, q, w.margin, precision="bf16", shard="points"), ref)
    mg.set_scene(pts)
    _same(mg.query_min(None, q, w.margin, precision="bf16", shard="points"), ref)
    mg.close()


def test_parallel_point_sharded_query_pipes_a_large_chunk():
    """parallel.point_sharded_query (the torchrun path): a chunk of >= 2^21 points is uploaded in
    2^20-point pieces on a side stream and folded piece by piece — same bits as one call."""
    import torch
    from paper_2402_15281_b200 import parallel
    w = WORKLOADS["c3"]
    params = S.init_params(w.program, 59, w.bound)
    pts, q = w.make(seed=59, motions=2, points=(1 << 21) + 777)
    model = S.Model(w.program, params)
    ref = model.query_min(pts, q, w.margin, precision="bf16")
    dev = torch.device("cuda", 0)
    qd = torch.from_numpy(q).to(dev)
    for host in (pts, torch.from_numpy(pts).pin_memory().numpy()):  # pageable and pinned callers
        mn, am, fr = parallel.point_sharded_query(model, host, qd, w.margin, 1, 0, precision="bf16", device=dev)
        torch.cuda.synchronize()
        assert np.array_equal(mn.cpu().numpy(), ref.min) and np.array_equal(am.cpu().numpy(), ref.argmin)
        assert np.array_equal(fr.cpu().numpy().astype(bool), ref.free)

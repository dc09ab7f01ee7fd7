"""CPU tests of the multi-GPU host logic (world_size 2, gloo): shard ranges, the packed
(delta, index) key algebra, and the MIN all-reduce with the u64->int64 order remap.
The per-shard compute here is the oracle; on the GPU it is svn_query_min_keys_device."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2402_15281_b200 as S
from oracle import oracle as O
from paper_2402_15281_b200.parallel import decode_keys_np, pack_keys_np, shard_range
from paper_2402_15281_b200.workloads import WORKLOADS


def test_shard_range_partitions():
    for n in (0, 1, 7, 64, 1000, 2**24):
        for w in (1, 2, 3, 4, 8):
            parts = [shard_range(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, d) in zip(parts[:-1], parts[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in parts if b > a]
            assert not sizes or max(sizes) - min(sizes) <= (n + w - 1) // w


def _reference_min(vals):
    """nn.cpp:476-478 argmin: best=0, strict '<'."""
    best = 0
    for i in range(1, len(vals)):
        if vals[i] < vals[best]:
            best = i
    return vals[best], best


@pytest.mark.parametrize("case", ["random", "ties", "nan0", "nan_mid", "negzero", "inf"])
def test_key_min_matches_reference_argmin(case):
    rng = np.random.default_rng(0)
    v = rng.normal(size=1000).astype(np.float32)
    if case == "ties":
        v = np.round(v, 1).astype(np.float32)
        v[[10, 20, 500]] = v.min()
    if case == "nan0":
        v[0] = np.nan
    if case == "nan_mid":
        v[[3, 700]] = np.nan
    if case == "negzero":
        v = np.abs(v)
        v[5], v[9] = np.float32(-0.0), np.float32(0.0)
    if case == "inf":
        v[42] = -np.inf
    keys = pack_keys_np(v, np.arange(v.size))
    mn, am, fr = decode_keys_np(keys.min(keepdims=True), 0.0)
    rv, ri = _reference_min(list(v))
    assert am[0] == ri
    assert (np.isnan(mn[0]) and np.isnan(rv)) or mn[0] == rv
    # sharded min of mins == global min (any split)
    for cut in (1, 333, 999):
        k2 = min(keys[:cut].min(), keys[cut:].min())
        assert k2 == keys.min()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    from paper_2402_15281_b200.parallel import allreduce_keys_min
    w = WORKLOADS["c2"]
    params = S.init_params(w.program, 5, "he")
    pts, q = w.make(seed=5, motions=3, points=900)
    pts[0] = np.nan  # exercise the NaN-at-index-0 rule on motion rows through the shard boundary
    # point sharding: this rank's points, global indices
    b, e = shard_range(pts.shape[0], world, rank)
    _, _, _, pp = O.query_min(w.program, params, pts[b:e], q, w.margin, per_point=True)
    keys = np.stack([pack_keys_np(pp[m], np.arange(b, e)).min() for m in range(q.shape[0])])
    t = torch.from_numpy(keys.view(np.int64).copy())
    allreduce_keys_min(t)
    mn, am, fr = decode_keys_np(t.numpy().view(np.uint64), w.margin)
    # motion sharding: this rank's motions
    mb, me = shard_range(q.shape[0], world, rank)
    mres = O.query_min(w.program, params, pts, q[mb:me], w.margin)
    gathered = [None] * world
    dist.all_gather_object(gathered, (mb, me, [x.tolist() for x in mres[:3]]))
    if rank == 0:
        result_q.put((mn.tolist(), am.tolist(), fr.tolist(), gathered))
    dist.destroy_process_group()


def test_world2_gloo_point_and_motion_sharding_equal_unsharded():
    w = WORKLOADS["c2"]
    params = S.init_params(w.program, 5, "he")
    pts, q = w.make(seed=5, motions=3, points=900)
    pts[0] = np.nan
    omin, oarg, ofree, _ = O.query_min(w.program, params, pts, q, w.margin, per_point=True)
    ctx = mp.get_context("spawn")
    qout = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, qout)) for r in range(2)]
    for p in procs:
        p.start()
    res = qout.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    mn, am, fr, gathered = res
    assert am == oarg.tolist() and fr == ofree.tolist()
    assert all((np.isnan(a) and np.isnan(b)) or a == b for a, b in zip(mn, omin.tolist()))
    # motion shards concatenate to the unsharded result
    cat_min = sum((g[2][0] for g in sorted(gathered)), [])
    cat_arg = sum((g[2][1] for g in sorted(gathered)), [])
    assert cat_arg == oarg.tolist()
    assert all((np.isnan(a) and np.isnan(b)) or a == b for a, b in zip(cat_min, omin.tolist()))

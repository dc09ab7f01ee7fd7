"""Multi-GPU sharding of the hot path.  One process per GPU.

Motion sharding (default): motions are independent (per-motion min, no cross-motion
state — nn.cpp:460-480), so rank r evaluates the contiguous motion range
shard_range(M, world, r) against the full cloud.  There is no data-path
collective; results are bit-identical to a 1-GPU run.

Point sharding (single-motion batches, e.g. 1 motion x 2^24 points): rank r
evaluates points shard_range(P, world, r) and folds its rows into per-motion
packed keys  (orderable(delta) << 32) | global_point_index.  One MIN all-reduce of
8 bytes per motion (NCCL over NVLink) combines the shards; the lowest-index
tie-break and the NaN-at-index-0 rule of nn.cpp:476-478 hold by construction,
so the result is bit-identical to 1 GPU.

The collective runs on u64 keys through torch.distributed's signed int64 MIN:
flipping bit 63 maps unsigned order onto signed order (key ^ 2^63).
"""
from __future__ import annotations

import numpy as np

SIGN = np.int64(-(2 ** 63))  # bit 63 as an int64


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous near-equal partition (parallel.cpp:33-41 style: ceil chunks)."""
    chunk = (n + world - 1) // world
    b = min(n, rank * chunk)
    e = min(n, b + chunk)
    return b, e


# --------------------------------------------------------------- key algebra --
def orderable_np(delta: np.ndarray) -> np.ndarray:
    """Host mirror of svn::orderable (fused.cuh): float -> u32 with unsigned order == float order."""
    u = np.asarray(delta, np.float32).view(np.uint32).astype(np.uint64)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    u = np.where(u == 0x80000000, 0, u)
    o = np.where(u & 0x80000000, (~u) & 0xFFFFFFFF, u | 0x80000000)
    return np.where(nan, 0xFFFFFFFF, o).astype(np.uint64)


def pack_keys_np(delta: np.ndarray, index: np.ndarray) -> np.ndarray:
    """Host mirror of svn::row_key: u64 keys; NaN at global index 0 -> key 0."""
    delta = np.asarray(delta, np.float32)
    index = np.asarray(index, np.uint64)
    k = (orderable_np(delta) << np.uint64(32)) | index
    return np.where(np.isnan(delta) & (index == 0), np.uint64(0), k).astype(np.uint64)


def decode_keys_np(keys: np.ndarray, margin: float):
    """Host mirror of svn::decode_key -> (min float32, argmin int32, free bool)."""
    keys = np.asarray(keys, np.uint64)
    hi = (keys >> np.uint64(32)).astype(np.uint64)
    idx = (keys & np.uint64(0xFFFFFFFF)).astype(np.int64).astype(np.int32)
    u = np.where(hi & 0x80000000, hi & 0x7FFFFFFF, (~hi) & 0xFFFFFFFF).astype(np.uint32)
    v = u.view(np.float32).copy()
    nan = (keys == 0) | (hi == 0xFFFFFFFF)
    v[nan] = np.nan
    idx[keys == 0] = 0
    return v, idx, v.astype(np.float64) > margin


def to_signed(keys_u64):
    """u64 keys (stored in an int64 tensor or array) -> int64 whose signed order is the u64 order."""
    return keys_u64 ^ int(SIGN) if hasattr(keys_u64, "bitwise_xor") else keys_u64 ^ SIGN


def allreduce_keys_min(keys, group=None):
    """MIN all-reduce of packed u64 keys held in an int64 torch tensor (in place)."""
    import torch.distributed as dist
    keys.bitwise_xor_(int(SIGN))
    dist.all_reduce(keys, op=dist.ReduceOp.MIN, group=group)
    keys.bitwise_xor_(int(SIGN))
    return keys


PIECE_POINTS = 1 << 20  # point_sharded_query: upload granularity of a large chunk

# ------------------------------------------------------------- GPU drivers ---
def motion_sharded_query(model, points, q01, margin, world: int, rank: int, precision="bf16", stream=None):
    """This rank's motion shard on its GPU; returns (motion_begin, min, argmin, free) device tensors."""
    import torch
    M = q01.shape[0]
    b, e = shard_range(M, world, rank)
    dev = points.device
    n = max(0, e - b)
    mn = torch.empty(n, dtype=torch.float32, device=dev)
    am = torch.empty(n, dtype=torch.int32, device=dev)
    fr = torch.empty(n, dtype=torch.uint8, device=dev)
    if n:
        from .api import whole_batch
        with whole_batch(M, points.shape[0]):  # the whole batch's tile shape: same bits for every world size
            model.query_min_device(points, q01[b:e].contiguous(), margin, mn, am, fr, None, precision=precision,
                                   stream=stream)
    return b, mn, am, fr


def point_sharded_query(model, points_full_host: np.ndarray, q01, margin, world: int, rank: int,
                        precision="bf16", group=None, stream=None, device=None):
    """Point-chunk sharding with one NCCL MIN all-reduce of 8 B per motion.
    points_full_host: float32 [P, 3] (each rank uploads only its chunk)."""
    import torch
    from .api import keys_finalize_device, keys_init_device, whole_batch
    P = points_full_host.shape[0]
    b, e = shard_range(P, world, rank)
    dev = device or q01.device
    M = q01.shape[0]
    keys = torch.empty(M, dtype=torch.int64, device=dev)
    keys_init_device(keys, stream=stream)
    if e - b >= 2 * PIECE_POINTS and torch.device(dev).type == "cuda":
        # a large chunk travels in pieces on a side stream while the compute stream folds the
        # pieces already on the device into the keys (bit-identical: min over packed keys)
        cur = stream if stream is not None else torch.cuda.current_stream(dev)
        side = torch.cuda.Stream(device=dev)
        buf = torch.empty((e - b, 3), dtype=torch.float32, device=dev)
        buf.record_stream(side)
        side.wait_stream(cur)
        with whole_batch(M, P):
            for p0 in range(0, e - b, PIECE_POINTS):
                n = min(PIECE_POINTS, e - b - p0)
                src = torch.from_numpy(np.ascontiguousarray(points_full_host[b + p0:b + p0 + n]))
                with torch.cuda.stream(side):
                    buf[p0:p0 + n].copy_(src, non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(side)
                cur.wait_event(ev)
                model.query_keys_device(buf[p0:p0 + n], b + p0, q01, keys, precision=precision, stream=stream)
    elif e > b:
        pts = torch.from_numpy(np.ascontiguousarray(points_full_host[b:e])).to(dev)
        with whole_batch(M, P):
            model.query_keys_device(pts, b, q01, keys, precision=precision, stream=stream)
    if world > 1:
        allreduce_keys_min(keys, group)
    mn = torch.empty(M, dtype=torch.float32, device=dev)
    am = torch.empty(M, dtype=torch.int32, device=dev)
    fr = torch.empty(M, dtype=torch.uint8, device=dev)
    keys_finalize_device(keys, margin, mn, am, fr, stream=stream)
    return mn, am, fr

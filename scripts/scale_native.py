"""Scaling of the single-process multi-GPU path (svn_query_min_multi, one worker thread per
GPU) over the GPUs of this box: weak scaling of motion shards (c3's per-GPU size per device)
and strong scaling of point shards (c5single: one motion, 2^24 points, one NCCL MIN
all-reduce; also against the resident scene).  Host buffers in, results out (the e2e contract of svn_query_min); wall time of
the synchronous call, median of a few calls.  python scripts/scale_native.py [--max-gpus N]"""
import argparse
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2402_15281_b200 as S  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402


def timed(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-gpus", type=int, default=torch.cuda.device_count())
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    counts = [n for n in (1, 2, 4, 8) if n <= args.max_gpus]
    base = None
    for n in counts:
        w = WORKLOADS["c3"]
        params = S.init_params(w.program, 0, w.bound)
        pts, q = w.make(seed=0, motions=w.motions * n)  # weak: c3's 1024 motions per GPU
        mg = S.MultiModel(w.program, params, devices=list(range(n)))
        sec = timed(lambda: mg.query_min(pts, q, w.margin, precision="bf16", shard="motions"), args.reps)
        qps = q.shape[0] * pts.shape[0] / sec
        base = base or qps
        print(json.dumps({"mode": "motions (weak)", "n_gpus": n, "queries_per_s": qps, "seconds": sec,
                          "efficiency_vs_1": qps / (base * n)}), flush=True)
        mg.close()
    base = base_res = None
    for n in counts:
        w = WORKLOADS["c5single"]
        params = S.init_params(w.program, 0, w.bound)
        pts, q = w.make(seed=0)
        mg = S.MultiModel(w.program, params, devices=list(range(n)))
        sec = timed(lambda: mg.query_min(pts, q, w.margin, precision="bf16", shard="points"), args.reps)
        qps = pts.shape[0] / sec
        base = base or qps
        print(json.dumps({"mode": "points (strong)", "n_gpus": n, "queries_per_s": qps, "seconds": sec,
                          "speedup_vs_1": qps / base}), flush=True)
        # the same against the scene kept resident on the devices (svn_multi_set_scene)
        mg.set_scene(pts)
        sec = timed(lambda: mg.query_min(None, q, w.margin, precision="bf16", shard="points"), args.reps)
        base_res = base_res or pts.shape[0] / sec
        print(json.dumps({"mode": "points (strong), resident scene", "n_gpus": n, "queries_per_s": pts.shape[0] / sec,
                          "seconds": sec, "speedup_vs_1": pts.shape[0] / sec / base_res}), flush=True)
        mg.close()


if __name__ == "__main__":
    main()

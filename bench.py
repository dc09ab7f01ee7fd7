#!/usr/bin/env python3
"""bench.py — point x motion SDF queries/s of the swept-volume proxy hot path.

One step = one pass of the hot path over one batch: every (point x motion) pair of
the workload through the fused MLP, per-motion min/argmin and the margin class.

Default workload (N=1): BASELINE.json configs[4] ("c5"), the config the metric's
1/2/4/8-GPU sweep is quoted on: DeepSDF 8x512 concat@4, bf16 with fp32 accumulate,
32768 motions x 262144 points (~21 s per step on one B200).  Other configs:
--config c1|c2|c3|c4|c5single|paper.  configs[1] ("c2") states fp32 weights: its FP32
path runs in the reference's order on FFMA (bit-identical) and `--precision fp32_split`
runs it fp32-grade on tcgen05.

--gpus N (strong scaling): the FIXED workload is split over N ranks, one process per
GPU — by motion (contiguous motion ranges, no data-path collective) when the workload
has at least N motions, else by point chunk (one 8-byte-per-motion NCCL MIN
all-reduce of packed keys).  Launched by torchrun, or — without torchrun — bench.py
re-launches itself under torch.distributed.run with N ranks; a world size that
differs from --gpus aborts.

Timing: W warm-up steps, then K steps bracketed by barrier + synchronize; device
time from CUDA events on the launching stream, max over ranks.  L2 is flushed
(a 256 MiB write, outside the per-step events) before every timed step.  Clocks are
sampled by nvidia-smi every 100 ms over the timed region, extended with untimed steps
to at least 1 s when the K steps are shorter.
`--impl reference` times the reference CPU path on a bounded sample of the same workload,
on all host threads: the reference's own nn.cpp as built by oracle/ref into oracle/_ref
(predict_min_distance per motion from worker threads) on the Fig. 2 twin of the config's
network — the only architecture the reference implements — with the C restatement on the
config's own network alongside (and alone when oracle/_ref is absent); it loads nothing
from the product package's native library.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "point x motion SDF queries/sec"
UNIT = "queries/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--precision", default=None, help="override: bf16 | fp16 | fp32 | fp32_exact | fp32_split")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--motions", type=int, default=None, help="experiment override (not a BASELINE config)")
    ap.add_argument("--points", type=int, default=None, help="experiment override (not a BASELINE config)")
    ap.add_argument("--mode", default=None, choices=["motion", "point"],
                    help="multi-GPU sharding override: motion or point")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.tmp = None
        self.t0 = None

    def __enter__(self):
        self.t0 = time.perf_counter()
        try:
            self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.tmp, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def elapsed(self) -> float:
        return time.perf_counter() - self.t0

    def __exit__(self, *exc):
        self.window_s = self.elapsed()
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.proc is None or self.tmp is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.tmp.flush()
        rows = []
        for line in Path(self.tmp.name).read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.tmp.name)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [s for s in sm if smax and s > 0.5 * max(smax)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons, "samples": len(rows),
                "window_s": round(getattr(self, "window_s", 0.0), 3)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def build_native_oracle():
    """The reference builds with -O3 -march=native (proj/CMakeLists.txt:31-38): rebuild the
    oracle that way on this host for the timed CPU baseline."""
    from oracle import oracle as O
    out = Path(tempfile.mkdtemp(prefix="svn_oracle_"))
    try:
        return O.lib(O.build(march="native", out=out)), "native"
    except Exception:
        return O.lib(), "x86-64-v3"


def cpu_sample(w, threads, seconds=10.0):
    """Bounded sample of the workload for the CPU path: `threads` motions x a point count
    sized for ~`seconds` of CPU work (the oracle runs ~1.4e10 FLOP/s per core here)."""
    fq = w.program.flops_per_query()
    budget = 1.4e10 * seconds * max(1, threads)  # FLOPs for the whole sample
    M = max(1, min(w.motions, threads))
    per_motion = int(max(256, min(w.points, budget / M / fq)))
    return M, per_motion


def run_cpu(w, params, seed, threads, lib, steps, warmup, seconds=10.0):
    """Times the oracle on the bounded sample; returns (queries/s, description, sample, outputs)."""
    from oracle import oracle as O
    M, P = cpu_sample(w, threads, seconds)
    pts, q = w.make(seed=seed, motions=M, points=P)
    times = []
    res = None
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        res = O.query_min(w.program, params, pts, q, w.margin, threads=threads, library=lib)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    sec = statistics.median(times)
    run_cpu.last_ms = sec * 1e3
    return (M * P / sec, f"{M} motions x {P} points of {w.key} ({M * P} queries), {len(times)} runs, median",
            (pts, q), res)


def reference_build_leg(w, seed, threads, seconds=8.0, repeats=1):
    """The reference's OWN nn.cpp (oracle/_ref/libref_nn.so: compiled unmodified here against the
    Eigen-API subset, -O3 -march=x86-64-v3) on the same cloud and motions, one
    predict_min_distance call per motion from `threads` worker threads (bench.cpp:156,193).  The
    reference implements the Fig. 2 architecture only (nn.hpp:16-42), so it runs the Fig. 2
    twin of the workload's network (same width and dof, hidden - 1 blocks);
    the port runs the same twin next to it, and their bits are compared.  None when the
    prebuilt library did not travel with the repo."""
    try:
        from oracle import oracle as O
        from oracle import ref_oracle as R
        from paper_2402_15281_b200 import program as PR
        if not R.available():
            return None
        prog = w.program
        twin = prog if prog.name.startswith("fig2") else PR.fig2(len(prog.layers) - 1, prog.width, prog.dof)
        M, P = cpu_sample(w, threads, seconds)
        pts, q = w.make(seed=seed, motions=M, points=P)
        with tempfile.TemporaryDirectory(prefix="svn_ref_") as d:
            ck = str(Path(d) / "twin.ckpt")
            params = R.init_model(len(twin.layers) - 1, twin.width, twin.dof, seed, ck)
            secs = []
            for _ in range(max(1, repeats)):
                mn, idx, sec = R.time_predict_min_distance(ck, pts, q, threads)
                secs.append(sec)
            sec = statistics.median(secs)
        t0 = time.perf_counter()
        omin, oarg, _, _ = O.query_min(twin, params, pts, q, w.margin, threads=threads)
        port_sec = time.perf_counter() - t0
        return {"value": M * P / sec, "unit": UNIT, "cores": threads, "kind": "reference", "ms_per_sample": sec * 1e3,
                "network": f"{twin.name} (Fig. 2 twin of {prog.name})" if twin is not prog else twin.name,
                "flop_per_query": twin.flops_per_query(),
                "sample": f"{M} motions x {P} points ({M * P} queries), predict_min_distance per motion "
                          f"(nn.cpp:460-480) on {threads} threads; reference nn.cpp built -O3 -march=x86-64-v3 "
                          f"against the Eigen-API subset (oracle/ref)",
                "port_on_same_network": {"value": M * P / port_sec, "unit": UNIT,
                                         "bits_equal": bool(np.array_equal(omin.astype(np.float64), mn)
                                                            and np.array_equal(oarg, idx))}}
    except Exception as e:  # the baseline leg must not take the bench line down
        return {"unavailable": f"{type(e).__name__}: {e}"}


def bounds_for(network: str, prec: str):
    g = ROOT / "tests" / "golden"
    f = g / f"{prec}_bounds.json"
    if prec not in ("bf16", "fp16", "fp32_split") or not f.exists():
        return 0.0
    d = json.loads(f.read_text())
    return float(d[network]["bound"]) if network in d else None


def class_compare(mn_a, fr_a, am_a, mn_ref, fr_ref, am_ref, margin, bound):
    amb = np.abs(mn_ref.astype(np.float64) - margin) <= bound
    mism = fr_a != fr_ref
    return {"motions": int(mn_ref.size), "max_abs_min_err": float(np.max(np.abs(mn_a.astype(np.float64) - mn_ref))),
            "class_mismatches": int(mism.sum()), "ambiguous": int(amb.sum()),
            "mismatches_outside_band": int((mism & ~amb).sum()), "argmin_equal": int((am_a == am_ref).sum()),
            "free_fraction_ref": float(fr_ref.mean())}


def reference_arm(args, w):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O  # the reference arm loads no product code
    params = O.init_params(w.program, args.seed, w.bound)
    threads = os.cpu_count() or 1
    lib, march = build_native_oracle()
    steps, warm = max(1, args.steps), max(0, min(args.warmup, 1))
    per_step = max(2.0, min(10.0, 120.0 / (steps + warm)))  # whole arm within ~2 minutes
    val, sample, _, _ = run_cpu(w, params, args.seed, threads, lib, steps, warm, per_step)
    med_ms = getattr(run_cpu, "last_ms", None)
    # the reference's own call is single-threaded (nn.cpp:116): one thread, ~5 s sample
    v1, s1, _, _ = run_cpu(w, params, args.seed, 1, lib, 1, 0, 5.0)
    ref_build = reference_build_leg(w, args.seed, threads, per_step, repeats=min(steps, 3))
    port = {"value": val, "unit": UNIT, "cores": threads, "kind": "port", "network": w.program.name,
            "sample": sample + f"; oracle restatement of nn.cpp:95-130 (-O3 -march={march}), "
                               f"{threads} threads on {cpu_model()}",
            "single_thread": {"value": v1, "unit": UNIT, "cores": 1, "sample": s1}}
    if ref_build and "value" in ref_build:
        # the reference's own code compiled here is the arm's number (on the Fig. 2 twin, the only
        # architecture it implements); the port on the config's own network rides along
        head, head_ms = dict(ref_build, port=port), ref_build["ms_per_sample"]
    else:
        head, head_ms = dict(port, reference_build=ref_build), med_ms
    line = {"metric": METRIC, "value": head["value"], "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head_ms,
            "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded)",
            "config": {"workload": w.key, "description": w.description, "network": w.program.name,
                       "reference_network": head.get("network", w.program.name)},
            "cpu_baseline": head,
            "e2e": {"value": head["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def relaunch_under_torchrun(args) -> int:
    """`bench.py --gpus N` without torchrun: run this same command as N ranks."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    world, rank, local = dist_env()
    from paper_2402_15281_b200.workloads import WORKLOADS
    w = WORKLOADS[args.config]
    if args.motions or args.points:
        import dataclasses
        w = dataclasses.replace(w, key=w.key + "-override", motions=args.motions or w.motions,
                                points=args.points or w.points)
    prec = args.precision or w.precision
    peaks, peak_src = load_peaks()

    if args.impl == "reference":
        return reference_arm(args, w)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; refusing to report a mislabelled run",
              file=sys.stderr)
        return 2

    import torch
    import torch.distributed as dist
    import paper_2402_15281_b200 as S

    # SVN_BENCH_BACKEND / SVN_BENCH_DEVICE exist only to exercise the multi-rank code path
    # on a one-GPU box (gloo, every rank on device 0); production runs use NCCL, rank = GPU.
    backend = os.environ.get("SVN_BENCH_BACKEND", "nccl")
    local = int(os.environ.get("SVN_BENCH_DEVICE", local))
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    # ---- workload (fixed, split over ranks), resident in HBM ------------------
    # motion mode: rank r evaluates motions shard_range(M, world, r) against the full
    #   cloud; no collective.
    # point mode (fewer motions than ranks): rank r evaluates points
    #   shard_range(P, world, r); one NCCL MIN all-reduce of 8 B per motion per step.
    from paper_2402_15281_b200.parallel import allreduce_keys_min, shard_range
    mode = args.mode or ("motion" if w.motions >= world else "point")
    M_total, P = w.motions, w.points
    if mode == "motion":
        mb, me = shard_range(M_total, world, rank)
        pts_np, q_np = w.make(seed=args.seed, motions=me - mb, motion_offset=mb)
        pb, pe = 0, P
    else:
        mb, me = 0, M_total
        pts_np, q_np = w.make(seed=args.seed)
        pb, pe = shard_range(P, world, rank)
    M = me - mb
    params = S.init_params(w.program, args.seed, w.bound)
    model = S.Model(w.program, params, device=local)
    pts = torch.from_numpy(np.ascontiguousarray(pts_np[pb:pe])).to(dev)
    q = torch.from_numpy(q_np).to(dev)
    mn = torch.empty(M, dtype=torch.float32, device=dev)
    am = torch.empty(M, dtype=torch.int32, device=dev)
    fr = torch.empty(M, dtype=torch.uint8, device=dev)
    keys = torch.empty(M, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        if mode == "motion":
            model.query_min_device(pts, q, w.margin, mn, am, fr, None, precision=prec, stream=stream)
        else:
            S.keys_init_device(keys, stream=stream)
            model.query_keys_device(pts, pb, q, keys, precision=prec, stream=stream)
            if world > 1:
                allreduce_keys_min(keys)
            S.keys_finalize_device(keys, w.margin, mn, am, fr, stream=stream)

    # every rank runs the tile shape of the whole (fixed) workload — the same bits at every N
    # (svn_set_whole_batch; set once for the warm-up and timed steps, cleared before the other legs)
    shards = S.whole_batch(M_total, P)
    if world > 1:
        shards.__enter__()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    S.launch_count_reset()
    S.kernel_timing_begin()
    extra_steps = 0
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        launches = S.launch_count()
        k_ms, k_n = S.kernel_timing_end()
        # clock record over >= 1 s: keep the same load running (untimed) when K steps were shorter
        while clocks.elapsed() < 1.0:
            step()
            torch.cuda.synchronize(dev)
            extra_steps += 1
    if world > 1:
        shards.__exit__(None, None, None)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = sum(step_ms) / len(step_ms)
    kernel_ms = k_ms / max(1, k_n)
    if world > 1:
        t = torch.tensor([ms, kernel_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kernel_ms = float(t[0]), float(t[1])
    total_queries = M_total * P
    value = total_queries / (ms * 1e-3)

    # ---- roofline of the dominant kernel (the fused MLP) ----------------------
    flop_q = w.program.flops_per_query()
    achieved_tf = M * (pe - pb) * flop_q / (kernel_ms * 1e-3) / 1e12
    if prec in ("bf16", "fp16"):  # fp16 operands run at the same kind::f16 instruction rate
        peak = float(peaks["bf16_tflops"])
        roof = {"bound": "tensor", "achieved": achieved_tf, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved_tf / peak, "traffic": None,
                "peak_source": f"{peak_src} bf16_tflops (burst)",
                "frac_of_sustained": achieved_tf / float(peaks.get("bf16_tflops_sustained", peak)),
                "flop_per_query": flop_q, "kernel_ms": kernel_ms}
    elif prec == "fp32_split":
        # fp32-accurate on tcgen05: every product is three f16 MMAs (hi.hi, hi.lo', lo'.hi), so
        # the algorithmic-FLOP ceiling of the scheme is the measured f16/bf16 peak / 3.
        peak = float(peaks["bf16_tflops"]) / 3.0
        roof = {"bound": "tensor", "achieved": achieved_tf, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved_tf / peak, "traffic": None,
                "peak_source": f"{peak_src} bf16_tflops / 3 (split-fp16: 3 tensor products per fp32 product)",
                "flop_per_query": flop_q, "kernel_ms": kernel_ms}
    else:
        formula = 148 * 128 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
        fp = ROOT / "profiles" / "fp32_peak.json"
        if fp.exists():  # MEASURED_PEAKS.json has no FP32 figure: the highest FP32 FMA rate measured
            peak = float(json.loads(fp.read_text())["ffma_tflops"])  # on the box (packed FFMA2 tile)
            src = "measured FP32 peak: FFMA2 register-tile microbenchmark (profiles/fp32_peak.json)"
        else:
            peak, src = formula, "formula 148 SM x 128 FFMA lanes x 2 x sm_max_mhz"
        roof = {"bound": "fp32-simt", "achieved": achieved_tf, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved_tf / peak, "traffic": None, "peak_source": src,
                "frac_of_formula": achieved_tf / formula, "flop_per_query": flop_q, "kernel_ms": kernel_ms}
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        try:
            tr = json.loads(prof.read_text()).get(f"{w.key}:{prec}")
            if tr:
                roof["traffic"] = tr.get("dram_bytes_per_launch")
                roof["traffic_source"] = tr.get("source")
        except Exception:
            pass

    # ---- e2e through the public host API (host buffers, copies inside) --------
    e2e = None
    if not args.no_e2e and mode == "motion":
        hp = torch.from_numpy(pts_np).pin_memory().numpy()
        hq = torch.from_numpy(q_np).pin_memory().numpy()
        # warm the host path (staging block, scratch arena sized by the previous call): the full batch
        # when a step takes under 2 s (a first full-size call was seen to cost up to ~0.1 s extra), a few
        # motions of it when a step takes longer
        model.query_min(hp, hq if ms < 2000 else hq[: min(M, 8)], w.margin, precision=prec)
        n_e = 1 if ms > 2000 else max(1, min(args.steps, 3))
        if world > 1:
            dist.barrier()
        t_e = []
        for _ in range(n_e):
            t0 = time.perf_counter()
            model.query_min(hp, hq, w.margin, precision=prec)
            t_e.append(time.perf_counter() - t0)
        e_ms = statistics.mean(t_e) * 1e3
        # the reference's callers pass pageable std::vector memory: the staging-copy path
        t0 = time.perf_counter()
        model.query_min(pts_np, q_np, w.margin, precision=prec)
        pg_ms = (time.perf_counter() - t0) * 1e3
        if world > 1:
            t = torch.tensor([e_ms, pg_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms, pg_ms = float(t[0]), float(t[1])
        e2e = {"value": total_queries / (e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(hp.nbytes + hq.nbytes),
               "d2h_bytes_per_step": int(M * (4 + 4 + 1)), "ms_per_step": e_ms, "steps": n_e,
               "ms_samples": [round(t * 1e3, 3) for t in t_e],
               "api": "svn_query_min (C-ABI, pinned host buffers)",
               "pageable": {"value": total_queries / (pg_ms * 1e-3), "ms_per_step": pg_ms,
                            "api": "svn_query_min (C-ABI, pageable host buffers: staged copy)"}}

    elif not args.no_e2e:
        # point mode: every rank copies ITS point chunk and the motions from pinned host memory,
        # folds the chunk into the keys, the ranks meet in the MIN all-reduce, and rank 0's
        # (min, argmin, free) come back to the host — all inside the timed region
        from paper_2402_15281_b200.parallel import point_sharded_query
        hfull = torch.from_numpy(pts_np).pin_memory().numpy()  # each rank reads only its chunk of it
        hq = torch.from_numpy(q_np).pin_memory()
        hchunk = hfull[pb:pe]

        def e_step():
            dq = hq.to(dev, non_blocking=True)
            r = point_sharded_query(model, hfull, dq, w.margin, world, rank, precision=prec, stream=stream, device=dev)
            return tuple(t.cpu() for t in r)

        e_step()
        n_e = 1 if ms > 2000 else max(1, min(args.steps, 3))
        t_e = []
        for _ in range(n_e):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            e_step()
            t_e.append(time.perf_counter() - t0)
        e_ms = statistics.mean(t_e) * 1e3
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t[0])
        e2e = {"value": total_queries / (e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(hchunk.size * 4 + hq.numel() * 4), "d2h_bytes_per_step": int(M * (4 + 4 + 1)),
               "ms_per_step": e_ms, "steps": n_e,
               "api": "parallel.point_sharded_query: svn_query_min_keys_device + u64 MIN all-reduce + "
                      "svn_keys_finalize_device (each rank's point chunk from pinned host memory, in 2^20-point pieces "
                      "on a side stream; bytes per rank)"}

    # ---- CPU baseline + parity (rank 0) ----------------------------------------
    cpu = None
    parity = None
    if rank == 0 and not args.no_cpu_baseline and world == 1:
        threads = os.cpu_count() or 1
        lib, march = build_native_oracle()
        val, sample, (spts, sq), ores = run_cpu(w, params, args.seed, threads, lib, 1, 0)
        cpu = {"value": val, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": sample + f"; oracle restatement of nn.cpp:95-130 (-O3 -march={march}) on {cpu_model()}",
               "reference_build": reference_build_leg(w, args.seed, threads, 5.0)}
        if not args.no_parity:
            parity = {"bound": bounds_for(w.program.name, prec), "precision": prec}
            g = model.query_min(spts, sq, w.margin, precision=prec)
            parity["vs_oracle_on_cpu_sample"] = class_compare(g.min, g.free, g.argmin, ores[0], ores[2], ores[1],
                                                              w.margin, parity["bound"] or 0.0)
            from oracle import oracle as O
            nps = min(4096, spts.shape[0])
            gp = model.query_min(spts[:nps], sq[:2], w.margin, precision=prec, per_point=True).per_point
            op = O.query_min(w.program, params, spts[:nps], sq[:2], w.margin, per_point=True, threads=2,
                             library=lib)[3]
            parity["vs_oracle_on_cpu_sample"]["per_point_max_abs_err"] = float(np.max(np.abs(gp - op)))
            parity["vs_oracle_on_cpu_sample"]["per_point_checked"] = int(gp.size)
    if rank == 0 and not args.no_parity and mode == "motion" and prec in ("bf16", "fp16", "fp32_split"):
        # bf16 (or split) against the bit-identical FP32 path over >= 256 motions x the full cloud,
        # as measured (seeded net) and with the output bias calibrated so the median per-motion
        # min sits on the margin (the seeded nets are nearly all in collision)
        parity = parity or {"bound": bounds_for(w.program.name, prec), "precision": prec}
        nm = min(M, 256)
        bnd = parity["bound"] or 0.0
        ref = model.query_min(pts_np, q_np[:nm], w.margin, precision="fp32")
        mine = (mn[:nm].cpu().numpy(), fr[:nm].cpu().numpy().astype(bool), am[:nm].cpu().numpy())
        parity["vs_fp32_path_full_cloud"] = class_compare(*mine, ref.min, ref.free, ref.argmin, w.margin, bnd)
        cal = params.copy()
        cal[-1] += np.float32(w.margin - float(np.median(ref.min)))
        cm = S.Model(w.program, cal, device=local)
        rc = cm.query_min(pts_np, q_np[:nm], w.margin, precision="fp32")
        gc = cm.query_min(pts_np, q_np[:nm], w.margin, precision=prec)
        parity["calibrated_output_bias"] = class_compare(gc.min, gc.free, gc.argmin, rc.min, rc.free, rc.argmin,
                                                         w.margin, bnd)
        if prec in ("bf16", "fp16") and bounds_for(w.program.name, "fp32_split"):
            # the exact-for-every-motion classification on the same calibrated case: this precision
            # for the batch, fp32_split / the FP32 path for the motions near the margin
            # (svn_query_min_cascade); class mismatches against the FP32 path must be 0
            t0 = time.perf_counter()
            cr, st = cm.query_min_cascade(pts_np, q_np[:nm], w.margin, bnd, bounds_for(w.program.name, "fp32_split"),
                                          coarse=prec)
            t_c = time.perf_counter() - t0
            t0 = time.perf_counter()
            cm.query_min(pts_np, q_np[:nm], w.margin, precision=prec)
            t_p = time.perf_counter() - t0
            parity["cascade_on_calibrated"] = {"motions": nm, "stage_motions": list(st),
                                               "class_mismatches": int((cr.free != rc.free).sum()),
                                               "ms": t_c * 1e3, "ms_coarse_alone": t_p * 1e3}
        cm.close()

    if rank == 0:
        cl = clocks.summary()
        cl["extra_untimed_steps"] = extra_steps
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": prec, "data": "synthetic (seeded; see workloads.py)",
                "config": {"workload": w.key, "description": w.description, "network": w.program.name,
                           "motions": M_total, "points": P, "queries_per_step": total_queries,
                           "margin": w.margin, "parallelism": f"{mode}-shard x{world}",
                           "per_rank": {"motions": M, "points": pe - pb},
                           "l2": "flushed (256 MiB write) before every timed step, outside the step events"},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": cl, "parity": parity, "free_fraction": float(fr.float().mean().item())}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

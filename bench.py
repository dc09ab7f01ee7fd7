#!/usr/bin/env python3
"""bench.py — point x motion SDF queries/s of the swept-volume proxy hot path.

One step = one pass of the hot path over one batch: every (point x motion) pair of
the workload through the fused MLP, per-motion min/argmin and the margin class.

Default workload (N=1): BASELINE.json configs[2] ("c3"): DeepSDF 8x512 concat@4,
bf16 with fp32 accumulate, 1024 motions x 65536 points.  configs[1] ("c2") states fp32
weights: its FP32 path runs in the reference's order on FFMA (bit-identical; no tensor
pipe, so it cannot carry the "% of tensor-pipe peak" half of the metric) and
`--precision fp32_split` runs it fp32-grade on tcgen05; configs[4] ("c5") is the same
network as c3 at 128x its size; other configs: --config c1|c2|c4|c5|c5single.
With --gpus N (torchrun, one rank per GPU) every rank evaluates its own motion
shard of the c5 motion stream with c3's per-GPU size (weak scaling, no collective
on the data path).

Timing: W warm-up steps, then K steps bracketed by barrier + synchronize; device
time from CUDA events on the launching stream, max over ranks.  L2 is flushed
(a 256 MiB write, outside the per-step events) before every timed step.
`--impl reference` times the reference CPU path (the oracle restatement built with
-march=native, all host threads) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
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
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--precision", default=None, help="override: bf16 | fp32 | fp32_exact | fp32_split")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--motions", type=int, default=None, help="experiment override (not a BASELINE config)")
    ap.add_argument("--points", type=int, default=None, help="experiment override (not a BASELINE config)")
    ap.add_argument("--mode", default=None, choices=["motion", "point"],
                    help="multi-GPU sharding: motion (default) or point (single-motion workloads)")
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
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.tmp = None

    def __enter__(self):
        try:
            self.tmp = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.tmp, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
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
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons, "samples": len(rows)}


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
    from oracle import oracle as O
    M, P = cpu_sample(w, threads, seconds)
    pts, q = w.make(seed=seed, motions=M, points=P)
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        O.query_min(w.program, params, pts, q, w.margin, threads=threads, library=lib)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    sec = statistics.median(times)
    run_cpu.last_ms = sec * 1e3
    return M * P / sec, f"{M} motions x {P} points of {w.key} ({M * P} queries), {len(times)} runs, median"


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
        if rank != 0:
            return 0
        import paper_2402_15281_b200 as S  # init_params only (host, no GPU)
        params = S.init_params(w.program, args.seed, w.bound)
        threads = os.cpu_count() or 1
        lib, march = build_native_oracle()
        steps, warm = max(1, args.steps), max(0, min(args.warmup, 1))
        per_step = max(2.0, min(10.0, 120.0 / (steps + warm)))  # whole arm within ~2 minutes
        val, sample = run_cpu(w, params, args.seed, threads, lib, steps, warm, per_step)
        med_ms = getattr(run_cpu, "last_ms", None)
        # the reference's own call is single-threaded (nn.cpp:116): one thread, ~5 s sample
        v1, s1 = run_cpu(w, params, args.seed, 1, lib, 1, 0, 5.0)
        line = {"metric": METRIC, "value": val, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": med_ms,
                "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded)",
                "config": {"workload": w.key, "description": w.description, "network": w.program.name},
                "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "port",
                                 "sample": sample + f"; oracle restatement of nn.cpp:95-130 (-O3 -march={march}), "
                                                    f"{threads} threads on {cpu_model()}",
                                 "single_thread": {"value": v1, "unit": UNIT, "cores": 1, "sample": s1}},
                "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

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

    # ---- workload, resident in HBM ------------------------------------------
    # motion mode (weak scaling): rank r evaluates its own shard of the c5 motion
    #   stream (motions [r*M, (r+1)*M)) against the full cloud; no collective.
    # point mode (strong scaling, single-motion workloads): the cloud is split into
    #   rank chunks; one NCCL MIN all-reduce of 8 B per motion per step.
    mode = args.mode or ("point" if w.motions == 1 and world > 1 else "motion")
    from paper_2402_15281_b200.parallel import allreduce_keys_min, shard_range
    M, P = w.motions, w.points
    if mode == "motion":
        pts_np, q_np = w.make(seed=args.seed, motions=M, motion_offset=rank * M)
        pb, pe = 0, P
    else:
        pts_np, q_np = w.make(seed=args.seed, motions=M)
        pb, pe = shard_range(P, world, rank)
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

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    S.launch_count_reset()
    S.kernel_timing_begin()
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
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = sum(step_ms) / len(step_ms)
    kernel_ms = k_ms / max(1, k_n)
    if world > 1:
        t = torch.tensor([ms, kernel_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kernel_ms = float(t[0]), float(t[1])
    total_queries = M * P * world if mode == "motion" else M * P
    value = total_queries / (ms * 1e-3)

    # ---- roofline of the dominant kernel (the fused MLP) ----------------------
    flop_q = w.program.flops_per_query()
    achieved_tf = M * (pe - pb) * flop_q / (kernel_ms * 1e-3) / 1e12
    if prec == "bf16":
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
        except Exception:
            pass

    # ---- e2e through the public host API (host buffers, copies inside) --------
    e2e = None
    if not args.no_e2e and mode == "motion":
        hp = torch.from_numpy(pts_np).pin_memory().numpy()
        hq = torch.from_numpy(q_np).pin_memory().numpy()
        model.query_min(hp, hq, w.margin, precision=prec)  # warm the host path
        if world > 1:
            dist.barrier()
        t_e = []
        for _ in range(max(1, min(args.steps, 3))):
            t0 = time.perf_counter()
            model.query_min(hp, hq, w.margin, precision=prec)
            t_e.append(time.perf_counter() - t0)
        e_ms = statistics.mean(t_e) * 1e3
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t[0])
        e2e = {"value": total_queries / (e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(hp.nbytes + hq.nbytes),
               "d2h_bytes_per_step": int(M * (4 + 4 + 1)), "ms_per_step": e_ms,
               "api": "svn_query_min (C-ABI, host buffers)"}

    # ---- CPU baseline (rank 0, N=1 only) ---------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        lib, march = build_native_oracle()
        val, sample = run_cpu(w, params, args.seed, threads, lib, 1, 0)
        cpu = {"value": val, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": sample + f"; oracle restatement of nn.cpp:95-130 (-O3 -march={march}) on {cpu_model()}"}

    if rank == 0:
        cl = clocks.summary()
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "weak" if mode == "motion" else "strong",
                "vs_baseline": None, "dtype": prec, "data": "synthetic (seeded; see workloads.py)",
                "config": {"workload": w.key, "description": w.description, "network": w.program.name,
                           "motions_per_gpu": M, "points": P, "queries_per_step": total_queries,
                           "margin": w.margin, "parallelism": f"{mode}-shard x{world}",
                           "l2": "flushed (256 MiB write) before every timed step, outside the step events"},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": cl, "free_fraction": float(fr.float().mean().item())}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

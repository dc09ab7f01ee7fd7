"""Parity report: every BASELINE config's network through the CUDA path (C-ABI) against the
CPU oracle, on bounded seeded samples, written as JSON (profiles/r2_parity_report.json).

Test infrastructure (it imports oracle/), run on a GPU box:
    python tests/parity_report.py [--out profiles/r2_parity_report.json]

Per (config, precision) it records the per-point max |delta_gpu - delta_oracle| against the
stated tolerance (fp32: 1e-5 — met bit-identically, fp32_split and bf16: the frozen bounds of
tests/golden), whether
min/argmin/class agree, and the motions whose oracle min lies within the tolerance of the
margin ("ambiguous", north_star: counted and reported). The margin is also moved onto the
data (output bias set so the median oracle min equals the margin) so the classification is
exercised on both sides; that variant is reported as "<config>+calibrated".
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2402_15281_b200 as S  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

_B = json.loads((ROOT / "tests" / "golden" / "bf16_bounds.json").read_text())
BF16_BOUND = {k: v["bound"] for k, v in _B.items() if isinstance(v, dict)}
_H = json.loads((ROOT / "tests" / "golden" / "fp16_bounds.json").read_text())
FP16_BOUND = {k: v["bound"] for k, v in _H.items() if isinstance(v, dict)}
_F = json.loads((ROOT / "tests" / "golden" / "fp32_split_bounds.json").read_text())
FP32_SPLIT_BOUND = {k: v["bound"] for k, v in _F.items() if isinstance(v, dict)}

# (config, motions, points, precisions): samples sized so the oracle takes seconds
CASES = [
    ("c1", 1, 4096, ["fp32", "fp32_split", "bf16", "fp16"]),
    ("c2", 64, 2048, ["fp32", "fp32_split", "bf16", "fp16"]),
    ("c3", 16, 2048, ["bf16", "fp16", "fp32", "fp32_split"]),
    ("c4", 16, 2048, ["bf16", "fp16", "fp32", "fp32_split"]),
]


def tol(prec: str, program) -> float:
    if prec == "fp32_split":
        return FP32_SPLIT_BOUND[program.name]
    if prec == "fp16":
        return FP16_BOUND.get(program.name, float("nan"))
    return {"fp32_exact": 0.0, "fp32": 1e-5}.get(prec, BF16_BOUND.get(program.name, float("nan")))


def f64_truth(w, params, pts, q):
    """The same network in fp64 (oracle_forward_eval_f64 on the replicated rows): the yardstick
    for how close an fp32 computation gets to the exact value."""
    M, P = q.shape[0], pts.shape[0]
    raw = np.concatenate([np.repeat(pts[None].astype(np.float64), M, 0).reshape(-1, 3),
                          np.repeat(q.reshape(M, 1, -1).astype(np.float64), P, 1).reshape(M * P, -1)], 1)
    return O.forward_eval(w.program, params.astype(np.float64), raw, np.float64).reshape(M, P)


def one(w, params, pts, q, prec, threads, oracle_out, truth=None):
    omin, oarg, ofree, opp = oracle_out
    r = S.Model(w.program, params).query_min(pts, q, w.margin, precision=prec, per_point=True)
    t = tol(prec, w.program)
    err = np.abs(r.per_point.astype(np.float64) - opp.astype(np.float64))
    amb = np.abs(omin.astype(np.float64) - w.margin) <= t
    arg_eq = r.argmin == oarg
    d_at = opp[np.arange(len(oarg)), r.argmin].astype(np.float64)
    arg_ok = arg_eq | (np.abs(d_at - omin.astype(np.float64)) <= t)
    return {
        "precision": prec,
        "tolerance": t,
        "max_abs_err": float(err.max()),
        "mean_abs_err": float(err.mean()),
        "within_tolerance": bool(err.max() <= t),
        "bit_identical": bool(np.array_equal(r.per_point, opp)),
        "min_equal_to_own_per_point_min": bool(np.array_equal(r.min, r.per_point.min(axis=1))),
        "argmin_equal": int(arg_eq.sum()),
        "argmin_equal_or_within_tolerance": int(arg_ok.sum()),
        "class_agree_outside_ambiguous": bool(np.array_equal(r.free[~amb], ofree[~amb])),
        "ambiguous_motions": int(amb.sum()),
        "free_fraction_gpu": float(r.free.mean()),
        "free_fraction_oracle": float(ofree.mean()),
        **({"max_abs_err_vs_fp64": float(np.abs(r.per_point.astype(np.float64) - truth).max()),
            "oracle_f32_max_abs_err_vs_fp64": float(np.abs(opp.astype(np.float64) - truth).max())}
           if truth is not None and prec != "bf16" else {}),
    }


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r2_parity_report.json"))
    ap.add_argument("--seed", type=int, default=2024)
    args = ap.parse_args()
    threads = os.cpu_count() or 1
    report = {"what": "CUDA path (C-ABI) vs CPU oracle (oracle/sweptnet_oracle.c) on seeded samples",
              "oracle_threads": threads, "cases": []}
    for key, M, P, precs in CASES:
        w = WORKLOADS[key]
        params = S.init_params(w.program, args.seed, w.bound)
        pts, q = w.make(seed=args.seed, motions=M, points=P)
        for calibrated in (False, True):
            p = params
            t0 = time.time()
            out = O.query_min(w.program, p, pts, q, w.margin, per_point=True, threads=threads)
            if calibrated:
                if M < 4:
                    continue
                p = params.copy()
                p[-1] += np.float32(w.margin - np.median(out[0].astype(np.float64)))
                out = O.query_min(w.program, p, pts, q, w.margin, per_point=True, threads=threads)
            t_or = time.time() - t0
            truth = None if calibrated else f64_truth(w, p, pts, q)
            case = {"config": key + ("+calibrated" if calibrated else ""), "network": w.program.name,
                    "motions": M, "points": P, "margin": w.margin, "oracle_seconds": round(t_or, 2),
                    "results": [one(w, p, pts, q, prec, threads, out, truth) for prec in precs]}
            report["cases"].append(case)
            for r in case["results"]:
                print(f"{case['config']:14s} {r['precision']:10s} max|err| {r['max_abs_err']:.3e} "
                      f"(tol {r['tolerance']:.1e}) class-ok {r['class_agree_outside_ambiguous']} "
                      f"ambiguous {r['ambiguous_motions']}/{M} argmin {r['argmin_equal']}/{M}"
                      + (f" | vs fp64 {r['max_abs_err_vs_fp64']:.2e} (oracle f32 vs fp64 "
                         f"{r['oracle_f32_max_abs_err_vs_fp64']:.2e})" if "max_abs_err_vs_fp64" in r else ""),
                      flush=True)
    report["all_within_tolerance"] = all(r["within_tolerance"] for c in report["cases"] for r in c["results"])
    report["all_class_agree"] = all(r["class_agree_outside_ambiguous"] for c in report["cases"] for r in c["results"])
    Path(args.out).write_text(json.dumps(report, indent=1) + "\n")
    print("wrote", args.out, "all_within_tolerance", report["all_within_tolerance"], "all_class_agree",
          report["all_class_agree"])
    return 0 if report["all_within_tolerance"] and report["all_class_agree"] else 1


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python3
"""Summarise an ncu report: key throughput metrics + opcode mix + top stall lines."""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
for k in keys:
    if k in h:
        i = h.index(k)
        print(f"{k} = {v[i]} {units[i]}")
# cycles where no instruction issued, by the reason the sampled warp was stalled
ni = {k[len("smsp__pcsamp_warps_issue_stalled_"):-len("_not_issued")]: float(x or 0)
      for k, x in zip(h, v) if k.startswith("smsp__pcsamp_warps_issue_stalled_") and k.endswith("_not_issued")}
sel = float(v[h.index("smsp__pcsamp_warps_issue_stalled_selected")] or 0) if "smsp__pcsamp_warps_issue_stalled_selected" in h else 0
if ni and sel:
    tot_ni = sum(ni.values())
    print(f"issue samples: selected {sel:.0f}, not issued {tot_ni:.0f}; not-issued by stall reason (% of all):")
    for k2, x in sorted(ni.items(), key=lambda t: -t[1])[:8]:
        print(f"  {k2:22s} {x / (sel + tot_ni) * 100:5.1f}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
data = rows[2:]
iS, iW, iE = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
tot = sum(float(r[iW] or 0) for r in data) or 1
ex, st = Counter(), Counter()
for r in data:
    op = r[iS].strip().split()
    if not op:
        continue
    o = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
    ex[o] += float(r[iE] or 0)
    st[o] += float(r[iW] or 0)
T = sum(ex.values()) or 1
print("opcode mix (exec %, stall %):")
for o, val in ex.most_common(16):
    print(f"  {o:10s} {val / T * 100:5.1f}  {st[o] / tot * 100:5.1f}")
print("top stall lines:")
for r in sorted(data, key=lambda r: -float(r[iW] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"  {float(r[iW] or 0) / tot * 100:5.1f}%  {r[iS][:100]}")

#!/usr/bin/env python3
"""Per-CUDA-source-line warp-stall samples of one kernel in an ncu report.

usage: ncu_lines.py REPORT.ncu-rep LIB.so CUBIN_NAME KERNEL_MANGLED [top]
Aligns ncu's SASS listing (in order) with `nvdisasm -g` of the same cubin."""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter

rep, lib, cubin, kern = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
data = rows[2:]
iS, iW = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", cubin, os.path.abspath(lib)], cwd=d, capture_output=True)
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cubin)], capture_output=True, text=True).stdout
dis = dis.split(f".text.{kern}:", 1)[1].split("//--------------------- .", 1)[0]
line = None
ins = []
for ln in dis.splitlines():
    m = re.search(r'## File "([^"]+)", line (\d+)', ln)
    if m:
        line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
        ins.append(line)
if len(ins) != len(data):
    print(f"warning: {len(ins)} disassembled vs {len(data)} profiled instructions", file=sys.stderr)
tot = sum(float(r[iW] or 0) for r in data) or 1
c = Counter()
for r, l in zip(data, ins):
    c[l] += float(r[iW] or 0)
for l, v in c.most_common(top):
    print(f"{v / tot * 100:5.1f}%  {l}")

# top instructions with their dominant stall reasons
sr = [i for i, n in enumerate(hh) if n.startswith("stall_") and "Not Issued" not in n]
print("\ntop instructions:")
order = sorted(range(len(data)), key=lambda i: -float(data[i][iW] or 0))[:top]
for i in order:
    r = data[i]
    reasons = sorted(((float(r[k] or 0), hh[k][6:]) for k in sr), reverse=True)[:3]
    rs = " ".join(f"{n}:{v / tot * 100:.1f}" for v, n in reasons if v)
    print(f"{float(r[iW] or 0) / tot * 100:5.1f}%  {ins[i] if i < len(ins) else '?':24s} {r[iS][:60]:60s} {rs}")

#!/usr/bin/env python3
"""Per-CTA start / ready / end times of the width-256 bf16 kernel (globaltimer), from a build
with SVN_NVCC_DEFINES=SVN_CTA_TIMES:
    SVN_NVCC_DEFINES=SVN_CTA_TIMES python scripts/cta_times.py [motions]
Prints the spread of CTA starts, prologue ends and exits relative to the first start."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2402_15281_b200 as S  # noqa: E402
from paper_2402_15281_b200 import abi  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

import torch  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 64
w = WORKLOADS["c2"]
params = S.init_params(w.program, 0, w.bound)
pts_np, q_np = w.make(seed=0, motions=M)
model = S.Model(w.program, params)
dev = torch.device("cuda", 0)
pts, q = torch.from_numpy(pts_np).to(dev), torch.from_numpy(q_np).to(dev)
mn = torch.empty(M, dtype=torch.float32, device=dev)
am = torch.empty(M, dtype=torch.int32, device=dev)
fr = torch.empty(M, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
ends = []
for i in range(6):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    model.query_min_device(pts, q, w.margin, mn, am, fr, None, precision="bf16", stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    if i >= 3:  # per-SM exit order of the last three launches
        b = (C.c_ulonglong * (4 * 148))()
        assert abi.lib().svn_debug_cta_times(b, 148) == 0
        tt = np.array(b, dtype=np.int64).reshape(148, 4)
        ends.append({int(r[3]): (r[2] - tt[:, 0].min()) / 1e3 for r in tt})
L = abi.lib()
buf = (C.c_ulonglong * (4 * 148))()
assert L.svn_debug_cta_times(buf, 148) == 0
t = np.array(buf, dtype=np.int64).reshape(148, 4)[:, :3]
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
r = (t - t0) / 1e3
print(f"M={M}: step {e0.elapsed_time(e1) * 1e3:.1f} us (K0 + fused, events); {len(t)} CTAs")
for name, col in (("start", 0), ("ready", 1), ("end", 2)):
    v = r[:, col]
    print(f"  {name:5s} us: min {v.min():7.1f}  median {np.median(v):7.1f}  max {v.max():7.1f}")
d = r[:, 2] - r[:, 1]
print(f"  ready->end per CTA: min {d.min():.1f} median {np.median(d):.1f} max {d.max():.1f} us")
# is "slow" a property of the SM?  rank correlation of the per-SM exit times between launches
sms = sorted(ends[0])
v = np.array([[e[sm] for sm in sms] for e in ends])
rk = np.argsort(np.argsort(v, axis=1), axis=1)
print("  per-SM exit-time rank correlation between launches:",
      " ".join(f"{np.corrcoef(rk[i], rk[j])[0, 1]:.2f}" for i in range(len(ends)) for j in range(i + 1, len(ends))))
slow = [sms[i] for i in np.argsort(-v.mean(axis=0))[:12]]
print("  12 slowest SMs (mean over launches):", slow)

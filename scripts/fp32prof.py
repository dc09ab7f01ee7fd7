"""Print the FP32 kernel phase counters (scripts/ab/fp32_prof.cu build, SVN_PROF=1 run)."""
import sys
line = [l for l in open(sys.argv[1]) if 'svn prof' in l][-1]
v = [int(x) for x in line.split(']')[1].split()]
for o, who in ((0, "thread 0"), (8, "thread 160")):
    tot = v[o] or 1
    print(who, " ".join(f"{n} {v[o + i] / tot * 100:5.1f}%" for i, n in enumerate(["total", "wait_full", "barrier", "epilogue+last_sync", "output"])))

"""Print the FP32 kernel's phase split (thread 0 of every CTA, summed): run bench.py with
SVN_PROF=1 on a library built with SVN_NVCC_DEFINES=SVN_KERNEL_PROF (scripts/build_variant.py)."""
import sys
line = [l for l in open(sys.argv[1]) if 'svn prof' in l][-1]
v = [int(x) for x in line.split(']')[1].split()]
tot = v[0] or 1
print(" ".join(f"{n} {v[i] / tot * 100:5.1f}%" for i, n in
               enumerate(["total", "weight_wait", "chunk_barrier", "epilogue", "output_layer"])))

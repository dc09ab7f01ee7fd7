# Wait/work accounting of the tensor-core kernels (SVN_KERNEL_PROF build, scripts/profsum.py):
#   gpurun -- 'bash scripts/prof_run.sh "--config paper --motions 1024" "--config c3 --motions 64"'
set -u
mkdir -p gpurun_out
SVN_NVCC_DEFINES="SVN_KERNEL_PROF" python paper_2402_15281_b200/build.py --force > gpurun_out/prof_build.log 2>&1; echo "build rc=$?"
i=0
for a in "$@"; do i=$((i+1))
  SVN_PROF=1 timeout 600 python bench.py $a --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/prof_$i.log 2>&1
  echo "== $a"; tail -1 gpurun_out/prof_$i.log | python scripts/benchline.py "$a"; python scripts/profsum.py gpurun_out/prof_$i.log
done

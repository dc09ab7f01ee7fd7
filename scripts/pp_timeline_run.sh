# Instrumented build (clock reads + one-round timeline of CTA 0) of the width-256 bf16 kernel
# and its timeline on the c2 network: gpurun -- 'bash scripts/pp_timeline_run.sh'
set -u
mkdir -p gpurun_out
SVN_NVCC_DEFINES="SVN_KERNEL_PROF SVN_PP_TIMELINE" python paper_2402_15281_b200/build.py --force > gpurun_out/tl_build.log 2>&1; echo "build rc=$?"
SVN_PROF=1 python bench.py --config c2 --precision bf16 --motions ${1:-256} --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-parity > gpurun_out/tl.log 2>&1
python scripts/pp_timeline.py gpurun_out/tl.log; python scripts/profsum.py gpurun_out/tl.log

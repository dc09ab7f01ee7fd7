# One-round timeline + wait counters of the width-256 bf16 kernel (instrumented build)
for m in 64 1024; do
SVN_LIB=scripts/ab/lib_pp_tl.so SVN_PROF=1 timeout 300 python bench.py --config c2 --precision bf16 --motions $m --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/pptl_$m.log 2>&1
python scripts/pp_timeline.py gpurun_out/pptl_$m.log
python scripts/profsum.py gpurun_out/pptl_$m.log
done

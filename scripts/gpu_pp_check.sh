timeout 600 python -m pytest tests -m gpu -x -q -k "plain_4x256 or 4x256 or edges or c2 or fp32_split or fig2" 2>&1 | tail -3
VAR=SVN_LIB VALUES="${VALUES:-scripts/ab/lib_prev.so paper_2402_15281_b200/_lib/libsweptnet_b200.so}" BENCH_ARGS="${BENCH_ARGS:---config c2 --precision bf16}" bash scripts/gpu_ab.sh
SVN_PROF=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_ARGS:---config c2 --precision bf16} > gpurun_out/profab_1.log 2>&1
python scripts/pp_timeline.py gpurun_out/profab_1.log

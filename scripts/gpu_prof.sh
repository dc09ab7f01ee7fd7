# ncu full capture of the bf16 fused kernel on the default bench workload
set -x
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-}"
timeout 600 $CMD > gpurun_out/bench_plain.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-fused_bf16} -s 1 -c 1 -o gpurun_out/${PROF:-prof} $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full.log

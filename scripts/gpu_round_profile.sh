# Evidence for profiles/: plain bench, launch list (ncu gpu__time_duration), one full capture.
set -x
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/bench_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_bf16 -s 1 -c 1 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; grep -m1 "model name" /proc/cpuinfo
timeout 900 python scripts/calibrate_bf16.py > gpurun_out/calib.log 2>&1; echo "calib rc=$?"
cat gpurun_out/calib.log | tail -8
cp gpurun_out/bf16_bounds.json tests/golden/bf16_bounds.json
timeout 900 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
tail -2 gpurun_out/bench_default.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/bench_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_bf16 -s 1 -c 1 -o gpurun_out/prof_c3 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -5 gpurun_out/ncu_full.log

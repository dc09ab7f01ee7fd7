# Round check: tests, smoke, default bench (as the driver runs it), c5 sweep, profiles
set -x
nproc; grep -m1 "model name" /proc/cpuinfo
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?"
timeout 1200 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.log 2>&1; echo "c5 rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/bench_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_bf16 -s 1 -c 1 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"

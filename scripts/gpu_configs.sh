# bench every config once at N=1 (no CPU baseline), for the per-config table in DESIGN.md
set -x
for c in c1 c2 c3 c4 c5single; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
  tail -1 gpurun_out/bench_$c.log | cut -c1-400
done
timeout 900 python bench.py --config c2 --precision bf16 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2bf16.log 2>&1; echo "c2bf16 rc=$?"
tail -1 gpurun_out/bench_c2bf16.log | cut -c1-400
timeout 900 python bench.py --config c1 --precision fp32_exact --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1exact.log 2>&1; echo "c1exact rc=$?"
timeout 900 python bench.py --config c2 --precision fp32_split --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2split.log 2>&1; echo "c2split rc=$?"

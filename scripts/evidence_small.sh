# Small-config bench lines with enough timed steps (c1/c2/paper: 3-step lines are noisy), the
# parity report, and the default c5 line in bf16 and fp16:  gpurun -- 'bash scripts/evidence_small.sh'
set -u
mkdir -p gpurun_out/cfg50
for a in "--config c1" "--config c1 --precision fp32_split" "--config c1 --precision bf16" "--config c1 --precision fp16" \
         "--config c2 --precision bf16" "--config c2 --precision fp16" "--config c2 --precision fp32_split" \
         "--config paper" "--config paper --precision fp16"; do
  n=$(echo "$a" | tr -d ' -')
  timeout 600 python bench.py $a --steps 50 --warmup 10 --no-cpu-baseline > gpurun_out/cfg50/$n.log 2>&1
  tail -1 gpurun_out/cfg50/$n.log | python scripts/benchline.py "$a"
done
timeout 900 python tests/parity_report.py --out gpurun_out/r2_parity_report.json > gpurun_out/parity_report.txt 2>&1; tail -1 gpurun_out/parity_report.txt
timeout 1500 python bench.py > gpurun_out/bench_c5.log 2>&1; tail -1 gpurun_out/bench_c5.log | python scripts/benchline.py "c5 default"
timeout 1500 python bench.py --precision fp16 --no-cpu-baseline > gpurun_out/bench_c5_fp16.log 2>&1; tail -1 gpurun_out/bench_c5_fp16.log | python scripts/benchline.py "c5 fp16"

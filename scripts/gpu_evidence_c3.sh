# Width-512 evidence on the current kernel (after the dynamic tile schedule): default bench,
# reference arm, c4, c5single, c5, the launch list and one ncu --set full of the fused kernel
set -x
nproc; nvidia-smi --query-gpu=name,serial --format=csv,noheader
timeout 900 python bench.py > gpurun_out/e3_default.log 2>&1; echo "default rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/e3_reference.log 2>&1; echo "reference rc=$?"
for c in c4 c5single; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/e3_$c.log 2>&1; echo "$c rc=$?"
done
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/e3_c5.log 2>&1; echo "c5 rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/e3_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e3_launches.csv $CMD > gpurun_out/e3_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_bf16 -s 1 -c 1 -o gpurun_out/e3_c3_full $CMD > gpurun_out/e3_ncu_full.log 2>&1; echo "ncu full rc=$?"

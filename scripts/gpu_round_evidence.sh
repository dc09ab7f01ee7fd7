# Round-end evidence for profiles/ on the current kernels: default bench (all legs),
# launch list of the default bench and one ncu --set full capture per fused kernel
# (each ncu pass only after its own command ran clean without ncu).
set -x
nproc; grep -m1 "model name" /proc/cpuinfo; nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv
timeout 900 python bench.py > gpurun_out/ev_default.log 2>&1; echo "default rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/ev_reference.log 2>&1; echo "reference rc=$?"
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev_c5.log 2>&1; echo "c5 rc=$?"
for c in c1 c2 c4 c5single; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_$c.log 2>&1; echo "$c rc=$?"
done
for p in fp32_split bf16; do
  timeout 900 python bench.py --config c1 --precision $p --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_c1_$p.log 2>&1; echo "c1 $p rc=$?"
  timeout 900 python bench.py --config c2 --precision $p --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_c2_$p.log 2>&1; echo "c2 $p rc=$?"
done
timeout 900 python bench.py --config c2 --precision bf16 --motions 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev_c2_bf16_m1024.log 2>&1; echo "c2 bf16 M=1024 rc=$?"
timeout 900 python bench.py --config paper --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_paper.log 2>&1; echo "paper rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/ev_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv $CMD > gpurun_out/ev_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_bf16 -s 1 -c 1 -o gpurun_out/ev_c3_full $CMD > gpurun_out/ev_ncu_full.log 2>&1; echo "ncu full c3 rc=$?"
for p in fp32 fp32_split bf16; do
  C="python bench.py --config c2 --precision $p --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
  timeout 300 $C > gpurun_out/ev_pw_$p.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_ -s 1 -c 1 -o gpurun_out/ev_c2_$p $C > gpurun_out/ev_ncu_c2_$p.log 2>&1; echo "ncu c2 $p rc=$?"
done

# Round-end evidence for profiles/: default bench (all legs), reference arm, c5 sweep,
# launch list and one full ncu capture of the fused kernel (each ncu pass after its command ran clean).
set -x
timeout 900 python bench.py > gpurun_out/ev_default.log 2>&1; echo "default rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/ev_reference.log 2>&1; echo "reference rc=$?"
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev_c5.log 2>&1; echo "c5 rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/ev_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv $CMD > gpurun_out/ev_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fused_bf16 -s 1 -c 1 -o gpurun_out/ev_full $CMD > gpurun_out/ev_ncu_full.log 2>&1; echo "ncu full rc=$?"

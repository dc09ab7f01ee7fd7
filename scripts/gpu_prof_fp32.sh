C="python bench.py --config c2 --precision fp32 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $C > gpurun_out/pf.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_fp32 -s 1 -c 1 -o gpurun_out/prof_fp32 $C > gpurun_out/ncu_fp32.log 2>&1; echo "ncu rc=$?"

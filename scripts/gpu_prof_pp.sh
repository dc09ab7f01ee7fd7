C2="python bench.py --config c2 --precision bf16 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $C2 > gpurun_out/p2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_bf16_pp -s 1 -c 1 -o gpurun_out/prof_pp2 $C2 > gpurun_out/ncu_pp.log 2>&1; echo "ncu pp rc=$?"

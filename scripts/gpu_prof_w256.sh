# ncu --set full of the three width-256 kernels on c2 (FP32 path, fp32_split, bf16 ping-pong)
set -x
for p in fp32 fp32_split bf16; do
  C="python bench.py --config c2 --precision $p --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
  timeout 300 $C > gpurun_out/pw_$p.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_ -s 1 -c 1 -o gpurun_out/prof_c2_$p $C > gpurun_out/ncu_c2_$p.log 2>&1; echo "ncu $p rc=$?"
done

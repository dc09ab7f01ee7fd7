# FP32-path rows of DESIGN.md §6 on the current kernel, the paper-network rows, and a fresh
# ncu capture of the FP32 kernel on c2 (after its command ran clean without ncu)
set -x
for c in c1 c2; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fe_$c.log 2>&1; echo "$c rc=$?"
done
bash scripts/gpu_paper.sh
C="python bench.py --config c2 --precision fp32 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $C > gpurun_out/fe_pw.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_ -s 1 -c 1 -o gpurun_out/fe_c2_fp32 $C > gpurun_out/fe_ncu.log 2>&1; echo "ncu rc=$?"

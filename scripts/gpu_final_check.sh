# End-of-session check on the committed code: GPU tests, smoke, default bench twice, reference arm
set -x
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -n 2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
timeout 900 python bench.py > gpurun_out/fc_default1.log 2>&1; echo "default rc=$?"
timeout 900 python bench.py > gpurun_out/fc_default2.log 2>&1; echo "default rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/fc_reference.log 2>&1; echo "reference rc=$?"
for p in fp32 fp32_split bf16; do
  timeout 600 python bench.py --config c2 --precision $p --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fc_c2_$p.log 2>&1; echo "c2 $p rc=$?"
done

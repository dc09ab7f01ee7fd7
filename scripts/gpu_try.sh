timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for c in c1 c2; do
  timeout 900 python bench.py --config $c --precision fp32 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}fp32.log 2>&1; echo "$c rc=$?"
  tail -1 gpurun_out/bench_${c}fp32.log | python scripts/benchline.py "$c fp32"
  tail -1 gpurun_out/bench_${c}fp32.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('e2e', d['e2e']['value']/1e6, 'kernel_ms', d['roofline'].get('kernel_ms'), 'ms', d['ms_per_step'])"
done
bash scripts/gpu_fp32modes.sh

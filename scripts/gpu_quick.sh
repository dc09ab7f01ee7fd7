# quick GPU iteration: parity tests + short bench (no CPU baseline)
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench_quick.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_quick.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('VALUE', d['value']/1e6, 'Mq/s', 'TF', d['roofline']['achieved'], 'frac', d['roofline']['frac'], 'clk', d['clocks'])"

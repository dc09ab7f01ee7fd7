set -u
mkdir -p gpurun_out
timeout 600 python scripts/calibrate_bf16.py fp16 2>&1 | tail -6
timeout 600 python scripts/calibrate_bf16.py bf16 2>&1 | tail -6
for p in bf16 fp16; do
  timeout 300 python bench.py --config c3 --precision $p --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity 2>&1 | tail -1 | python scripts/benchline.py "c3 $p"
  timeout 300 python bench.py --config c2 --precision $p --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-parity 2>&1 | tail -1 | python scripts/benchline.py "c2 $p"
  timeout 300 python bench.py --config paper --motions 1024 --precision $p --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity 2>&1 | tail -1 | python scripts/benchline.py "paper1024 $p"
done
bash scripts/gpu.sh test

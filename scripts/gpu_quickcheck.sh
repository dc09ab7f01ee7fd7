# Quick state check after a container re-create: GPU tests, smoke, default bench
set -x
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/qc_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/qc_default.log
timeout 600 python bench.py --config c2 --precision bf16 --no-cpu-baseline > gpurun_out/qc_c2bf16.log 2>&1; echo "c2 bf16 rc=$?"; tail -1 gpurun_out/qc_c2bf16.log

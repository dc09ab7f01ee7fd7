# Exercise bench.py's multi-rank path on a one-GPU box: 2 ranks over gloo, both on device 0
# (no inter-rank kernel dependencies: motion mode has no collective, point mode one MIN
# all-reduce of 8 B per motion through gloo). Checks the JSON contract, not scaling.
export SVN_BENCH_BACKEND=gloo SVN_BENCH_DEVICE=0
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 2 --warmup 3 --motions 64 --no-cpu-baseline > gpurun_out/mr_motion.log 2>&1; echo "motion rc=$?"
tail -1 gpurun_out/mr_motion.log | cut -c1-600
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus 2 --config c5single --points 2000000 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/mr_point.log 2>&1; echo "point rc=$?"
tail -1 gpurun_out/mr_point.log | cut -c1-600
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 \
  bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/mr_ref.log 2>&1; echo "reference rc=$?"
tail -1 gpurun_out/mr_ref.log | cut -c1-300
# the driver's own launch line at N=1 (NCCL, device_id from LOCAL_RANK)
unset SVN_BENCH_BACKEND SVN_BENCH_DEVICE
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29536 \
  bench.py --gpus 1 --steps 2 --warmup 3 > gpurun_out/mr_nccl1.log 2>&1; echo "nccl N=1 rc=$?"
tail -1 gpurun_out/mr_nccl1.log | cut -c1-300

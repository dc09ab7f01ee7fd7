# wait-time counters of the fused bf16 kernel (SVN_PROF=1), default bench workload
timeout 600 env SVN_PROF=1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/profc.log 2>&1; echo "rc=$?"
grep "svn prof" gpurun_out/profc.log | tail -1
tail -1 gpurun_out/profc.log | cut -c1-300

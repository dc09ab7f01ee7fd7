i=0
for v in ${VALUES}; do
  i=$((i+1))
  env ${VAR}=$v SVN_PROF=1 timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/profab_$i.log 2>&1
  echo "== ${VAR}=$v"; grep "svn prof" gpurun_out/profab_$i.log | tail -1
done

# A/B of kernel variants selected by env (VAR=name, VALUES="..."), alternated twice
i=0
for rep in 1 2; do
  for v in ${VALUES}; do
    i=$((i+1))
    env ${VAR}=$v timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/ab_$i.log 2>&1
    tail -1 gpurun_out/ab_$i.log | python scripts/benchline.py "${VAR}=$v"
  done
done

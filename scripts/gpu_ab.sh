# A/B of kernel variants selected by env (VAR=name, VALUES="..."), alternated twice
i=0
for rep in 1 2; do
  for v in ${VALUES}; do
    i=$((i+1))
    env ${VAR}=$v timeout 600 python bench.py --steps 4 --warmup 2 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/ab_$i.log 2>&1
    tail -1 gpurun_out/ab_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${VAR}=$v', round(d['value']/1e6,1), 'Mq/s', round(d['roofline']['achieved']), 'TF', 'clk', d['clocks']['sm_mhz'], 'cyc/q', round(d['ms_per_step']*1e-3*d['clocks']['sm_mhz']*1e6/d['config']['queries_per_step']*148, 1))"
  done
done

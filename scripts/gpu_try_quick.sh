# guarded first run of a new kernel: tiny case under a short timeout first
set -x
timeout 120 python -c "
import numpy as np, paper_2402_15281_b200 as S
from oracle import oracle as O
from paper_2402_15281_b200.workloads import WORKLOADS
for key in ['c3','c2']:
    w=WORKLOADS[key]; p=S.init_params(w.program,1,w.bound); pts,q=w.make(seed=1,motions=2,points=700)
    r=S.Model(w.program,p).query_min(pts,q,w.margin,precision='bf16',per_point=True)
    o=O.query_min(w.program,p,pts,q,w.margin,per_point=True,threads=8)
    print(key,'maxerr',np.abs(r.per_point-o[3]).max(), r.min, o[0], r.argmin, o[1])
" > gpurun_out/try.log 2>&1; echo "try rc=$?"
cat gpurun_out/try.log | tail -5
# quick GPU iteration: parity tests + short bench (no CPU baseline)
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench_quick.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_quick.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('VALUE', d['value']/1e6, 'Mq/s', 'TF', d['roofline']['achieved'], 'frac', d['roofline']['frac'], 'clk', d['clocks'])"

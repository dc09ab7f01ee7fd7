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

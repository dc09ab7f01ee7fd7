SVN_LIB=scripts/ab/lib_ppf2.so timeout 600 python -m pytest tests -m gpu -x -q -k "c2 or 256 or ragged or tile or many" 2>&1 | tail -n 2
VALUES="scripts/ab/lib_head6.so scripts/ab/lib_ppf2.so" bash scripts/gpu_ab_pp.sh

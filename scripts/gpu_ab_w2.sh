# A/B: two TMEM loads per wait::ld in the epilogue (pp at width 256, pair at width 512)
for rep in 1 2; do
for lib in scripts/ab/lib_base.so scripts/ab/lib_pp_w2.so; do
  for m in 64 1024; do
    SVN_LIB=$lib timeout 300 python bench.py --config c2 --precision bf16 --motions $m --steps 4 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | tail -n 1 | python scripts/benchline.py "$lib c2bf16 M=$m"
  done
done
for lib in scripts/ab/lib_base.so scripts/ab/lib_pair_w2.so; do
  SVN_LIB=$lib timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | tail -n 1 | python scripts/benchline.py "$lib c3"
done
done
SVN_LIB=scripts/ab/lib_pp_w2.so timeout 600 python -m pytest tests -m gpu -x -q -k "4x256 or c2 or fig2 or edges" 2>&1 | tail -n 2
SVN_LIB=scripts/ab/lib_pair_w2.so timeout 600 python -m pytest tests -m gpu -x -q -k "c3 or 512 or fig2 or edges" 2>&1 | tail -n 2

# A/B of the width-256 bf16 kernel: VALUES = libraries; c2 network in bf16 at 64 and 1024 motions
for rep in 1 2; do
for lib in ${VALUES}; do
  for m in 64 1024; do
    SVN_LIB=$lib timeout 300 python bench.py --config c2 --precision bf16 --motions $m --steps 4 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | tail -n 1 | python scripts/benchline.py "$lib c2bf16 M=$m"
  done
done
done

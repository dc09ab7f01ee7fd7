# A/B of FP32-path builds (VALUES = libraries): c2 (width 256) and c3's network (width 512, 64 motions)
for rep in 1 2; do
for lib in ${VALUES}; do
  SVN_LIB=$lib timeout 300 python bench.py --config c2 --steps 4 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | tail -n 1 | python scripts/benchline.py "$lib c2 fp32"
  SVN_LIB=$lib timeout 300 python bench.py --config c3 --precision fp32 --motions 64 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | tail -n 1 | python scripts/benchline.py "$lib c3net fp32 M=64"
done
done

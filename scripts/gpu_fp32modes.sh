for c in c3 c4; do for p in fp32 fp32_exact; do
timeout 600 python bench.py --config $c --precision $p --motions 32 --points 16384 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fm_${c}_$p.log 2>&1
tail -1 gpurun_out/fm_${c}_$p.log | python scripts/benchline.py "$c $p"
done; done

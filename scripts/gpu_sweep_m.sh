for m in ${MS:-16 32 64 128 256 512 1024}; do
  timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --config c2 --precision bf16 --motions $m > gpurun_out/sw_$m.log 2>&1
  python - "$m" <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/sw_{sys.argv[1]}.log").read().strip().splitlines()[-1])
r=d["roofline"]
print(sys.argv[1], f"{d['value']/1e6:.0f} Mq/s", "kernel_ms", round(r["kernel_ms"],4), "step_ms", round(d["ms_per_step"],4), "frac", round(r["frac"],3))
PY
done

for args in "--config paper" "--config paper --motions 1024" "--config paper --precision fp32" "--config paper --precision fp32 --motions 64"; do
  timeout 600 python bench.py $args --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/paper.log 2>&1
  python - "$args" <<'PY'
import json,sys
d=json.loads(open("gpurun_out/paper.log").read().strip().splitlines()[-1])
r=d["roofline"]; e=d.get("e2e") or {}
print(sys.argv[1], "|", f"{d['value']/1e6:.1f} Mq/s", f"step {d['ms_per_step']:.3f} ms", f"{r['achieved']:.0f} TF frac {r['frac']:.3f}", f"e2e {e.get('value',0)/1e6:.1f} Mq/s ({e.get('ms_per_step',0):.3f} ms)")
PY
done

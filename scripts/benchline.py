"""Print a compact summary of a bench.py JSON line read from stdin (label as argv[1])."""
import json
import sys

text = sys.stdin.read().strip()
label = sys.argv[1] if len(sys.argv) > 1 else ""
try:
    d = json.loads(text.splitlines()[-1])
except Exception:
    print(label, "NO JSON LINE:", text[-600:])
    sys.exit(0)
r = d.get("roofline") or {}
clk = (d.get("clocks") or {}).get("sm_mhz")
e = d.get("e2e") or {}
par = d.get("parity") or {}
ps = " ".join(f"{k}:mis{v.get('class_mismatches')}/amb{v.get('ambiguous')}/out{v.get('mismatches_outside_band')}"
              f"/err{v.get('max_abs_min_err', 0):.3g}" for k, v in par.items() if isinstance(v, dict))
print(label, f"{d['value'] / 1e6:.1f} Mq/s", f"step {d.get('ms_per_step', 0):.3f} ms",
      f"{r.get('achieved', 0):.0f} TF", f"frac {r.get('frac', 0):.3f}", f"clk {clk}",
      f"e2e {e.get('value', 0) / 1e6:.1f}", ps)

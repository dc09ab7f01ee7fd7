"""Print a compact summary of a bench.py JSON line read from stdin (label as argv[1])."""
import json
import sys

d = json.loads(sys.stdin.read().strip().splitlines()[-1])
r = d.get("roofline") or {}
clk = (d.get("clocks") or {}).get("sm_mhz")
print(sys.argv[1] if len(sys.argv) > 1 else "", f"{d['value'] / 1e6:.1f} Mq/s", f"{r.get('achieved', 0):.0f} TF",
      f"frac {r.get('frac', 0):.3f}", f"clk {clk}")

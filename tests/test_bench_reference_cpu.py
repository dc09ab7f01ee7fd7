"""bench.py's reference arm (the driver runs it next to ours on every round) on CPU: one
JSON line with the contract's keys, the CPU sample described, e2e with zero copies."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] and line["unit"] == "queries/s"
    assert line["value"] > 0 and line["higher_is_better"] is True and line["n_gpus"] == 1
    cb = line["cpu_baseline"]
    assert cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    if cb["kind"] == "reference":
        # the reference's own nn.cpp built here (oracle/_ref) on the Fig. 2 twin of the network, the
        # port on the config's own network alongside; the two agree bit for bit on the twin
        assert "Fig. 2 twin" in cb["network"] and cb["port_on_same_network"]["bits_equal"] is True
        port = cb["port"]
    else:
        port = cb
    assert port["kind"] == "port" and port["value"] > 0
    assert port["single_thread"]["cores"] == 1 and port["single_thread"]["value"] > 0
    assert line["e2e"] == {"value": line["value"], "unit": "queries/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["workload"] == "c1"


def test_reference_arm_loads_no_product_library():
    """The reference arm runs the oracle only: the product's native library must not be mapped."""
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c1', '--steps', '1', "
            "'--warmup', '0']\ntry:\n    runpy.run_path('bench.py', run_name='__main__')\nexcept SystemExit:\n    pass\n"
            "maps = open('/proc/self/maps').read()\nprint('PRODUCT_LOADED' if 'libsweptnet_b200' in maps else 'CLEAN')")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().splitlines()[-1] == "CLEAN"

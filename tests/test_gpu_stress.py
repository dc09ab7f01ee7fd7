"""A short run of scripts/stress.py: random (network, motions, points, margin) cases through the
host API in bf16 / fp16 / fp32_split against the bit-identical FP32 path (min within the frozen
bound, class outside the band) and the cascade's class on every motion.  The round-2 soak ran
7371 such cases (500 s) without a failure."""
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.gpu
def test_randomised_soak_20s():
    out = subprocess.run([sys.executable, str(ROOT / "scripts" / "stress.py"), "20", "7"], capture_output=True,
                         text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0 and "stress ok" in out.stdout, out.stdout[-2000:] + out.stderr[-2000:]

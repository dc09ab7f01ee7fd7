"""The reference-side binding of INTEGRATION.md compiles and links — against the REAL reference.

integration/sweptnet_b200.patch (guards nn.cpp's float forward_eval instantiation and the
predict_min_distance body, declares the forward_eval<float> specialisation in nn.hpp) applied
to an unmodified copy of /root/reference/proj, plus the shim integration/nn_b200.cpp, built
-DSWEPTNET_B200 with the rest of nn.cpp (forward_eval<double>, forward<float/double>, training)
and linked against libsweptnet_b200.so with a driver that calls the reference API
(oracle/ref/Makefile `dropin` -> oracle/_ref/ref_dropin_driver; it runs on the GPU in
tests/test_gpu_dropin.py).  INTEGRATION.md quotes both files verbatim.
"""
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = Path("/root/reference/proj")


def test_integration_md_quotes_the_tested_files():
    doc = (ROOT / "INTEGRATION.md").read_text()
    diff = re.findall(r"```diff\n(.*?)```", doc, flags=re.S)
    cpp = [b for b in re.findall(r"```cpp\n(.*?)```", doc, flags=re.S) if "src/nn_b200.cpp" in b.splitlines()[0]]
    assert diff == [(ROOT / "integration" / "sweptnet_b200.patch").read_text()]
    assert cpp == [(ROOT / "integration" / "nn_b200.cpp").read_text()]


@pytest.mark.skipif(not REF.exists(), reason="needs the reference sources (/root/reference)")
def test_patched_reference_compiles_and_links_against_the_product():
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle" / "ref"), "dropin"], check=True)
    exe = ROOT / "oracle" / "_ref" / "ref_dropin_driver"
    assert exe.exists()
    syms = subprocess.run(["nm", "-C", str(exe)], capture_output=True, text=True, check=True).stdout
    # the double path keeps the reference's CPU body; the float path and predict_min_distance
    # are the shim's and call the C-ABI
    assert "sweptnet::forward_eval<double>" in syms and "sweptnet::forward_eval<float>" in syms
    assert "svn_predict_min_distance" in syms and "svn_forward_eval" in syms
    dyn = subprocess.run(["ldd", str(exe)], capture_output=True, text=True, check=True).stdout
    assert "libsweptnet_b200.so" in dyn and "not found" not in dyn

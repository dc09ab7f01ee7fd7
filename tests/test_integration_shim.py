"""INTEGRATION.md's shim (the C++ file a maintainer adds to the reference) compiles against
include/sweptnet_b200.h: the code block is extracted from the document and built with g++
against a stand-in for the reference's nn.hpp interface (tests/cpp/mock_reference; Eigen is
absent here and on the GPU boxes), so the document cannot drift from the C-ABI."""
import re
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_integration_shim_compiles(tmp_path):
    doc = (ROOT / "INTEGRATION.md").read_text()
    blocks = re.findall(r"```cpp\n(.*?)```", doc, flags=re.S)
    shim = [b for b in blocks if "src/nn_b200.cpp" in b]
    assert len(shim) == 1, "INTEGRATION.md must hold exactly one src/nn_b200.cpp block"
    src = tmp_path / "nn_b200.cpp"
    src.write_text(shim[0])
    subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Werror", "-DSWEPTNET_B200",
                    f"-I{ROOT / 'tests/cpp/mock_reference'}", f"-I{ROOT / 'include'}", str(src)],
                   check=True, capture_output=False)

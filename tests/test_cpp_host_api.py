"""The C++ host API (include/sweptnet_b200.hpp) compiles against the C-ABI library and,
on a GPU, reproduces the reference's predict_min_distance / forward_eval relations."""
import subprocess
from pathlib import Path

import pytest

from paper_2402_15281_b200 import abi

ROOT = Path(__file__).resolve().parent.parent


def _build(tmp_path):
    abi.lib()  # make sure the library is built
    exe = tmp_path / "host_api_demo"
    libdir = abi.LIB_PATH.parent
    subprocess.run(["g++", "-std=c++17", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "tests/cpp/host_api_demo.cpp"),
                    f"-L{libdir}", "-lsweptnet_b200", f"-Wl,-rpath,{libdir}", "-o", str(exe)], check=True)
    return exe


def test_cpp_host_api_compiles(tmp_path):
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_cpp_host_api_runs(tmp_path):
    out = subprocess.run([str(_build(tmp_path))], capture_output=True, text=True, timeout=120)
    print(out.stdout, out.stderr)
    assert out.returncode == 0

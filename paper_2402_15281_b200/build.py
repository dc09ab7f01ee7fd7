"""Build the native library in-tree: paper_2402_15281_b200/_lib/libsweptnet_b200.so.

Every .cu under csrc/ is compiled for sm_100a only (tcgen05 / TMEM / bulk-async
copies are sm_100a features; there is no other target and no fallback) and
linked with a static CUDA runtime into one shared library exporting the C-ABI of
include/sweptnet_b200.h.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libsweptnet_b200.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-fvisibility=hidden,-O3",
    "-cudart", "static",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or Path(cand).exists()):
            return cand
    return "nvcc"


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*")) + [ROOT / "include" / "sweptnet_b200.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps if p.is_file())


def _defines() -> list[str]:
    # e.g. SVN_NVCC_DEFINES="SVN_KERNEL_PROF SVN_PP_TIMELINE" for the instrumented kernels
    return [f"-D{d}" for d in os.environ.get("SVN_NVCC_DEFINES", "").split() if d]


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    LIBDIR.mkdir(parents=True, exist_ok=True)
    # several processes may import the package at once (torchrun ranks): one builds under an
    # exclusive lock, the others wait and then find the library fresh
    import fcntl
    with open(LIBDIR / ".build.lock", "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        if not force and not _stale():
            return LIB
        return _build_locked(verbose)


def _build_locked(verbose: bool) -> Path:
    objs = []
    for src in sources():
        obj = LIBDIR / f"{src.stem}.{os.getpid()}.o"
        cmd = [nvcc(), *NVCC_FLAGS, *_defines(), "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    tmp = LIB.with_suffix(f".so.{os.getpid()}.tmp")
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
           "-o", str(tmp), *objs, "-lpthread", "-ldl", "-lrt"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))

"""Build an A/B variant of the native library: python scripts/build_variant.py OUT.so [file.cu=/path/alt.cu ...]

Copies csrc/ to a scratch directory, swaps in the given alternative sources, and builds
with the package's own flags (the result is used via SVN_LIB=scripts/ab/... with `scripts/gpu.sh ab`)."""
import shutil
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2402_15281_b200 import build as B  # noqa: E402

out = Path(sys.argv[1]).resolve()
tmp = Path(tempfile.mkdtemp())
shutil.copytree(B.CSRC, tmp / "pkg" / "csrc")
shutil.copytree(B.ROOT / "include", tmp / "include")
for spec in sys.argv[2:]:
    name, alt = spec.split("=", 1)
    shutil.copy(alt, tmp / "pkg" / "csrc" / name)
B.CSRC = tmp / "pkg" / "csrc"
B.LIBDIR = tmp / "lib"
B.LIB = out
B.build(force=True)
print(out)

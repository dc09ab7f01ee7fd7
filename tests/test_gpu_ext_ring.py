"""Width-512 bf16: the per-motion extension rows built inside the fused kernel (output warps,
per-CTA ring of two tile slots) give exactly the bits of the K0-built per-motion stream
(SVN_BF16_EXT=k0, the round-1 path; the ring is forced with SVN_BF16_EXT=ring — by default it is
used only when the per-motion stream would exceed L2, > 16 MB) — same fp32 fold, same splits, only where they live.
Covers dense queries with many tiles per motion (the ring slot is reused across tiles of a
motion), tiny clouds (every tile a new motion), forward_eval with mixed motions (tile table),
a trained-like Fig. 2 net with BN and non-identity normaliser, and the DeepSDF second concat."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import paper_2402_15281_b200 as S
from paper_2402_15281_b200.workloads import WORKLOADS
import ref_golden as G
out = {}
for key, M, P in (("c3", 5, 3000), ("c3", 40, 100), ("c4", 3, 2500)):
    w = WORKLOADS[key]
    pts, q = w.make(seed=7, motions=M, points=P)
    m = S.Model(w.program, S.init_params(w.program, 7, w.bound))
    r = m.query_min(pts, q, w.margin, precision="bf16", per_point=True)
    out[f"{key}_{M}_pp"] = r.per_point; out[f"{key}_{M}_min"] = r.min; out[f"{key}_{M}_arg"] = r.argmin
    nr = min(600, P)
    rows = np.concatenate([pts[:nr], q[np.arange(nr) % M]], axis=1).astype(np.float32)
    out[f"{key}_{M}_fwd"] = m.forward_eval(rows, precision="bf16")
Z, names = G.load()
g, prog, _, p = G.params(Z, "fig2_5x512_mknorm")
out["fig2"] = S.Model(prog, p).forward_eval(g["raw"], precision="bf16")
np.savez(sys.argv[2], **out)
"""


def _run(tmp_path, k0):
    env = dict(os.environ)
    env["SVN_BF16_EXT"] = "k0" if k0 else "ring"
    out = tmp_path / ("k0.npz" if k0 else "ring.npz")
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT), str(out)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


def test_in_kernel_extension_rows_bit_identical_to_k0_stream(tmp_path):
    ring, k0 = _run(tmp_path, False), _run(tmp_path, True)
    assert sorted(ring.files) == sorted(k0.files)
    for f in ring.files:
        assert np.array_equal(ring[f], k0[f]), f

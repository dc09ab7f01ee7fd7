"""Independent fp64 oracle of the layer program, in torch (CPU).

TEST INFRASTRUCTURE ONLY.  A second implementation that shares no code with
sweptnet_oracle.c: batched matrix products in float64 instead of per-row fma
chains, BN folded in float64.  Agreement with the C restatement (fp64 instance)
to ~1e-12 and with its fp32 instance to a few 1e-6 is the cross-check that the C
restatement encodes the reference semantics (/root/reference/proj/src/nn.cpp:95-130)
rather than a self-consistent mistake.
"""
from __future__ import annotations

import numpy as np
import torch


def unpack(program, params: np.ndarray):
    """Split the flat parameter buffer (layout: paper_2402_15281_b200/program.py)."""
    p = torch.as_tensor(np.asarray(params, dtype=np.float64))
    N, inn = program.width, program.input_dim
    o = 0
    shift = p[o:o + inn]; o += inn
    scale = p[o:o + inn]; o += inn
    layers = []
    for l, ly in enumerate(program.layers):
        K = program.layer_k(l)
        W = p[o:o + N * K].reshape(K, N).T  # column-major [N x K]
        o += N * K
        b = p[o:o + N]; o += N
        s = t = None
        if ly.affine:
            g, beta, mu, var = (p[o + i * N:o + (i + 1) * N] for i in range(4))
            o += 4 * N
            s = g / torch.sqrt(var + 1e-5)
            t = beta - mu * s
        layers.append((W, b, s, t))
    wo = p[o:o + N]; o += N
    bo = p[o]
    assert o + 1 == p.numel()
    return shift, scale, layers, wo, bo


def forward(program, params, raw) -> np.ndarray:
    shift, scale, layers, wo, bo = unpack(program, params)
    z = (torch.as_tensor(np.asarray(raw, dtype=np.float64)) - shift) * scale
    h = None
    for l, (ly, (W, b, s, t)) in enumerate(zip(program.layers, layers)):
        inp = z if l == 0 else (torch.cat([h, z], dim=1) if ly.concat else h)
        a = inp @ W.T + b
        r = torch.clamp(a, min=0.0) if ly.act else a
        if ly.affine:
            r = r * s + t
        h = h + r if (l > 0 and ly.residual) else r
    return (h @ wo + bo).numpy()


def query(program, params, points, q01) -> np.ndarray:
    """Per-point delta [M, P] for every motion."""
    pts = np.asarray(points, np.float64).reshape(-1, 3)
    q = np.asarray(q01, np.float64).reshape(-1, 2 * program.dof)
    out = np.empty((q.shape[0], pts.shape[0]))
    for m in range(q.shape[0]):
        raw = np.concatenate([pts, np.repeat(q[m][None], pts.shape[0], 0)], axis=1)
        out[m] = forward(program, params, raw)
    return out

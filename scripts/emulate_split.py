#!/usr/bin/env python3
"""CPU emulation of the fp32_split arithmetic on a plain or DeepSDF network (c2/c3/c4), to find
which part of the tensor-core path carries its error against the oracle: operand storage
(fp16 hi + lo'*2^-11 planes), the dropped lo'*lo' term, or the accumulation inside the
tensor core (one rounding per K=16 MMA instruction, round-to-nearest or toward zero).

    python scripts/emulate_split.py [--dump gpurun_out/split_dump.npz]

With --dump (per-point fp32_split output of the same seed from the GPU, scripts/split_dump.py)
it also reports how close each model comes to the GPU's bits."""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import oracle as O  # noqa: E402
from paper_2402_15281_b200.workloads import WORKLOADS  # noqa: E402

LO = 2.0 ** 11
BIASFIX = 0.0  # experiment: sign(main) * steps * ulp(main) * BIASFIX added to main


def split16(x):
    hi = x.astype(np.float16).astype(np.float64)
    lo = ((x.astype(np.float32) - hi.astype(np.float32)) * np.float32(LO)).astype(np.float16).astype(np.float64)
    return hi, lo


def split16_3(x):
    hi, lo = split16(x)
    r = x.astype(np.float64) - hi - lo / LO
    lo2 = (r * LO * LO).astype(np.float16).astype(np.float64)
    return hi, lo, lo2


def rz32(x):
    r = x.astype(np.float32)
    over = np.abs(r.astype(np.float64)) > np.abs(x)
    r[over] = np.nextafter(r[over], np.float32(0))
    return r


def rn32(x):
    return x.astype(np.float32)


def chain(blocks, rnd, init=None):
    """blocks: list of fp64 arrays (exact block sums); accumulate with one rounding per block."""
    acc = np.zeros_like(blocks[0], dtype=np.float32) if init is None else init
    for b in blocks:
        acc = rnd(acc.astype(np.float64) + b)
    return acc


def mm_blocks(a, w, kb=16):
    """exact per-K-block partial products: a [R, K] fp64, w [K, N] fp64 -> list of [R, N]"""
    K = a.shape[1]
    return [a[:, k:k + kb] @ w[k:k + kb] for k in range(0, K, kb)]


def out_dot(h, wo, bo):
    """the split kernel's output dot (width 256): epilogue thread ch of a row covers columns
    [64 ch, 64 ch + 64) of each 128-column n-half, in order, into four fp32 FMA partial sums
    (column mod 4); (x + y) + (z + w) per thread; delta = (thread 0 + thread 1) + b_o"""
    parts = []
    for ch in range(2):
        p = [np.zeros(h.shape[0], np.float32) for _ in range(4)]
        cols = list(range(64 * ch, 64 * ch + 64)) + list(range(128 + 64 * ch, 128 + 64 * ch + 64))
        for c in cols:
            p[c % 4] = (p[c % 4].astype(np.float64) + np.float64(wo[c]) * h[:, c].astype(np.float64)).astype(np.float32)
        parts.append((p[0] + p[1]) + (p[2] + p[3]))
    return ((parts[0] + parts[1]) + np.float32(bo)).astype(np.float32)


def run(prog, params, pts, q, model, rnd, halves=1):
    N, dof = prog.width, prog.dof
    in_ = 3 + 2 * dof
    p = params.astype(np.float32)
    shift, scale = p[:in_], p[in_:2 * in_]
    off = 2 * in_
    Ws, bs = [], []
    for l in range(prog.n_layers):
        K = prog.layer_k(l)
        Ws.append(p[off:off + N * K].reshape(K, N))  # [K, N]: row k = column k of W
        off += N * K
        bs.append(p[off:off + N])
        off += N
        assert not prog.layers[l].affine
    wo, bo = p[off:off + N], p[off + N]
    M, P = q.shape[0], pts.shape[0]
    out = np.zeros((M, P), np.float32)
    zx = ((pts - shift[:3]) * scale[:3]).astype(np.float32)
    for m in range(M):
        zq = ((q[m] - shift[3:]) * scale[3:]).astype(np.float32)
        zh, zl = split16(zx)
        h = None
        for l in range(prog.n_layers):
            K = Ws[l].shape[0]
            ly = prog.layers[l]
            # concat layers: b_m = b + Wq.zq in fp32 FMA order (K0), x part through the K=16 extension
            if l == 0 or ly.concat:
                bm = bs[l].copy()
                xo = 0 if l == 0 else N
                for k in range(2 * dof):
                    bm = (bm.astype(np.float64) + np.float64(zq[k]) * Ws[l][xo + 3 + k].astype(np.float64)).astype(np.float32)
                wxr = Ws[l][xo:xo + 3]
            else:
                bm, wxr = bs[l], np.zeros((3, N), np.float32)
            if model == "exact":
                a = zx.astype(np.float64) @ wxr.astype(np.float64) + bm
                if h is not None:
                    a = a + h.astype(np.float64) @ Ws[l][:N].astype(np.float64)
                v = a.astype(np.float32)
            else:
                bh, bl = split16(bm)
                wxh, wxl = split16(wxr)
                ext_main = bh[None, :] + zh @ wxh
                ext_corr = bl[None, :] + zh @ wxl + zl @ wxh
                if h is None:
                    main, corr = rnd(ext_main), rnd(ext_corr)
                elif model == "split_exactacc":
                    ah, al = split16(h)
                    wh, wl = split16(Ws[l][:N])
                    main = (ext_main + ah @ wh).astype(np.float32)
                    corr = (ext_corr + ah @ wl + al @ wh).astype(np.float32)
                else:
                    ah, al = split16(h)
                    wh, wl = split16(Ws[l][:N])
                    step = N // halves
                    parts = []
                    for i, s0 in enumerate(range(0, N, step)):
                        blocks = ([ext_main] if i == 0 else []) + mm_blocks(ah[:, s0:s0 + step], wh[s0:s0 + step])
                        parts.append(chain(blocks, rnd))
                    cb = [ext_corr]
                    for s0 in range(0, N, 16):
                        cb.append(ah[:, s0:s0 + 16] @ wl[s0:s0 + 16])
                        cb.append(al[:, s0:s0 + 16] @ wh[s0:s0 + 16])
                    corr = chain(cb, rnd)
                    main = parts[0]
                    for x in parts[1:]:
                        main = (main.astype(np.float64) + x).astype(np.float32)
                    if BIASFIX:
                        md = main.astype(np.float64)
                        ulp = np.spacing(np.abs(main)).astype(np.float64)
                        main = (md + np.sign(md) * (N // 16 + 1) * ulp * BIASFIX).astype(np.float32)
                v = (main.astype(np.float64) + corr.astype(np.float64) / LO).astype(np.float32)
            h = np.maximum(v, 0) if ly.act else v
        out[m] = out_dot(h, wo, bo) if model != "exact" else (h.astype(np.float64) @ wo.astype(np.float64) + bo).astype(np.float32)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--motions", type=int, default=4)
    ap.add_argument("--points", type=int, default=4096)
    ap.add_argument("--dump", default=None)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--biasfix", type=float, default=0.0)
    a = ap.parse_args()
    global BIASFIX
    BIASFIX = a.biasfix
    w = WORKLOADS[a.config]
    prog = w.program
    pts, q = w.make(seed=a.seed, motions=16, points=a.points)
    q = q[:a.motions]
    params = O.init_params(prog, a.seed, w.bound)
    _, _, _, opp = O.query_min(prog, params, pts, q, w.margin, per_point=True, threads=8)
    M = q.shape[0]
    raw = np.concatenate([np.repeat(pts[None].astype(np.float64), M, 0).reshape(-1, 3),
                          np.repeat(q.reshape(M, 1, -1).astype(np.float64), pts.shape[0], 1).reshape(M * pts.shape[0], -1)], 1)
    f64 = O.forward_eval(prog, params.astype(np.float64), raw, np.float64).reshape(M, -1)
    gpu = None
    if a.dump:
        d = np.load(a.dump)
        gpu = d["per_point"][:M]
    print(f"|delta| max {np.abs(f64).max():.3f}; oracle f32 vs f64 {np.abs(opp - f64).max():.3e}")
    for name, model, rnd, halves in [("exact fp32 products, one rounding", "exact", rn32, 1),
                                     ("split storage, exact accumulation", "split_exactacc", rn32, 1),
                                     ("split, RN per MMA", "split", rn32, 1),
                                     ("split, RZ per MMA", "split", rz32, 1),
                                     ("split, RZ per MMA, main in 2 K-halves", "split", rz32, 2),
                                     ("split, RZ per MMA, main in 4 K-quarters", "split", rz32, 4)]:
        e = run(prog, params, pts, q, model, rnd, halves)
        line = (f"{name:45s} vs oracle {np.abs(e - opp).max():.3e}  vs f64 {np.abs(e - f64).max():.3e}")
        if gpu is not None:
            line += f"  vs GPU {np.abs(e - gpu).max():.3e} (bit-equal {np.mean(e == gpu) * 100:.1f}%)"
        print(line, flush=True)
    if gpu is not None:
        print(f"{'GPU fp32_split':45s} vs oracle {np.abs(gpu - opp).max():.3e}  vs f64 {np.abs(gpu - f64).max():.3e}")


if __name__ == "__main__":
    main()

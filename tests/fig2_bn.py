"""Fig. 2 networks with non-trivial BatchNorm statistics (as a trained SVCKPT01 checkpoint
would carry): helper shared by the GPU tests of the bf16 affine fold."""
import numpy as np


def randomize_bn(program, params, seed, negative_gamma_layer=None):
    """Return a copy of params with random biases and BN (gamma, beta, mean, var) on every
    affine layer; optionally one layer gets a negative gamma in some columns."""
    rng = np.random.default_rng(seed)
    p = params.copy()
    N, in_ = program.width, 3 + 2 * program.dof
    off = 2 * in_
    for l, ly in enumerate(program.layers):
        K = in_ if l == 0 else N + (in_ if ly.concat else 0)
        off += N * K
        p[off:off + N] = rng.uniform(-0.1, 0.1, N)  # bias
        off += N
        if ly.affine:
            g = rng.uniform(0.5, 1.5, N)
            if negative_gamma_layer == l:
                g[: N // 8] *= -1.0
            p[off:off + N] = g
            p[off + N:off + 2 * N] = rng.uniform(-0.2, 0.2, N)      # beta
            p[off + 2 * N:off + 3 * N] = rng.uniform(-0.2, 0.2, N)  # running mean
            p[off + 3 * N:off + 4 * N] = rng.uniform(0.5, 2.0, N)   # running var
            off += 4 * N
    p[off + N] = 0.05  # output bias
    return p.astype(np.float32)

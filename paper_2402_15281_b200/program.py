"""Layer programs: the network families the hot path evaluates.

The reference's MlpT (/root/reference/proj/include/sweptnet/nn.hpp:16-44) is the
paper's Fig. 2 residual network only.  BASELINE.json's configs also name plain
MLPs and a DeepSDF-style MLP, which MlpT cannot express.  A *program* is a list
of hidden layers with flags {concat, act, affine, residual}; the C-ABI and the
oracle both consume it, so every family runs through one kernel.

Parameter buffer layout (floats), shared with include/sweptnet_b200.h:
    norm_shift[in], norm_scale[in],
    per layer l: W_l column-major [N x K_l], b_l[N], (+ gamma, beta, mean, var if affine)
    output_weight[N], output_bias
K_0 = in; K_l = N + concat_l * in.  For Fig. 2 this is the SVCKPT01 body (nn.cpp:507-520).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Layer:
    concat: bool
    act: bool
    affine: bool = False
    residual: bool = False

    def flags(self) -> tuple[int, int, int, int]:
        return (int(self.concat), int(self.act), int(self.affine), int(self.residual))


@dataclass(frozen=True)
class LayerProgram:
    name: str
    width: int
    dof: int
    layers: tuple[Layer, ...] = field(default_factory=tuple)

    @property
    def input_dim(self) -> int:
        return 3 + 2 * self.dof

    @property
    def n_layers(self) -> int:
        return len(self.layers)

    def flags_array(self) -> np.ndarray:
        return np.array([l.flags() for l in self.layers], dtype=np.int32).reshape(-1)

    def layer_k(self, l: int) -> int:
        if l == 0:
            return self.input_dim
        return self.width + (self.input_dim if self.layers[l].concat else 0)

    def param_floats(self) -> int:
        n, N = 2 * self.input_dim, self.width
        for l, ly in enumerate(self.layers):
            n += N * self.layer_k(l) + N + (4 * N if ly.affine else 0)
        return n + N + 1

    def trainable_params(self) -> int:
        """MlpT::param_count (nn.cpp:19-24)."""
        n, N = 0, self.width
        for l, ly in enumerate(self.layers):
            n += N * self.layer_k(l) + N + (2 * N if ly.affine else 0)
        return n + N + 1

    # FLOPs per (point x motion) query after the per-motion q-fold:
    # 2*3*N for layer 0's x part, 2*N*(N + 3*concat) per hidden layer, 2*N output.
    def flops_per_query(self) -> int:
        N = self.width
        f = 2 * 3 * N
        for ly in self.layers[1:]:
            f += 2 * N * (N + (3 if ly.concat else 0))
        return f + 2 * N

    def tensor_flops_per_query(self) -> int:
        """The width x width part, the part that runs on tcgen05."""
        return 2 * self.width * self.width * (self.n_layers - 1)

    def weight_bytes(self, dtype_bytes: int) -> int:
        return (self.n_layers - 1) * self.width * self.width * dtype_bytes


def fig2(n_blocks: int, width: int, dof: int) -> LayerProgram:
    """The reference network (nn.hpp:11-15, nn.cpp:116-128): input linear, then
    n_blocks x [Linear([h; z]) -> ReLU -> BN -> + h]."""
    layers = [Layer(concat=True, act=False)] + [Layer(True, True, True, True)] * n_blocks
    return LayerProgram(f"fig2_{n_blocks}x{width}", width, dof, tuple(layers))


def plain(hidden: int, width: int, dof: int) -> LayerProgram:
    """Plain MLP: `hidden` ReLU layers of `width` (BASELINE.json configs 0, 1, 3)."""
    layers = [Layer(concat=True, act=True)] + [Layer(concat=False, act=True)] * (hidden - 1)
    return LayerProgram(f"plain_{hidden}x{width}", width, dof, tuple(layers))


def deepsdf(hidden: int, width: int, dof: int, skip_at: int = 4) -> LayerProgram:
    """DeepSDF-style MLP: plain, with the input re-concatenated at layer `skip_at`
    (BASELINE.json configs 2 and 4)."""
    layers = [Layer(concat=True, act=True)]
    for l in range(1, hidden):
        layers.append(Layer(concat=(l == skip_at), act=True))
    return LayerProgram(f"deepsdf_{hidden}x{width}_skip{skip_at}", width, dof, tuple(layers))

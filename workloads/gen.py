"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO K-FAC arithmetic.  It draws the *inputs* of the
preconditioner - the captured layer inputs a_{i-1}, the output gradients g_i
("save the activation of the previous layer and gradient with
respect to the output") and the averaged weight gradient grad L_i (Alg. 1,
P:341) - with the distributions fixed in DESIGN.md "Input recipe":

  * network inputs: N(0,1) for conv1 (normalised images), U[0,1) for the MLP's
    fc1 (pixel-like);
  * hidden-layer inputs: ReLU(N(0,1));
  * output gradients: N(0, 1/d_G) (unit expected squared norm per row);
  * weight gradient: the layer's backprop weight gradient of those g and a,
    grad = g^T [patches | 1] / n, produced by the *library* convolution
    weight-gradient (torch.nn.grad.conv2d_weight) in fp64 and rounded to fp32
    once, laid out (C_out, k_h, k_w, C_in | bias) to match the (k_h, k_w, c)
    patch-column convention (reading R8).

Every tensor is drawn from numpy's counter-based Philox generator keyed on
(seed, rank, layer, tensor-kind), so both sides see bit-identical fp32 inputs.
"""
from __future__ import annotations

import numpy as np

from .shapes import Layer, LINEAR

KIND_ACT, KIND_GOUT = 1, 2


def rng(seed: int, rank: int, layer: int, kind: int) -> np.random.Generator:
    key = (int(rank) << 40) | (int(layer) << 8) | int(kind)
    return np.random.Generator(np.random.Philox(key=[int(seed) & (2**64 - 1), key]))


def activations(layer: Layer, idx: int, seed: int = 0, rank: int = 0,
                first_dist: str | None = None) -> np.ndarray:
    """a_{i-1} for layer `idx`: NHWC (conv) or (rows, C_in) (linear), fp32."""
    g = rng(seed, rank, idx, KIND_ACT)
    shape = layer.act_shape
    if idx == 0:
        dist = first_dist or ("uniform" if layer.kind == LINEAR else "normal")
        if dist == "uniform":
            return g.random(shape, dtype=np.float32)
        return g.standard_normal(shape, dtype=np.float32)
    x = g.standard_normal(shape, dtype=np.float32)
    np.maximum(x, 0.0, out=x)
    return x


def output_grads(layer: Layer, idx: int, seed: int = 0, rank: int = 0,
                 sigma: float | None = None) -> np.ndarray:
    """g_i: (rows, C_out) fp32 ~ N(0, sigma^2), sigma = 1/sqrt(d_G) by default."""
    g = rng(seed, rank, idx, KIND_GOUT)
    x = g.standard_normal(layer.gout_shape, dtype=np.float32)
    s = np.float32(sigma if sigma is not None else 1.0 / np.sqrt(layer.d_g))
    x *= s
    return x


def weight_grad(layer: Layer, act: np.ndarray, gout: np.ndarray, device: str = "cpu") -> np.ndarray:
    """Backprop weight gradient of the layer (library ops, fp64), fp32 result.

    Layout: (d_G, d_A) row-major, columns (k_h, k_w, c_in) then the bias column.
    """
    import torch
    n = layer.rows
    g = torch.from_numpy(gout).to(device=device, dtype=torch.float64)
    if layer.kind == LINEAR:
        x = torch.from_numpy(act).to(device=device, dtype=torch.float64)
        w = g.t() @ x
    else:
        x = torch.from_numpy(act).to(device=device, dtype=torch.float64).permute(0, 3, 1, 2)
        go = g.reshape(layer.batch, layer.h_out, layer.w_out, layer.c_out).permute(0, 3, 1, 2)
        w = torch.nn.grad.conv2d_weight(
            x.contiguous(), (layer.c_out, layer.c_in, layer.k_h, layer.k_w), go.contiguous(),
            stride=(layer.stride_h, layer.stride_w), padding=(layer.pad_h, layer.pad_w))
        w = w.permute(0, 2, 3, 1).reshape(layer.c_out, -1)      # (C_out, kh, kw, C_in)
    if layer.bias_col:
        w = torch.cat([w, g.sum(0, keepdim=True).t()], dim=1)
    w = (w / n).to(torch.float32).cpu().numpy()
    return np.ascontiguousarray(w)


def layer_inputs(layers, seed: int = 0, rank: int = 0, with_grad: bool = True, device: str = "cpu",
                 sigma: float | None = None):
    """Lists (act, gout, grad) for every layer of a config."""
    acts, gouts, grads = [], [], []
    for i, l in enumerate(layers):
        a = activations(l, i, seed, rank)
        g = output_grads(l, i, seed, rank, sigma)
        acts.append(a)
        gouts.append(g)
        if with_grad:
            grads.append(weight_grad(l, a, g, device))
    return acts, gouts, grads


def random_spd(d: int, seed: int, rank_deficit: int = 0, scale: float = 1.0) -> np.ndarray:
    """Seeded random symmetric PSD matrix X^T X / m (fp64), used by unit tests."""
    g = np.random.Generator(np.random.Philox(key=[seed, 0xE16]))
    m = max(1, d - rank_deficit) if rank_deficit else d + 3
    x = g.standard_normal((m, d))
    return scale * (x.T @ x) / m


def random_matrix(shape, seed: int, kind: int = 7) -> np.ndarray:
    g = np.random.Generator(np.random.Philox(key=[seed, 0xA000 + kind]))
    return g.standard_normal(shape)

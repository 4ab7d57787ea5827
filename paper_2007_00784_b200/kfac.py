"""KFAC(model): the paper's user-facing preconditioner (Listing 1) on top of the
C-ABI path.

    preconditioner = KFAC(model, lr=0.1, damping=1e-3, ...)
    for data, target in loader:
        optimizer.zero_grad()
        loss = criterion(model(data), target)
        loss.backward()              # (+ the data-parallel gradient allreduce, Alg. 1)
        preconditioner.step()        # weight/bias gradients replaced by their K-FAC preconditioned
        optimizer.step()             #   values in place

What it does (every arithmetic step runs in libkfac's kernels through KFACPreconditioner):
  * Linear and Conv2D layers only; groups = 1, dilation = 1, zero padding.
  * Forward pre-hooks save each layer's input a_{i-1}, full backward hooks save the gradient with
    respect to its output g_i -- only on iterations whose factors are updated.
  * Layouts are marshalled for the ABI: activations NHWC (a free view when the model runs
    channels_last), output gradients (rows x C_out), the weight gradient as (C_out, k_h, k_w, C_in)
    with the bias gradient as the last column (R8); the result is written back into
    `weight.grad` / `bias.grad`.
  * Output gradients are multiplied by the batch size (grad_scale="batch"): with a mean-reduced loss
    backprop hands every sample a 1/N-scaled gradient, and G = g^T g / n needs per-sample gradients
    (R6 leaves this scaling to the caller; this is that caller).
  * Schedules: factors every `factor_update_freq` steps, eigendecompositions every
    `kfac_update_freq` steps (the paper refreshes factors 10x as often, R17); damping multiplied by
    `damping_decay_rate` at each step in `damping_decay_steps`; kfac_update_freq multiplied by
    `update_freq_decay_rate` at each step in `update_freq_decay_steps`.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence

import torch
import torch.nn as nn

from .preconditioner import KFACPreconditioner

LINEAR, CONV2D = 0, 1


class LayerDesc:
    """Same fields as workloads.shapes.Layer / kfac_layer_t (the ABI's layer descriptor)."""

    __slots__ = ("name", "kind", "batch", "c_in", "h_in", "w_in", "c_out", "h_out", "w_out", "k_h", "k_w",
                 "stride_h", "stride_w", "pad_h", "pad_w", "bias_col")

    def __init__(self, **kw):
        for k in self.__slots__:
            setattr(self, k, kw[k])

    @property
    def rows(self):
        return self.batch * self.h_out * self.w_out

    @property
    def d_a(self):
        return self.c_in * self.k_h * self.k_w + self.bias_col

    @property
    def d_g(self):
        return self.c_out

    def as_tuple(self):
        return tuple(getattr(self, k) for k in self.__slots__[1:])


def _pair(v):
    return (v, v) if isinstance(v, int) else tuple(v)


def supported(m: nn.Module) -> bool:
    if isinstance(m, nn.Linear):
        return True
    if isinstance(m, nn.Conv2d):
        return (m.groups == 1 and _pair(m.dilation) == (1, 1) and m.padding_mode == "zeros"
                and not isinstance(m.padding, str))
    return False


class KFAC:
    def __init__(self, model: nn.Module, lr: float = 0.1, damping: float = 1e-3, xi: float = 0.95,
                 kappa: float = 1e-3, kfac_update_freq: int = 10, factor_update_freq: int = 1,
                 damping_decay_steps: Sequence[int] = (), damping_decay_rate: float = 0.5,
                 update_freq_decay_steps: Sequence[int] = (), update_freq_decay_rate: float = 1.0,
                 variant: str = "eigen", exchange: str = "bcast-eig", grad_scale: str = "batch",
                 process_group=None, skip_modules: Sequence[nn.Module] = (), factor_comm: str = "allreduce"):
        self.model = model
        self.lr, self.damping, self.xi, self.kappa = lr, damping, xi, kappa
        self.kfac_update_freq, self.factor_update_freq = int(kfac_update_freq), int(factor_update_freq)
        self.damping_decay_steps = set(int(s) for s in damping_decay_steps)
        self.damping_decay_rate = damping_decay_rate
        self.update_freq_decay_steps = set(int(s) for s in update_freq_decay_steps)
        self.update_freq_decay_rate = update_freq_decay_rate
        self.variant, self.exchange, self.grad_scale = variant, exchange, grad_scale
        self.process_group = process_group
        self.factor_comm = factor_comm
        skip = set(id(m) for m in skip_modules)
        self.modules: List[nn.Module] = [m for m in model.modules() if supported(m) and id(m) not in skip]
        self.names = {id(m): n for n, m in model.named_modules()}
        self._acts: Dict[int, torch.Tensor] = {}
        self._gouts: Dict[int, torch.Tensor] = {}
        self._handles = []
        for m in self.modules:
            self._handles.append(m.register_forward_pre_hook(self._save_input))
            self._handles.append(m.register_full_backward_hook(self._save_grad_output))
        self.steps = 0
        self.pc: Optional[KFACPreconditioner] = None
        self._grads = self._grad_flat = None
        self._seeded = False

    # ------------------------------------------------------------------ hooks --
    def _capturing(self) -> bool:
        return self.model.training and torch.is_grad_enabled() and self.steps % self.factor_update_freq == 0

    def _save_input(self, module, inputs):
        if self._capturing():
            self._acts[id(module)] = inputs[0].detach()

    def _save_grad_output(self, module, grad_input, grad_output):
        # autograd runs backward hooks with grad mode off: capture whenever the forward did
        if id(module) in self._acts:
            self._gouts[id(module)] = grad_output[0].detach()

    # ------------------------------------------------------------- marshalling --
    def _describe(self, m: nn.Module, a: torch.Tensor, g: torch.Tensor) -> LayerDesc:
        bias = int(m.bias is not None)
        if isinstance(m, nn.Linear):
            rows = a.numel() // a.shape[-1]
            return LayerDesc(name=self.names[id(m)], kind=LINEAR, batch=rows, c_in=m.in_features, h_in=1, w_in=1,
                             c_out=m.out_features, h_out=1, w_out=1, k_h=1, k_w=1, stride_h=1, stride_w=1,
                             pad_h=0, pad_w=0, bias_col=bias)
        kh, kw = _pair(m.kernel_size)
        sh, sw = _pair(m.stride)
        ph, pw = _pair(m.padding)
        return LayerDesc(name=self.names[id(m)], kind=CONV2D, batch=a.shape[0], c_in=m.in_channels,
                         h_in=a.shape[2], w_in=a.shape[3], c_out=m.out_channels, h_out=g.shape[2], w_out=g.shape[3],
                         k_h=kh, k_w=kw, stride_h=sh, stride_w=sw, pad_h=ph, pad_w=pw, bias_col=bias)

    @staticmethod
    def _act_nhwc(m, a):
        if isinstance(m, nn.Linear):
            return a.reshape(-1, a.shape[-1]).float().contiguous()
        # free when the model runs channels_last (the NCHW tensor is then NHWC in memory)
        return a.float().permute(0, 2, 3, 1).contiguous()

    def _gout_rows(self, m, g, batch):
        scale = float(batch) if self.grad_scale == "batch" else 1.0
        if isinstance(m, nn.Linear):
            x = g.reshape(-1, g.shape[-1]).float()
        else:
            x = g.float().permute(0, 2, 3, 1).reshape(-1, g.shape[1])
        return (x * scale).contiguous() if scale != 1.0 else x.contiguous()

    @staticmethod
    def _weight_grad_2d(m):
        w = m.weight.grad
        if isinstance(m, nn.Conv2d):
            w = w.permute(0, 2, 3, 1)
        return w.reshape(w.shape[0], -1)

    # -------------------------------------------------------------------- step --
    def _build(self, descs):
        self.pc = KFACPreconditioner(descs, damping=self.damping, xi=self.xi, kappa=self.kappa, lr=self.lr,
                                     variant=self.variant, exchange=self.exchange, process_group=self.process_group,
                                     factor_comm=self.factor_comm)
        self._grads, self._grad_flat = KFACPreconditioner.grad_buffer(descs, self.pc.device, return_flat=True)

    def _schedules(self):
        if self.steps in self.damping_decay_steps:
            self.damping *= self.damping_decay_rate
        if self.steps in self.update_freq_decay_steps:
            self.kfac_update_freq = max(1, int(round(self.kfac_update_freq * self.update_freq_decay_rate)))

    @torch.no_grad()
    def step(self, lr: Optional[float] = None):
        """Precondition every registered layer's gradient in place (call after backward, before
        optimizer.step()).  lr: the current learning rate for the KL-clip (Eq. 18)."""
        if lr is not None:
            self.lr = lr
        self._schedules()
        update_factors = self.steps % self.factor_update_freq == 0
        if update_factors:
            missing = [self.names[id(m)] for m in self.modules if id(m) not in self._gouts]
            if missing:
                raise RuntimeError(f"KFAC.step(): no captured activations/gradients for {missing[:4]} "
                                   "(call after loss.backward() in training mode)")
            descs = [self._describe(m, self._acts[id(m)], self._gouts[id(m)]) for m in self.modules]
            if self.pc is None:
                self._build(descs)
            else:
                self.pc.layers = descs        # batch/rows may change; factor dimensions do not
        elif self.pc is None:
            raise RuntimeError("KFAC.step(): the first step must update the factors")
        pc = self.pc
        pc.damping, pc.kappa, pc.lr = self.damping, self.kappa, self.lr
        for m, gbuf in zip(self.modules, self._grads):
            w = self._weight_grad_2d(m)
            gbuf[:, :w.shape[1]].copy_(w)
            if m.bias is not None:
                gbuf[:, w.shape[1]].copy_(m.bias.grad)
        refresh = self.steps % self.kfac_update_freq == 0 or not pc.have_eigen
        if refresh and not update_factors and pc.reduce_owner:
            raise RuntimeError("KFAC.step(): factor_comm='reduce-owner' needs the factors updated on every "
                               "eigen-refresh step (kfac_update_freq a multiple of factor_update_freq)")
        if update_factors:
            acts = [self._act_nhwc(m, self._acts[id(m)]) for m in self.modules]
            gouts = [self._gout_rows(m, self._gouts[id(m)], self._acts[id(m)].shape[0]) for m in self.modules]
            pc.update_factors(acts, gouts, first=not self._seeded, refresh=refresh)
            self._seeded = True
            self._acts.clear()
            self._gouts.clear()
        if refresh:
            pc.compute_eigen()
        P = pc.precondition(self._grads)
        for m, p in zip(self.modules, P):
            w = m.weight.grad
            nw = self._weight_grad_2d(m).shape[1]
            if isinstance(m, nn.Conv2d):
                kh, kw = _pair(m.kernel_size)
                w.copy_(p[:, :nw].reshape(w.shape[0], kh, kw, w.shape[1]).permute(0, 3, 1, 2))
            else:
                w.copy_(p[:, :nw].reshape(w.shape))
            if m.bias is not None:
                m.bias.grad.copy_(p[:, nw])
        self.steps += 1
        return P

    def remove_hooks(self):
        for h in self._handles:
            h.remove()
        self._handles = []

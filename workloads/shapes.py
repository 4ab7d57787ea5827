"""Layer tables of the paper's workloads (shapes only, no K-FAC arithmetic).

The paper preconditions Linear and Conv2D layers only (PAPER.md:417-418,
Sec. V "Our implementation supports K-FAC updates for Linear and Conv2D
layers").  The configurations are BASELINE.json's `configs`:

  mlp   : 2-layer MLP 784->64->10, batch 128                (configs[0])
  r32   : ResNet-32 / CIFAR-10 32x32, batch 128 per GPU      (configs[1])
  r50   : ResNet-50 / ImageNet 224x224, batch 32 per GPU     (configs[2])
  r101  : ResNet-101 / ImageNet 224x224, batch 32 per GPU    (configs[4])
  r152  : ResNet-152 (Table V's third model)      (context only)

ResNet-50/101/152 follow the torchvision v1.5 layout (stride on the 3x3 conv;
DESIGN.md reading R18).  ResNet-32 uses the parameter-free option-A shortcuts
of He et al. (31 convs + 1 fc).  Each layer is a `Layer` with the same field
meaning as `kfac_layer_t` in include/kfac.h, in torchvision module order
(conv1, bn, conv2, conv3, downsample per block, fc last).
"""
from __future__ import annotations

from dataclasses import dataclass, asdict
from typing import List

LINEAR = 0
CONV2D = 1


@dataclass(frozen=True)
class Layer:
    name: str
    kind: int           # LINEAR or CONV2D
    batch: int          # N (images) for conv; rows for linear
    c_in: int
    h_in: int
    w_in: int
    c_out: int
    h_out: int
    w_out: int
    k_h: int
    k_w: int
    stride_h: int
    stride_w: int
    pad_h: int
    pad_w: int
    bias_col: int = 1   # append the homogeneous ones column

    @property
    def rows(self) -> int:
        """n = N * H_out * W_out."""
        return self.batch * self.h_out * self.w_out

    @property
    def d_a(self) -> int:
        return self.c_in * self.k_h * self.k_w + self.bias_col

    @property
    def d_g(self) -> int:
        return self.c_out

    @property
    def act_shape(self):
        if self.kind == LINEAR:
            return (self.batch, self.c_in)
        return (self.batch, self.h_in, self.w_in, self.c_in)   # NHWC

    @property
    def gout_shape(self):
        return (self.rows, self.c_out)

    @property
    def grad_shape(self):
        return (self.d_g, self.d_a)

    def as_tuple(self):
        d = asdict(self)
        d.pop("name")
        return tuple(d.values())


def linear(name, batch, fin, fout, bias_col=1) -> Layer:
    return Layer(name, LINEAR, batch, fin, 1, 1, fout, 1, 1, 1, 1, 1, 1, 0, 0, bias_col)


def conv(name, batch, cin, cout, k, stride, hin, bias_col=1) -> Layer:
    pad = k // 2
    hout = (hin + 2 * pad - k) // stride + 1
    return Layer(name, CONV2D, batch, cin, hin, hin, cout, hout, hout, k, k,
                 stride, stride, pad, pad, bias_col)


def mlp(batch: int = 128) -> List[Layer]:
    return [linear("fc1", batch, 784, 64), linear("fc2", batch, 64, 10)]


def resnet32(batch: int = 128) -> List[Layer]:
    layers = [conv("conv1", batch, 3, 16, 3, 1, 32)]
    h, cin = 32, 16
    for stage, cout in enumerate((16, 32, 64)):
        for blk in range(5):
            s = 2 if (blk == 0 and stage > 0) else 1
            layers.append(conv(f"layer{stage+1}.{blk}.conv1", batch, cin, cout, 3, s, h))
            h = layers[-1].h_out
            layers.append(conv(f"layer{stage+1}.{blk}.conv2", batch, cout, cout, 3, 1, h))
            cin = cout
    layers.append(linear("fc", batch, 64, 10))
    return layers


def _bottleneck_resnet(blocks, batch: int, num_classes: int = 1000) -> List[Layer]:
    layers = [conv("conv1", batch, 3, 64, 7, 2, 224)]
    h = 56                      # after 3x3/2 max-pool
    cin = 64
    for li, (planes, nblk) in enumerate(zip((64, 128, 256, 512), blocks)):
        for b in range(nblk):
            s = 2 if (b == 0 and li > 0) else 1
            p = f"layer{li+1}.{b}"
            layers.append(conv(p + ".conv1", batch, cin, planes, 1, 1, h))
            layers.append(conv(p + ".conv2", batch, planes, planes, 3, s, h))
            h2 = layers[-1].h_out
            layers.append(conv(p + ".conv3", batch, planes, planes * 4, 1, 1, h2))
            if b == 0:
                layers.append(conv(p + ".downsample", batch, cin, planes * 4, 1, s, h))
            cin = planes * 4
            h = h2
    layers.append(linear("fc", batch, 2048, num_classes))
    return layers


def resnet50(batch: int = 32) -> List[Layer]:
    return _bottleneck_resnet((3, 4, 6, 3), batch)


def resnet101(batch: int = 32) -> List[Layer]:
    return _bottleneck_resnet((3, 4, 23, 3), batch)


def resnet152(batch: int = 32) -> List[Layer]:
    return _bottleneck_resnet((3, 8, 36, 3), batch)


CONFIGS = {
    "mlp": mlp,
    "r32": resnet32,
    "r50": resnet50,
    "r101": resnet101,
    "r152": resnet152,
}

# Hyper-parameters per config: damping gamma, xi (weight
# on the new batch estimate, reading R5), kappa, lr.
HPARAMS = {
    "mlp": dict(damping=3e-3, xi=0.95, kappa=1e-3, lr=0.1),
    "r32": dict(damping=3e-3, xi=0.95, kappa=1e-3, lr=0.1),      # lr = W*0.1
    "r50": dict(damping=1e-3, xi=0.95, kappa=1e-3, lr=0.0125),   # gamma P:542/P:610; lr W*0.0125
    "r101": dict(damping=1e-3, xi=0.95, kappa=1e-3, lr=0.0125),
    "r152": dict(damping=1e-3, xi=0.95, kappa=1e-3, lr=0.0125),
}


def layers_for(config: str, batch: int | None = None) -> List[Layer]:
    fn = CONFIGS[config]
    return fn() if batch is None else fn(batch)


def factor_dims(layers: List[Layer]):
    """Factor list in the paper's interleaved order [A_0, G_0, A_1, G_1, ...]
     -> (dims, layer_of_factor)."""
    dims, layer_of = [], []
    for i, l in enumerate(layers):
        dims += [l.d_a, l.d_g]
        layer_of += [i, i]
    return dims, layer_of

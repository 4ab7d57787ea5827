"""GPU: KFAC(model).step() (Listing 1) on a real torch model with hooks, against the oracle.

A small CNN (3x3 conv with bias, stride-2 3x3 conv without bias, linear with bias) in training mode
on random data with a mean-reduced cross-entropy loss.  The test records every layer's input,
output gradient (x batch size, the KFAC default) and weight/bias gradient itself, lays them out as
the oracle expects (NHWC, (C_out, k_h, k_w, C_in | bias)), runs oracle.full_step on them and compares
with the .grad tensors KFAC.step() wrote back: factors <= 1e-4, P <= 1e-3 (north_star bars)."""
import numpy as np
import pytest
import torch
import torch.nn as nn

from conftest import relF
from workloads import shapes

pytestmark = pytest.mark.gpu


class Net(nn.Module):
    def __init__(self):
        super().__init__()
        self.c1 = nn.Conv2d(3, 8, 3, 1, 1)
        self.c2 = nn.Conv2d(8, 16, 3, 2, 1, bias=False)
        self.fc = nn.Linear(16 * 4 * 4, 10)

    def forward(self, x):
        x = torch.relu(self.c1(x))
        x = torch.relu(self.c2(x))
        return self.fc(x.flatten(1))


def _layer(name, m, a, g):
    if isinstance(m, nn.Linear):
        return shapes.linear(name, a.shape[0], m.in_features, m.out_features, bias_col=int(m.bias is not None))
    L = shapes.conv(name, a.shape[0], m.in_channels, m.out_channels, m.kernel_size[0], m.stride[0], a.shape[2],
                    bias_col=int(m.bias is not None))
    assert L.h_out == g.shape[2]
    return L


def test_kfac_model_step_matches_oracle(orc):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2007_00784_b200.build import build
    build()
    from paper_2007_00784_b200.kfac import KFAC
    torch.manual_seed(0)
    net = Net().cuda()
    x = torch.randn(6, 3, 8, 8, device="cuda")
    y = torch.randint(0, 10, (6,), device="cuda")
    hp = dict(damping=3e-3, xi=0.95, kappa=1e-3, lr=0.1)
    kfac = KFAC(net, lr=hp["lr"], damping=hp["damping"], xi=hp["xi"], kappa=hp["kappa"])
    rec = {}
    mods = [net.c1, net.c2, net.fc]
    hooks = [m.register_forward_pre_hook(lambda m, i: rec.__setitem__((id(m), "a"), i[0].detach().clone()))
             for m in mods]
    hooks += [m.register_full_backward_hook(lambda m, gi, go: rec.__setitem__((id(m), "g"), go[0].detach().clone()))
              for m in mods]
    loss = nn.functional.cross_entropy(net(x), y)
    loss.backward()
    for h in hooks:
        h.remove()
    layers, acts, gouts, grads = [], [], [], []
    for name, m in zip(("c1", "c2", "fc"), mods):
        a, g = rec[(id(m), "a")], rec[(id(m), "g")]
        layers.append(_layer(name, m, a, g))
        n = a.shape[0]
        if isinstance(m, nn.Linear):
            acts.append(a.cpu().numpy().astype(np.float32))
            gouts.append((g * n).cpu().numpy().astype(np.float32))
            w = m.weight.grad
        else:
            acts.append(a.permute(0, 2, 3, 1).contiguous().cpu().numpy().astype(np.float32))
            gouts.append((g * n).permute(0, 2, 3, 1).reshape(-1, g.shape[1]).cpu().numpy().astype(np.float32))
            w = m.weight.grad.permute(0, 2, 3, 1)
        W = w.reshape(w.shape[0], -1)
        if m.bias is not None:
            W = torch.cat([W, m.bias.grad[:, None]], 1)
        grads.append(W.cpu().numpy().astype(np.float32))
    ref = orc.full_step(layers, acts, gouts, grads, hp["damping"], hp["lr"], hp["kappa"])
    kfac.step()
    torch.cuda.synchronize()
    for i, m in enumerate(mods):
        assert relF(kfac.pc.A[i].double().cpu().numpy(), ref["A"][i]) <= 1e-4
        assert relF(kfac.pc.G[i].double().cpu().numpy(), ref["G"][i]) <= 1e-4
        w = m.weight.grad.permute(0, 2, 3, 1) if isinstance(m, nn.Conv2d) else m.weight.grad
        got = w.reshape(w.shape[0], -1)
        if m.bias is not None:
            got = torch.cat([got, m.bias.grad[:, None]], 1)
        assert relF(got.double().cpu().numpy(), ref["P"][i]) <= 1e-3, i
    assert abs(kfac.pc.nu.item() - ref["nu"]) <= 1e-4 * ref["nu"]


def test_kfac_model_schedules():
    """Eigen refresh every kfac_update_freq steps, damping decayed at the scheduled steps."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2007_00784_b200.kfac import KFAC
    torch.manual_seed(1)
    net = Net().cuda()
    kfac = KFAC(net, lr=0.1, damping=1e-2, kfac_update_freq=3, damping_decay_steps=[2, 4], damping_decay_rate=0.5)
    calls = []
    orig = kfac.__class__._build

    for it in range(6):
        net.zero_grad()
        nn.functional.cross_entropy(net(torch.randn(4, 3, 8, 8, device="cuda")),
                                    torch.randint(0, 10, (4,), device="cuda")).backward()
        before = kfac.pc.info.clone() if kfac.pc is not None else None
        kfac.step()
        calls.append(kfac.damping)
        assert all(torch.isfinite(p.grad).all() for p in net.parameters())
    assert calls == [1e-2, 1e-2, 5e-3, 5e-3, 2.5e-3, 2.5e-3]
    assert kfac.steps == 6
    del orig, before

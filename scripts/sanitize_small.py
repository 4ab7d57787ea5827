"""Small shapes through every engine of libkfac, for compute-sanitizer (memcheck / racecheck /
synccheck):  compute-sanitizer --tool memcheck python scripts/sanitize_small.py
Covers: the factor SYRK (tcgen05 planes engine incl. a channel-padded conv, SIMT tile), the fold and
packed outputs, the eigensolver (Jacobi, one-stage tridiagonal reduction, the two-stage reduction
forced at d = 1041, divide and conquer, back-transformation), the explicit inverse, the
preconditioning GEMM chain and the KL-clip."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_00784_b200 import _lib  # noqa: E402
from workloads import shapes  # noqa: E402
from workloads.gen import layer_inputs  # noqa: E402

dev = torch.device("cuda")
layers = [shapes.conv("c7s2c3", 2, 3, 64, 7, 2, 24), shapes.conv("c3", 2, 16, 72, 3, 1, 10),
          shapes.linear("fc", 40, 130, 12)]
acts, gouts, grads = layer_inputs(layers, seed=0)


def ld(n):
    return (n + 3) // 4 * 4


A = [torch.zeros(l.d_a, ld(l.d_a), device=dev) for l in layers]
G = [torch.zeros(l.d_g, ld(l.d_g), device=dev) for l in layers]
_lib.kfac_update_factors(layers, [torch.from_numpy(a).to(dev) for a in acts],
                         [torch.from_numpy(g).to(dev) for g in gouts], A, G, 0.95, True, 1.0)
torch.cuda.synchronize()
print("factors ok", flush=True)

rng = np.random.default_rng(1)
dims = [17, 65, 300, 1041]
Fs = []
for n in dims:
    X = rng.standard_normal((max(8, n // 2), n)).astype(np.float32)
    F = torch.zeros(n, ld(n), device=dev)
    F[:, :n] = torch.from_numpy(X.T @ X / X.shape[0]).to(dev)
    Fs.append(F)
# --one-stage: every tridiagonal factor on the one-stage reduction (synccheck: the two-stage bulge
# chase signals with mbarrier arrivals that no thread of the producer waits on, which synccheck flags)
one_stage = "--one-stage" in sys.argv
for flags in ((16,) if one_stage else (0, 4 | 8)):        # default routing, then the two-stage path
    Q = [torch.zeros_like(F) for F in Fs]
    v = [torch.zeros(n, device=dev) for n in dims]
    info = torch.zeros(len(dims), dtype=torch.int32, device=dev)
    _lib.kfac_compute_eigen(Fs, Q, v, info, flags)
    torch.cuda.synchronize()
    assert int(info.abs().max()) == 0
    print("eigen ok flags", flags, flush=True)

# every factor <= ~880: the cluster-resident small-factor reduction (d = 300 on a 2-CTA cluster)
Q = [torch.zeros_like(F) for F in Fs[1:3]]
v = [torch.zeros(n, device=dev) for n in dims[1:3]]
info = torch.zeros(2, dtype=torch.int32, device=dev)
_lib.kfac_compute_eigen(Fs[1:3], Q, v, info, 0)
torch.cuda.synchronize()
assert int(info.abs().max()) == 0
print("eigen ok (small-factor cluster path)", flush=True)

Finv = [torch.zeros_like(F) for F in Fs[:3]]
info = torch.zeros(3, dtype=torch.int32, device=dev)
_lib.kfac_compute_inverse(Fs[:3], 1e-3, Finv, info)
torch.cuda.synchronize()
print("inverse ok", flush=True)

QA = [torch.zeros_like(a) for a in A]
QG = [torch.zeros_like(g) for g in G]
vA = [torch.zeros(l.d_a, device=dev) for l in layers]
vG = [torch.zeros(l.d_g, device=dev) for l in layers]
_lib.kfac_compute_eigen(A + G, QA + QG, vA + vG, None, 16 if one_stage else 0)
W, out = [], []
for g in grads:
    g = torch.as_tensor(np.asarray(g), dtype=torch.float32)
    buf = torch.zeros(g.shape[0], ld(g.shape[1]), device=dev)
    buf[:, : g.shape[1]] = g.to(dev)
    W.append(buf[:, : g.shape[1]])                         # d_G x d_A view, leading dimension ld(d_A)
    out.append(torch.zeros_like(buf)[:, : g.shape[1]])
_lib.kfac_precondition(W, QG, vG, QA, vA, 1e-3, 0, out)
_lib.kfac_kl_clip(out, W, 0.1, 1e-3)
torch.cuda.synchronize()
print("precondition + kl ok", flush=True)

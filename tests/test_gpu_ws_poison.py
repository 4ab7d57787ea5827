"""The eigensolver's result must not depend on the workspace contents (kfac.h: the workspace is
caller-owned scratch, no state is carried between calls).  Every call here runs on a workspace
filled with NaN bytes, so a read of a workspace word the call did not write first poisons the
output: Q and the eigenvalues must come out finite and meet the LAPACK bars of test_gpu_sbr."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TRIDIAG, TWO_STAGE, ONE_STAGE = 4, 8, 16


@pytest.fixture(scope="module")
def lib():
    from paper_2007_00784_b200.build import build
    build()
    from paper_2007_00784_b200 import _lib
    return _lib


def _dev(x):
    n, m = x.shape
    t = torch.zeros(n, (m + 3) // 4 * 4, dtype=torch.float32, device="cuda")
    t[:, :m] = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    return t


def _wishart(rng, n, rows):
    X = rng.standard_normal((rows, n))
    X[:, -1] = 1.0
    return (X.T @ X / rows).astype(np.float32)


def _run(lib, dims, rows, flags, seed):
    rng = np.random.default_rng(seed)
    Fs = [_wishart(rng, n, r) for n, r in zip(dims, rows)]
    fd = [_dev(F) for F in Fs]
    Q = [torch.zeros_like(f) for f in fd]
    v = [torch.zeros(n, device="cuda") for n in dims]
    info = torch.full((len(dims),), -7, dtype=torch.int32, device="cuda")
    ws = lib.Workspace()
    need = lib.lib.kfac_compute_eigen_workspace_size(lib._i32(dims), len(dims))
    ws.get(need).fill_(0xFF)                                      # every byte NaN-patterned
    lib.kfac_compute_eigen(fd, Q, v, info=info, flags=flags, ws=ws)
    torch.cuda.synchronize()
    assert (info.cpu().numpy() == 0).all()
    for n, F, q, w in zip(dims, Fs, Q, v):
        Qn = q[:, :n].double().cpu().numpy()
        vn = w.double().cpu().numpy()
        assert np.isfinite(Qn).all() and np.isfinite(vn).all(), f"non-finite output for d = {n}"
        F64 = F.astype(np.float64)
        w_ref = np.clip(np.linalg.eigvalsh(F64), 0, None)
        assert np.abs(vn - w_ref).max() <= 2e-6 * w_ref.max()
        assert np.abs(Qn.T @ Qn - np.eye(n)).max() <= 2e-5
        R = (Qn * vn) @ Qn.T
        assert np.linalg.norm(R - F64) / np.linalg.norm(F64) <= 1e-5


@pytest.mark.parametrize("n,rows,flags", [(1041, 300, TRIDIAG | TWO_STAGE), (1024, 3000, TRIDIAG | TWO_STAGE),
                                          (1041, 300, TRIDIAG | ONE_STAGE), (785, 200, TRIDIAG),
                                          (65, 40, 0), (300, 100, TRIDIAG), (2305, 800, TRIDIAG | TWO_STAGE)])
def test_eigen_on_poisoned_workspace(lib, n, rows, flags):
    _run(lib, [n], [rows], flags, seed=n + rows)


def test_mixed_batch_on_poisoned_workspace(lib):
    dims = [65, 1041, 513, 2305, 1153, 300, 1600, 17]
    rows = [40, 300, 200, 900, 500, 100, 700, 10]
    _run(lib, dims, rows, TRIDIAG | TWO_STAGE, seed=11)


def test_inverse_on_poisoned_workspace(lib):
    """Explicit damped inverse (Eq. 8 variant) on a NaN-filled workspace: finite and equal to the
    fp64 inverse of F + gamma I (numpy, not the CUDA path) to the fp32 output rounding."""
    dims = [5, 65, 300, 1041]
    rng = np.random.default_rng(4)
    Fs = [_wishart(rng, n, max(8, n // 2)).astype(np.float64) for n in dims]
    damping = 1e-3
    Finv = [torch.zeros(n, (n + 3) // 4 * 4, dtype=torch.float32, device="cuda") for n in dims]
    info = torch.full((len(dims),), -1, dtype=torch.int32, device="cuda")
    ws = lib.Workspace()
    need = lib.lib.kfac_compute_inverse_workspace_size(lib._i32(dims), len(dims))
    ws.get(need).fill_(0xFF)
    lib.kfac_compute_inverse([_dev(F) for F in Fs], damping, Finv, info=info, ws=ws)
    torch.cuda.synchronize()
    assert (info.cpu().numpy() == 0).all()
    for n, F, X in zip(dims, Fs, Finv):
        Xn = X[:, :n].double().cpu().numpy()
        assert np.isfinite(Xn).all()
        ref = np.linalg.inv(F.astype(np.float32).astype(np.float64) + damping * np.eye(n))
        assert np.linalg.norm(Xn - ref) / np.linalg.norm(ref) <= 1e-5


R50_SUB = ("conv1", "layer1.0.conv2", "layer2.0.conv2", "layer3.0.conv2", "layer4.0.conv2",
           "layer4.0.downsample", "fc")


@pytest.mark.parametrize("cfg,variant", [("mlp", "eigen"), ("r32", "eigen"), ("r32", "factored"),
                                         ("r32", "inverse"), ("r50sub", "eigen")])
def test_full_step_independent_of_workspace_contents(lib, monkeypatch, cfg, variant):
    """One full K-FAC update (factors, decomposition, preconditioning, KL-clip) through the
    preconditioner, with every workspace handed to the library refilled before each call -- once
    with zero bytes, once with 0xFF (NaN) bytes: the outputs must be bitwise identical, so no stage
    reads scratch it did not write first in the same call."""
    from paper_2007_00784_b200.preconditioner import KFACPreconditioner
    from workloads import shapes
    from workloads.gen import layer_inputs

    if cfg == "r50sub":        # full-size ResNet-50 layers: tensor-core SYRK, one-stage panels, Ozaki
        layers = [l for l in shapes.layers_for("r50") if l.name in R50_SUB]
        hp = shapes.HPARAMS["r50"]
    else:
        layers = shapes.mlp() if cfg == "mlp" else shapes.resnet32(batch=4)
        hp = shapes.HPARAMS[cfg]
    acts, gouts, grads = layer_inputs(layers, seed=3)
    orig_get = lib.Workspace.get
    out = {}
    for fill in (0x00, 0xFF):
        def get(self, nbytes, _fill=fill):
            buf = orig_get(self, nbytes)
            buf.fill_(_fill)
            return buf
        monkeypatch.setattr(lib.Workspace, "get", get)
        pc = KFACPreconditioner(layers, damping=hp["damping"], xi=hp["xi"], kappa=hp["kappa"],
                                lr=hp["lr"], variant=variant)
        g = KFACPreconditioner.grad_buffer(layers, "cuda")
        for t, w in zip(g, grads):
            t.copy_(torch.from_numpy(w))
        P = pc.step([torch.from_numpy(a).cuda() for a in acts], [torch.from_numpy(x).cuda() for x in gouts], g,
                    first=True)
        torch.cuda.synchronize()
        out[fill] = ([p.cpu().numpy().copy() for p in P], float(pc.nu.item()))
    monkeypatch.setattr(lib.Workspace, "get", orig_get)
    for a, b in zip(out[0x00][0], out[0xFF][0]):
        assert np.isfinite(b).all()
        assert np.array_equal(a, b)
    assert out[0x00][1] == out[0xFF][1]

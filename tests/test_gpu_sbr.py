"""GPU: the two-stage tridiagonalisation (eigen_sbr.cu) of the large factors, d >= 1024.

* stage 1 + stage 2 (kfac_debug_tridiag): the tridiagonal T of Q^T F Q keeps the spectrum of F to
  fp64 working precision (the whole reduction is fp64; bar 1e-11 ||F||, against 2e-6 for the fp32
  one-stage path) and the orthogonal invariants trace and Frobenius norm;
* the full solver (kfac_compute_eigen) through stage 1, stage 2, divide and conquer, the stage-2
  reflector blocks (Q2) and the stage-1 back-transformation (Q1): eigenvalues vs LAPACK, fp32
  orthogonality and reconstruction bars as for the one-stage path (tests/test_gpu_eigen_trd.py);
* ragged sizes around the band (n = 16k + 1, 16k + 2, ...), rank-deficient factors (rows < n, as
  every ResNet-50 layer4 3x3 A factor), the largest supported size, and one call mixing one-stage
  and two-stage factors.
The input is a seeded Wishart matrix X^T X / rows with a bias column (SURVEY §8(d) recipe)."""
import ctypes as C

import numpy as np
import pytest
import scipy.linalg as sla
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2007_00784_b200.build import build
    build()
    from paper_2007_00784_b200 import _lib
    L = _lib.lib
    L.kfac_debug_tridiag_ex.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_uint,
                                        C.c_void_p]
    L.kfac_debug_tridiag_ex.restype = C.c_int
    L.kfac_debug_tridiag.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    L.kfac_debug_tridiag.restype = C.c_int
    return _lib


TRIDIAG, TWO_STAGE, ONE_STAGE = 4, 8, 16


def _ld(n):
    return (n + 3) // 4 * 4


def _dev(x):
    n, m = x.shape
    t = torch.zeros(n, _ld(m), dtype=torch.float32, device="cuda")
    t[:, :m] = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    return t


def _wishart(rng, n, rows):
    X = rng.standard_normal((rows, n))
    X[:, -1] = 1.0
    return (X.T @ X / rows).astype(np.float32)


@pytest.mark.parametrize("n,rows", [(1024, 3000), (1025, 500), (1042, 2000), (2305, 6272), (4609, 1568)])
def test_two_stage_tridiagonal_spectrum(lib, n, rows):
    rng = np.random.default_rng(n + rows)
    F = _wishart(rng, n, rows).astype(np.float64)
    f = _dev(F)
    d = torch.zeros(n, dtype=torch.float64, device="cuda")
    e = torch.zeros(n, dtype=torch.float64, device="cuda")
    st = lib.lib.kfac_debug_tridiag_ex(f.data_ptr(), n, f.stride(0), d.data_ptr(), e.data_ptr(), TWO_STAGE, None)
    assert st == 0, lib.lib.kfac_last_error()
    d, e = d.cpu().numpy(), e.cpu().numpy()[: n - 1]
    assert np.all(np.isfinite(d)) and np.all(np.isfinite(e))
    w_ref = np.linalg.eigvalsh(F)
    w = sla.eigvalsh_tridiagonal(d, e)
    scale = np.abs(w_ref).max()
    assert np.abs(np.sort(w) - w_ref).max() <= 1e-11 * scale, np.abs(np.sort(w) - w_ref).max() / scale
    assert abs(d.sum() - np.trace(F)) <= 1e-11 * np.abs(F).sum()
    fro = np.sqrt((d ** 2).sum() + 2 * (e ** 2).sum())
    assert abs(fro - np.linalg.norm(F)) <= 1e-11 * np.linalg.norm(F)


def _check_eigen(F, Qn, vn):
    n = F.shape[0]
    F64 = F.astype(np.float64)
    w_ref = np.clip(np.linalg.eigvalsh(F64), 0, None)
    scale = w_ref.max()
    assert np.all(np.diff(vn) >= 0) and vn.min() >= 0
    assert np.abs(vn - w_ref).max() <= 2e-6 * scale
    assert np.abs(Qn.T @ Qn - np.eye(n)).max() <= 2e-5
    rec = (Qn * vn) @ Qn.T
    assert np.linalg.norm(rec - F64) / np.linalg.norm(F64) <= 1e-5


@pytest.mark.parametrize("n,rows", [(1024, 3000), (1041, 300), (2049, 1568), (2305, 6272), (4609, 1568),
                                    (5632, 6000)])
def test_two_stage_compute_eigen(lib, n, rows):
    rng = np.random.default_rng(3 * n + rows)
    F = _wishart(rng, n, rows)
    f = _dev(F)
    Q = torch.zeros_like(f)
    v = torch.zeros(n, device="cuda")
    info = torch.full((1,), -7, dtype=torch.int32, device="cuda")
    lib.kfac_compute_eigen([f], [Q], [v], info=info, flags=TRIDIAG | TWO_STAGE)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    _check_eigen(F, Q[:, :n].double().cpu().numpy(), v.double().cpu().numpy())


def test_two_stage_mixed_batch(lib):
    """One call with one-stage (d < 1024) and two-stage factors of different panel counts: the
    staggered stage-1 schedule, the per-cluster-size stage-2 launches and the per-factor reflector
    offset of the back-transformation."""
    dims = [65, 1025, 513, 2305, 1153, 300, 1600]
    rng = np.random.default_rng(5)
    Fs = [_wishart(rng, n, max(16, n // 2)) for n in dims]
    fd = [_dev(F) for F in Fs]
    Q = [torch.zeros_like(f) for f in fd]
    v = [torch.zeros(n, device="cuda") for n in dims]
    info = torch.full((len(dims),), -7, dtype=torch.int32, device="cuda")
    lib.kfac_compute_eigen(fd, Q, v, info=info, flags=TRIDIAG | TWO_STAGE)
    torch.cuda.synchronize()
    assert (info.cpu().numpy() == 0).all()
    for n, F, q, w in zip(dims, Fs, Q, v):
        _check_eigen(F, q[:, :n].double().cpu().numpy(), w.double().cpu().numpy())


def test_two_stage_bitwise_repeatable(lib):
    """Fixed-order reductions everywhere: two calls give identical eigenpairs."""
    n = 1153
    F = _wishart(np.random.default_rng(9), n, 400)
    f = _dev(F)
    out = []
    for _ in range(2):
        Q = torch.zeros_like(f)
        v = torch.zeros(n, device="cuda")
        lib.kfac_compute_eigen([f], [Q], [v], flags=TRIDIAG | TWO_STAGE)
        torch.cuda.synchronize()
        out.append((Q.cpu().numpy(), v.cpu().numpy()))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


def test_routing_default_and_forced(lib):
    """The default routing sends a lone mid-size factor (all of the call's d^3) to the two-stage
    reduction and KFAC_EIG_ONE_STAGE keeps it on the one-stage one: the default tridiagonal equals
    the forced two-stage one bit for bit and differs from the one-stage one (same spectrum)."""
    n = 1153
    F = _wishart(np.random.default_rng(21), n, 500).astype(np.float64)
    f = _dev(F)
    out = {}
    for name, fl in (("default", 0), ("two", TWO_STAGE), ("one", ONE_STAGE)):
        d = torch.zeros(n, dtype=torch.float64, device="cuda")
        e = torch.zeros(n, dtype=torch.float64, device="cuda")
        assert lib.lib.kfac_debug_tridiag_ex(f.data_ptr(), n, f.stride(0), d.data_ptr(), e.data_ptr(), fl, None) == 0
        out[name] = (d.cpu().numpy(), e.cpu().numpy()[: n - 1])
    assert np.array_equal(out["default"][0], out["two"][0]) and np.array_equal(out["default"][1], out["two"][1])
    assert not np.array_equal(out["one"][0], out["two"][0])
    w1 = sla.eigvalsh_tridiagonal(*out["one"])
    w2 = sla.eigvalsh_tridiagonal(*out["two"])
    assert np.abs(w1 - w2).max() <= 2e-6 * np.abs(w2).max()

"""GPU: the tridiagonalisation + divide-and-conquer eigensolver (eigen_trd.cu), stage by stage.

* C -= A B epilogue of both GEMM engines (the rank-2k trailing update and back-transformation);
* Householder reduction: eigenvalues of the GPU tridiagonal (d, e) (LAPACK dstebz via scipy, fp64)
  equal eigvalsh(F) to fp32-working-precision (|err| <= 2e-6 ||F||_2);
* divide and conquer on a given tridiagonal, on the classical hard cases (Wilkinson W+ pairs,
  glued copies, zero couplings, graded, constant diagonals, Clement) -- eigenvalues against LAPACK,
  residual ||T Z - Z L|| and orthogonality (fp32 eigenvector storage bounds both at ~1e-6);
* kfac_compute_eigen with KFAC_EIG_TRIDIAG on factor-like (rank-deficient Wishart) matrices.
Bars are derived from fp32 storage (2^-24 ~ 6e-8) times modest growth in n, stated per test."""
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
    L.kfac_debug_gemm.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int,
                                  C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    L.kfac_debug_gemm.restype = C.c_int
    L.kfac_debug_tridiag.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    L.kfac_debug_tridiag.restype = C.c_int
    L.kfac_debug_stedc.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    L.kfac_debug_stedc.restype = C.c_int
    L.kfac_debug_gemm64.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                    C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
    L.kfac_debug_gemm64.restype = C.c_int
    return _lib


def _ld(n):
    return (n + 3) // 4 * 4


def _dev(x):
    n, m = x.shape
    t = torch.zeros(n, _ld(m), dtype=torch.float32, device="cuda")
    t[:, :m] = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    return t


@pytest.mark.parametrize("engine", [0, 2])
@pytest.mark.parametrize("M,N,K", [(200, 130, 64), (77, 301, 32)])
def test_gemm_sub_epilogue(lib, engine, M, N, K):
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K))
    B = rng.standard_normal((K, N))
    C0 = rng.standard_normal((M, N))
    a, b, c = _dev(A), _dev(B), _dev(C0)
    if engine == 2 and (M < 64 or N < 64):
        pytest.skip("tensor-core engine needs M, N >= 64")
    st = lib.lib.kfac_debug_gemm(engine | 4, a.data_ptr(), a.stride(0), 0, b.data_ptr(), b.stride(0), 0,
                                 c.data_ptr(), c.stride(0), M, N, K, None, None)
    assert st == 0
    torch.cuda.synchronize()
    ref = C0.astype(np.float32).astype(np.float64) - A.astype(np.float32).astype(np.float64) @ B.astype(np.float32).astype(np.float64)
    got = c[:, :N].double().cpu().numpy()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 2e-6


@pytest.mark.parametrize("dts", [(0, 0, 0), (0, 1, 1), (1, 1, 1), (1, 0, 0)])
@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("epi", [0, 3])
@pytest.mark.parametrize("padded", [False, True])
def test_gemm64(lib, dts, ta, tb, epi, padded):
    """fp64-accumulating SIMT GEMM of the eigensolver: fp64 products of the (fp32 or fp64)
    operands, one rounding to the output type -> relF <= 1e-14 (fp64 out) / 2^-24 (fp32 out).
    padded: leading dimensions rounded up to 16 bytes, which selects the cp.async pipelined
    kernel (K = 77 leaves a ragged last slab and a partial 16-byte chunk)."""
    M, N, K = 150, 131, 77
    rng = np.random.default_rng(ta * 2 + tb + 10 * epi)
    dt = lambda c: torch.float64 if c else torch.float32

    def dev(x, code):
        t = torch.from_numpy(x).to(dt(code))
        if not padded:
            return t.cuda()
        ld = (x.shape[1] + 3) // 4 * 4
        buf = torch.zeros((x.shape[0], ld), dtype=dt(code), device="cuda")
        buf[:, :x.shape[1]] = t.cuda()
        return buf[:, :x.shape[1]]

    A = rng.standard_normal((K, M) if ta else (M, K))
    B = rng.standard_normal((N, K) if tb else (K, N))
    C0 = rng.standard_normal((M, N))
    a = dev(A, dts[0])
    b = dev(B, dts[1])
    c = dev(C0, dts[2])
    st = lib.lib.kfac_debug_gemm64(a.data_ptr(), dts[0], a.stride(0), ta, b.data_ptr(), dts[1], b.stride(0), tb,
                                   c.data_ptr(), dts[2], c.stride(0), M, N, K, epi, None)
    assert st == 0
    torch.cuda.synchronize()
    opA = a.double().cpu().numpy()
    opB = b.double().cpu().numpy()
    opA = opA.T if ta else opA
    opB = opB.T if tb else opB
    c0 = torch.from_numpy(C0).to(dt(dts[2])).double().numpy()
    ref = c0 - opA @ opB if epi == 3 else opA @ opB
    got = c.double().cpu().numpy()
    tol = 1e-14 if dts[2] == 1 else 1.2e-7
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= tol


def _wishart(rng, n, rows, bias=True):
    X = rng.standard_normal((rows, n))
    if bias:
        X[:, -1] = 1.0
    return X.T @ X / rows


def _tridiag(lib, F):
    n = F.shape[0]
    f = _dev(F)
    d = torch.zeros(n, dtype=torch.float64, device="cuda")
    e = torch.zeros(n, dtype=torch.float64, device="cuda")
    st = lib.lib.kfac_debug_tridiag(f.data_ptr(), n, f.stride(0), d.data_ptr(), e.data_ptr(), None)
    assert st == 0, lib.lib.kfac_last_error()
    return d.cpu().numpy(), e.cpu().numpy()[: n - 1]


@pytest.mark.parametrize("n,rows", [(40, 100), (64, 30), (100, 1000), (257, 64), (700, 300), (1153, 2000)])
def test_tridiagonal_reduction_preserves_spectrum(lib, n, rows):
    rng = np.random.default_rng(n)
    F = _wishart(rng, n, rows).astype(np.float32).astype(np.float64)
    d, e = _tridiag(lib, F)
    assert np.all(np.isfinite(d)) and np.all(np.isfinite(e))
    w_ref = np.linalg.eigvalsh(F)
    w = sla.eigvalsh_tridiagonal(d, e) if n > 1 else d
    scale = np.abs(w_ref).max()
    assert np.abs(np.sort(w) - w_ref).max() <= 2e-6 * scale
    # trace and Frobenius norm are invariants of the orthogonal similarity
    assert abs(d.sum() - np.trace(F)) <= 1e-6 * np.abs(F).sum()
    assert abs(np.sqrt((d ** 2).sum() + 2 * (e ** 2).sum()) - np.linalg.norm(F)) <= 1e-6 * np.linalg.norm(F)


def _tcases():
    rng = np.random.default_rng(7)
    cases = {}
    for n in (1, 2, 5, 32, 33, 64, 100, 513, 1000):
        cases[f"normal{n}"] = (rng.standard_normal(n), rng.standard_normal(max(n - 1, 0)))
    m = 50                                                # Wilkinson W+_{2m+1}: close pairs
    cases["wilkinson101"] = (np.abs(np.arange(-m, m + 1)).astype(float), np.ones(2 * m))
    d0, e0 = rng.standard_normal(40), rng.standard_normal(39)
    d = np.concatenate([d0] * 5)                          # glued identical blocks: clusters
    e = np.concatenate([np.concatenate([e0, [1e-10]])] * 5)[:-1]
    cases["glued200"] = (d, e)
    e = rng.standard_normal(299)
    e[::37] = 0.0                                         # exact splits
    cases["zeros300"] = (rng.standard_normal(300), e)
    cases["graded200"] = (10.0 ** (-np.arange(200) / 20), 10.0 ** (-np.arange(199) / 20 - 0.5))
    cases["constant150"] = (np.full(150, 2.0), np.full(149, 1e-3))
    n = 130                                               # Clement (Kac) matrix, symmetric form
    cases["clement130"] = (np.zeros(n), np.sqrt(np.arange(1, n) * np.arange(n - 1, 0, -1)))
    cases["diag96"] = (rng.standard_normal(96), np.zeros(95))
    # D&C column types: identical halves glued by a tiny coupling make almost every non-deflated
    # column of the top merges a rotation mix of an upper and a lower column (type 2), while an
    # unbalanced glue of different blocks keeps most columns pure (types 1 and 3)
    d1, e1 = rng.standard_normal(250), rng.standard_normal(249)
    cases["glued_halves1000"] = (np.concatenate([d1] * 4), np.concatenate([e1, [1e-12], e1, [1e-12], e1, [1e-12], e1]))
    d2, e2 = rng.standard_normal(700), rng.standard_normal(699)
    d3, e3 = 3.0 + rng.standard_normal(301), rng.standard_normal(300)
    cases["unbalanced1001"] = (np.concatenate([d2, d3]), np.concatenate([e2, [0.5], e3]))
    return cases


_TC = _tcases()


@pytest.mark.parametrize("name", list(_TC))
def test_divide_and_conquer(lib, name):
    d, e = _TC[name]
    n = len(d)
    dd = torch.from_numpy(d.copy()).cuda()
    ee = torch.from_numpy(np.concatenate([e, [0.0]])).cuda()
    Z = torch.full((n, _ld(n)), float("nan"), dtype=torch.float32, device="cuda")
    w = torch.zeros(n, dtype=torch.float64, device="cuda")
    st = lib.lib.kfac_debug_stedc(dd.data_ptr(), ee.data_ptr(), n, Z.data_ptr(), Z.stride(0), w.data_ptr(), None)
    assert st == 0, lib.lib.kfac_last_error()
    torch.cuda.synchronize()
    w = w.cpu().numpy()
    Zn = Z[:, :n].double().cpu().numpy()
    T = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    w_ref = np.linalg.eigvalsh(T)
    tn = max(np.abs(w_ref).max(), 1e-300)
    assert np.all(np.diff(w) >= 0)
    assert np.abs(w - w_ref).max() <= 1e-6 * tn, np.abs(w - w_ref).max() / tn
    assert np.abs(Zn.T @ Zn - np.eye(n)).max() <= 2e-6 * max(1.0, np.sqrt(n) / 4)
    R = T @ Zn - Zn * w
    assert np.linalg.norm(R) <= 2e-6 * np.sqrt(n) * tn


@pytest.mark.parametrize("n,rows", [(64, 200), (65, 20), (129, 1000), (300, 64), (577, 3000), (1153, 500)])
def test_compute_eigen_tridiag(lib, n, rows):
    rng = np.random.default_rng(n + rows)
    F = _wishart(rng, n, rows).astype(np.float32)
    f = _dev(F)
    Q = torch.zeros_like(f)
    v = torch.zeros(n, device="cuda")
    info = torch.full((1,), -7, dtype=torch.int32, device="cuda")
    lib.kfac_compute_eigen([f], [Q], [v], info=info, flags=4)
    torch.cuda.synchronize()
    assert int(info.item()) == 0
    Qn = Q[:, :n].double().cpu().numpy()
    vn = v.double().cpu().numpy()
    F64 = F.astype(np.float64)
    w_ref = np.clip(np.linalg.eigvalsh(F64), 0, None)
    scale = w_ref.max()
    assert np.all(np.diff(vn) >= 0) and vn.min() >= 0
    assert np.abs(vn - w_ref).max() <= 2e-6 * scale
    assert np.abs(Qn.T @ Qn - np.eye(n)).max() <= 2e-5
    rec = (Qn * vn) @ Qn.T
    assert np.linalg.norm(rec - F64) / np.linalg.norm(F64) <= 1e-5


def test_compute_eigen_tridiag_batched(lib):
    """Several factors with different D&C depths and panel counts in one call (per-factor
    ping-pong parity of the merge levels, CTA groups of the reduction, blocks of the
    back-transformation)."""
    dims = [33, 64, 65, 300, 1100, 97]
    rng = np.random.default_rng(11)
    Fs = [_wishart(rng, n, max(8, n // 3)).astype(np.float32) for n in dims]
    fd = [_dev(F) for F in Fs]
    Q = [torch.zeros_like(f) for f in fd]
    v = [torch.zeros(n, device="cuda") for n in dims]
    info = torch.full((len(dims),), -7, dtype=torch.int32, device="cuda")
    lib.kfac_compute_eigen(fd, Q, v, info=info, flags=4)
    torch.cuda.synchronize()
    assert (info.cpu().numpy() == 0).all()
    for n, F, q, w in zip(dims, Fs, Q, v):
        Qn = q[:, :n].double().cpu().numpy()
        wn = w.double().cpu().numpy()
        F64 = F.astype(np.float64)
        assert np.abs(Qn.T @ Qn - np.eye(n)).max() <= 2e-5, n
        assert np.linalg.norm((Qn * wn) @ Qn.T - F64) / np.linalg.norm(F64) <= 1e-5, n


@pytest.mark.parametrize("n", [65, 289, 785])
def test_small_cluster_path_matches_panel_path(lib, n):
    """The cluster-resident small-factor reduction (a call whose factors all fit one cluster,
    DESIGN.md 8b') and the grid-synchronised panel path (the same factor in a call with a large
    one) are two implementations of the same Householder reduction: both decompositions meet the
    fp32-storage bars against LAPACK, and their eigenvalues agree to the same bar (eigenvectors
    through the reconstruction: sign and order within clusters are free, R11)."""
    rng = np.random.default_rng(700 + n)
    F = _wishart(rng, n, max(16, n // 2)).astype(np.float32)
    big = _wishart(rng, 1000, 400).astype(np.float32)          # 1000 > ~870: forces the panel path
    res = []
    for fs in ([F], [F, big]):
        fd = [_dev(x) for x in fs]
        Q = [torch.zeros_like(f) for f in fd]
        v = [torch.zeros(x.shape[0], device="cuda") for x in fs]
        info = torch.full((len(fs),), -7, dtype=torch.int32, device="cuda")
        lib.kfac_compute_eigen(fd, Q, v, info=info, flags=4)
        torch.cuda.synchronize()
        assert (info.cpu().numpy() == 0).all()
        res.append((Q[0][:, :n].double().cpu().numpy(), v[0].double().cpu().numpy()))
    F64 = F.astype(np.float64)
    w_ref = np.clip(np.linalg.eigvalsh(F64), 0, None)
    scale = w_ref.max()
    for Qn, vn in res:
        assert np.abs(vn - w_ref).max() <= 2e-6 * scale
        assert np.abs(Qn.T @ Qn - np.eye(n)).max() <= 2e-5
        rec = (Qn * vn) @ Qn.T
        assert np.linalg.norm(rec - F64) / np.linalg.norm(F64) <= 1e-5
    assert np.abs(res[0][1] - res[1][1]).max() <= 2e-6 * scale

"""GPU: the fp64-accurate int8 tensor-core GEMM (Ozaki scheme, gemm_ozaki.cu) of the eigensolver.

Bound (derived in gemm_ozaki.cu's header): every operand row is scaled by 2^-e (e = exponent of its
largest |entry| + 1) and cut after s digits of 7 bits (s = kfac_debug_ozaki_digits(), 5 by default),
and digit pairs with i + j > s + 1 are dropped, so |C - A B| <= ~3 K 2^-(7s-1) max|A[m,:]| max|B[:,n]|
element by element.  The test grades against 2^-(7s-5) K max|A[m,:]| max|B[:,n]| (16x margin) and a
relative Frobenius error <= 1e-11 * 2^(7(6-s)) (fp32 would be ~1e-7), on rows spanning 2^+-20
(per-row exponents), every transposition, ragged M/N/K, the C -= A B epilogue and fp32 output."""
import ctypes as C

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2007_00784_b200.build import build
    build()
    from paper_2007_00784_b200 import _lib
    f = _lib.lib.kfac_debug_ozaki
    f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int,
                  C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
    f.restype = C.c_int
    _lib.lib.kfac_debug_ozaki_digits.restype = C.c_int
    return _lib


def _digits(lib):
    return int(lib.lib.kfac_debug_ozaki_digits())


def _dev(x, dtype=torch.float64):
    r, c = x.shape
    ld = (c + 1) // 2 * 2
    t = torch.zeros(r, ld, dtype=dtype, device="cuda")
    t[:, :c] = torch.from_numpy(x)
    return t


@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 64, 256), (300, 200, 517), (1000, 777, 4609)])
def test_ozaki_gemm_fp64_accuracy(lib, ta, tb, M, N, K):
    rng = np.random.default_rng(M * 7 + N * 3 + K + 10 * ta + tb)
    A = rng.standard_normal((M, K)) * np.exp2(rng.integers(-20, 21, size=(M, 1)))
    B = rng.standard_normal((K, N)) * np.exp2(rng.integers(-20, 21, size=(1, N)))
    A[5] = 0.0                                    # an all-zero row (exponent 0, zero digits)
    a = _dev(A.T.copy() if ta else A)
    b = _dev(B.T.copy() if tb else B)
    c = torch.full((M, (N + 1) // 2 * 2), float("nan"), dtype=torch.float64, device="cuda")
    st = lib.lib.kfac_debug_ozaki(a.data_ptr(), a.stride(0), ta, b.data_ptr(), b.stride(0), tb,
                                  c.data_ptr(), 1, c.stride(0), M, N, K, 0, None)
    assert st == 0, lib.lib.kfac_last_error()
    torch.cuda.synchronize()
    got = c[:, :N].cpu().numpy()
    ref = A @ B
    s = _digits(lib)
    bound = 2.0 ** -(7 * s - 5) * K * np.abs(A).max(1)[:, None] * np.abs(B).max(0)[None, :]
    assert np.isfinite(got).all()
    assert (np.abs(got - ref) <= bound).all(), np.max(np.abs(got - ref) / np.maximum(bound, 1e-300))
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-11 * 2.0 ** (7 * (6 - s))


@pytest.mark.parametrize("out32", [False, True])
def test_ozaki_gemm_sub_epilogue(lib, out32):
    M, N, K = 257, 129, 1153
    rng = np.random.default_rng(3)
    A, B, C0 = rng.standard_normal((M, K)), rng.standard_normal((K, N)), rng.standard_normal((M, N))
    dt = torch.float32 if out32 else torch.float64
    a, b, c = _dev(A), _dev(B), _dev(C0.astype(np.float32).astype(np.float64) if out32 else C0, dt)
    st = lib.lib.kfac_debug_ozaki(a.data_ptr(), a.stride(0), 0, b.data_ptr(), b.stride(0), 0,
                                  c.data_ptr(), 0 if out32 else 1, c.stride(0), M, N, K, 3, None)
    assert st == 0, lib.lib.kfac_last_error()
    torch.cuda.synchronize()
    c0 = C0.astype(np.float32).astype(np.float64) if out32 else C0
    ref = c0 - A @ B
    got = c[:, :N].double().cpu().numpy()
    tol = 2.0 ** -23 if out32 else 1e-11 * 2.0 ** (7 * (6 - _digits(lib)))
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= tol

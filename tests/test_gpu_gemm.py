"""GPU: the tcgen05 3xTF32 planes GEMM against fp64 numpy (and the SIMT engine) for every
operand majorness, ragged tiles and K tails.  3xTF32 with a truncation split keeps the
per-product relative error ~2^-20, so relF <= 2e-6 against fp64 is the bar (1xTF32 would
be ~1e-3)."""
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
    f = _lib.lib.kfac_debug_gemm
    f.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int,
                  C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    f.restype = C.c_int
    return _lib


def _pad(x):
    r, c = x.shape
    ld = (c + 3) // 4 * 4
    t = torch.zeros(r, ld, dtype=torch.float32, device="cuda")
    t[:, :c] = torch.from_numpy(x.astype(np.float32))
    return t


def _run(lib, engine, A, ta, B, tb, M, N, K, debug=None, expect=0):
    a, b = _pad(A), _pad(B)
    c = torch.full((M, (N + 3) // 4 * 4), float("nan"), device="cuda")
    st = lib.lib.kfac_debug_gemm(engine, a.data_ptr(), a.stride(0), ta, b.data_ptr(), b.stride(0), tb,
                                 c.data_ptr(), c.stride(0), M, N, K,
                                 C.c_void_p(torch.cuda.current_stream().cuda_stream),
                                 C.c_void_p(debug.data_ptr() if debug is not None else None))
    assert st == expect, lib.lib.kfac_last_error()
    if st:
        return None
    torch.cuda.synchronize()
    return c[:, :N].double().cpu().numpy()


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (200, 72, 45), (512, 385, 1153), (64, 130, 4609)])
@pytest.mark.parametrize("emit_planes", [False, True])
def test_tc_planes_gemm_matches_fp64(lib, ta, tb, M, N, K, emit_planes):
    """The pre-split planes engine (split_planes + gemm_tc_planes_kernel, the preconditioning
    chain's engine): same bar as the in-kernel split; with emit_planes the product leaves as
    TF32 planes (hi in C, lo in a second buffer) whose sum is the fp32 result."""
    rng = np.random.default_rng(M + N + K + 10 * ta + tb + 7)
    A = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32).astype(np.float64)
    B = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32).astype(np.float64)
    ref = (A.T if ta else A) @ (B.T if tb else B)
    lo = torch.zeros((M, (N + 3) // 4 * 4), device="cuda") if emit_planes else None
    got = _run(lib, 2, A, ta, B, tb, M, N, K, debug=lo)
    if emit_planes:
        lo_h = lo[:, :N].double().cpu().numpy()
        # both planes are exact TF32 values (low 13 mantissa bits zero)
        for plane in (torch.from_numpy(got).float(), lo[:, :N].cpu()):
            bits = plane.contiguous().view(torch.int32)
            assert int((bits & 0x1FFF).abs().sum()) == 0
        got = got + lo_h
    assert np.isfinite(got).all()
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= 2e-6, err

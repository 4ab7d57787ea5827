"""GPU: the tcgen05 3xTF32 GEMM core against fp64 numpy (and the SIMT engine) for every
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


def _run(lib, engine, A, ta, B, tb, M, N, K, debug=None):
    a, b = _pad(A), _pad(B)
    c = torch.full((M, (N + 3) // 4 * 4), float("nan"), device="cuda")
    st = lib.lib.kfac_debug_gemm(engine, a.data_ptr(), a.stride(0), ta, b.data_ptr(), b.stride(0), tb,
                                 c.data_ptr(), c.stride(0), M, N, K,
                                 C.c_void_p(torch.cuda.current_stream().cuda_stream),
                                 C.c_void_p(debug.data_ptr() if debug is not None else None))
    assert st == 0, lib.lib.kfac_last_error()
    torch.cuda.synchronize()
    return c[:, :N].double().cpu().numpy()


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (200, 72, 45), (512, 385, 1153), (64, 130, 4609)])
def test_tc_gemm_matches_fp64(lib, ta, tb, M, N, K):
    rng = np.random.default_rng(M + N + K + 10 * ta + tb)
    A = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32).astype(np.float64)
    B = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32).astype(np.float64)
    ref = (A.T if ta else A) @ (B.T if tb else B)
    got = _run(lib, 1, A, ta, B, tb, M, N, K)
    assert np.isfinite(got).all()
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= 2e-6, err
    simt = _run(lib, 0, A, ta, B, tb, M, N, K)
    assert np.linalg.norm(simt - ref) / np.linalg.norm(ref) <= 2e-6


@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4])
def test_tc_probe(lib, mode):
    """Minimal tcgen05 experiments: TMEM st/ld round trip and one 128x128x8 tf32 MMA with
    no-swizzle / 128B-swizzle K-major shared-memory descriptors."""
    f = lib.lib.kfac_debug_tc_probe
    f.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint, C.c_void_p]
    rng = np.random.default_rng(1)
    kk = 32 if mode >= 3 else 8
    A = rng.integers(-4, 5, size=(128, kk)).astype(np.float32)
    B = rng.integers(-4, 5, size=(128, kk)).astype(np.float32)
    a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    results = {}
    for name, idesc in [("default", 0), ("m_at_23", (1 << 4) | (2 << 7) | (2 << 10) | (16 << 17) | (8 << 23))]:
        out = torch.full((128, 128), float("nan"), device="cuda")
        bb = torch.from_numpy(B.T.copy()).cuda() if mode >= 4 else b
        assert f(mode, a.data_ptr(), bb.data_ptr(), out.data_ptr(), idesc, None) == 0
        torch.cuda.synchronize()
        o = out.cpu().numpy().astype(np.float64)
        if mode == 0:
            ref = np.arange(128)[:, None] * 1000.0 + (np.arange(128) % 32)[None, :]
        elif mode >= 4:
            Bkn = B.T.copy()                     # pass B as K x N (n contiguous)
            ref = A.astype(np.float64) @ Bkn.astype(np.float64)
        else:
            ref = A.astype(np.float64) @ B.T.astype(np.float64)
        results[name] = (np.abs(o - ref).max(), int((o == 0).sum()), o[0, :6].tolist(), ref[0, :6].tolist())
        print(mode, name, results[name])
        if mode in (0, 3, 4, 5):
            break
    assert results["default"][0] == 0, results


def test_tf32_operand_conversion_probe(lib):
    """Does the tensor core truncate or round fp32 operands to TF32?  A = 1 + 3*2^-12 (0.75 TF32
    ulp above 1), B = e_0: truncation gives exactly 1, round-to-nearest 1 + 2^-10.  The 3xTF32
    split (hi = rn_tf32(x), lo = rn_tf32(x - hi)) is exact either way; this records the mode."""
    f = lib.lib.kfac_debug_tc_probe
    f.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint, C.c_void_p]
    A = np.full((128, 8), 1.0 + 3 * 2.0 ** -12, np.float32)
    B = np.zeros((128, 8), np.float32)
    B[:, 0] = 1.0
    out = torch.full((128, 128), float("nan"), device="cuda")
    assert f(2, torch.from_numpy(A).cuda().data_ptr(), torch.from_numpy(B).cuda().data_ptr(), out.data_ptr(), 0, None) == 0
    torch.cuda.synchronize()
    v = float(out[0, 0])
    print("tf32 conversion of 1+3*2^-12 ->", repr(v), "truncation" if v == 1.0 else "round-to-nearest" if v == 1.0 + 2 ** -10 else "?")
    assert v in (1.0, 1.0 + 2 ** -10)


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

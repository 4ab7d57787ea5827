"""Diagnostics for the tridiagonal eigensolver path (run on a GPU box)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_00784_b200 import _lib  # noqa: E402

L = _lib.lib
L.kfac_debug_gemm.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int,
                              C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]


def gemm(engine, A, ta, B, tb, C0, ld=96):
    M = A.shape[1] if ta else A.shape[0]
    K = A.shape[0] if ta else A.shape[1]
    N = B.shape[0] if tb else B.shape[1]

    def dev(x, ld):
        t = torch.zeros(x.shape[0], ld, device="cuda")
        t[:, :x.shape[1]] = torch.from_numpy(x.astype(np.float32))
        return t
    ld = max(ld, (max(A.shape[1], B.shape[1], C0.shape[1]) + 3) // 4 * 4)
    a, b, c = dev(A, ld), dev(B, ld), dev(C0, ld)
    st = L.kfac_debug_gemm(engine, a.data_ptr(), ld, ta, b.data_ptr(), ld, tb, c.data_ptr(), ld, M, N, K, None, None)
    torch.cuda.synchronize()
    opA = A.T if ta else A
    opB = B.T if tb else B
    ref = (C0 - opA @ opB) if engine & 4 else opA @ opB
    got = c[:, :N].double().cpu().numpy()
    return st, np.linalg.norm(got - ref) / np.linalg.norm(ref)


rng = np.random.default_rng(0)
for (M, N, K) in [(64, 64, 64), (64, 65, 64), (63, 65, 63), (128, 129, 128)]:
    for ta in (0, 1):
        for tb in (0, 1):
            for epi in (0, 4):
                A = rng.standard_normal((K, M) if ta else (M, K))
                B = rng.standard_normal((N, K) if tb else (K, N))
                C0 = rng.standard_normal((M, N))
                for eng in (0, 1):
                    st, err = gemm(eng | epi, A, ta, B, tb, C0)
                    flag = "" if err < 1e-5 else "   <<<<<"
                    print(f"gemm M{M} N{N} K{K} ta{ta} tb{tb} epi{epi} eng{eng}: st={st} relerr={err:.2e}{flag}")

for n in (64, 65, 96, 97, 129, 300):
    X = rng.standard_normal((n // 2 + 3, n))
    F = (X.T @ X / X.shape[0]).astype(np.float32)
    ld = (n + 3) // 4 * 4
    f = torch.zeros(n, ld, device="cuda"); f[:, :n] = torch.from_numpy(F)
    q = torch.zeros(n, ld, device="cuda"); v = torch.zeros(n, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.kfac_compute_eigen([f], [q], [v], info=info, flags=4)
    torch.cuda.synchronize()
    Q = q[:, :n].double().cpu().numpy(); w = v.double().cpu().numpy()
    F64 = F.astype(np.float64)
    rec = np.linalg.norm((Q * w) @ Q.T - F64) / np.linalg.norm(F64)
    orth = np.abs(Q.T @ Q - np.eye(n)).max()
    werr = np.abs(w - np.clip(np.linalg.eigvalsh(F64), 0, None)).max() / np.abs(w).max()
    print(f"eig n={n}: rec={rec:.2e} orth={orth:.2e} werr={werr:.2e} info={int(info.item())}")

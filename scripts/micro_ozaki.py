"""Micro-benchmark: the Ozaki int8 tensor-core GEMM (kfac_debug_ozaki_ws, slicing included) against
the DMMA fp64 GEMM (kfac_debug_gemm64) and cuBLAS DGEMM on the eigensolver's shapes.  GPU only."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_00784_b200 import _lib  # noqa: E402

L = _lib.lib
L.kfac_debug_gemm64.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
L.kfac_debug_ozaki_ws.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                  C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_size_t, C.c_void_p]
L.kfac_debug_ozaki_bytes.argtypes = [C.c_int, C.c_int, C.c_int]
L.kfac_debug_ozaki_bytes.restype = C.c_size_t


def timeit(f, reps=5):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(M, N, K, ta, tb, epi):
    a = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda")
    b = torch.randn((N, K) if tb else (K, N), dtype=torch.float64, device="cuda")
    c = torch.randn((M, N), dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    nb = L.kfac_debug_ozaki_bytes(M, N, K)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    oz = lambda: L.kfac_debug_ozaki_ws(a.data_ptr(), a.stride(0), ta, b.data_ptr(), b.stride(0), tb, c.data_ptr(), 1,
                                       c.stride(0), M, N, K, epi, ws.data_ptr(), nb, s)
    dm = lambda: L.kfac_debug_gemm64(a.data_ptr(), 1, a.stride(0), ta, b.data_ptr(), 1, b.stride(0), tb,
                                     c.data_ptr(), 1, c.stride(0), M, N, K, epi, s)
    t_oz, t_dm = timeit(oz), timeit(dm)
    fl = 2.0 * M * N * K
    return t_oz, fl / t_oz / 1e9, t_dm, fl / t_dm / 1e9


for name, args in [("DC   4608^3", (4608, 4608, 4608, 0, 0, 0)),
                   ("DC   2304^3", (2304, 2304, 2304, 0, 0, 0)),
                   ("BT   Y=V^T X 512x4608x4608", (512, 4608, 4608, 1, 0, 0)),
                   ("BT   X-=V Y2 4608x4608x512", (4608, 4608, 512, 0, 0, 3)),
                   ("BT   Y2=T Y 512x4608x512", (512, 4608, 512, 0, 0, 0)),
                   ("DC   1152x2304x2304", (1152, 2304, 2304, 0, 0, 0)),
                   ("DC   576x1152x1152", (576, 1152, 1152, 0, 0, 0)),
                   ("DC   288x576x576", (288, 576, 576, 0, 0, 0)),
                   ("BT   X-=V Y2 2048x2048x512", (2048, 2048, 512, 0, 0, 3)),
                   ("BT   Y=V^T X 512x2048x2048", (512, 2048, 2048, 1, 0, 0))]:
    t_oz, f_oz, t_dm, f_dm = run(*args)
    print(f"{name:32s} ozaki {t_oz:8.3f} ms {f_oz:7.1f} TF/s | dmma {t_dm:8.3f} ms {f_dm:6.1f} TF/s | x{t_dm / t_oz:.2f}",
          flush=True)

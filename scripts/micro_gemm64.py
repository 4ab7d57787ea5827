"""Micro-benchmark of the eigensolver's fp64-accumulating GEMM (kfac_debug_gemm64) against
cuBLAS DGEMM (torch.matmul fp64) on the shapes the solver issues.  GPU only."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_00784_b200 import _lib  # noqa: E402

L = _lib.lib
L.kfac_debug_gemm64.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]


def run(M, N, K, ta, tb, dta, dtb, dtc, epi, reps=5):
    dt = lambda c: torch.float64 if c else torch.float32
    a = torch.randn((K, M) if ta else (M, K), dtype=dt(dta), device="cuda")
    b = torch.randn((N, K) if tb else (K, N), dtype=dt(dtb), device="cuda")
    c = torch.randn((M, N), dtype=dt(dtc), device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    f = lambda: L.kfac_debug_gemm64(a.data_ptr(), dta, a.stride(0), ta, b.data_ptr(), dtb, b.stride(0), tb,
                                    c.data_ptr(), dtc, c.stride(0), M, N, K, epi, s)
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tf = 2.0 * M * N * K / ms / 1e9
    return ms, tf


for name, args in [("DC   4096^3 f64", (4096, 4096, 4096, 0, 0, 1, 1, 1, 0)),
                   ("BT   Y=V^T X 512x4608x4608 (f32,f64)", (512, 4608, 4608, 1, 0, 0, 1, 1, 0)),
                   ("BT   X-=V Y2 4608x4608x512", (4608, 4608, 512, 0, 0, 0, 1, 1, 3)),
                   ("TRL  A-=VW^T 4576x4576x64 f32", (4576, 4576, 64, 0, 1, 0, 0, 0, 3))]:
    ms, tf = run(*args)
    print(f"{name:40s} {ms:8.3f} ms  {tf:6.2f} TF/s")
a = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
torch.matmul(a, a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    torch.matmul(a, a)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"{'cuBLAS DGEMM 4096^3':40s} {ms:8.3f} ms  {2 * 4096**3 / ms / 1e9:6.2f} TF/s")

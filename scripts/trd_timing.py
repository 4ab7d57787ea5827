"""Per-phase latency of the tridiagonalisation panel kernel for one factor (diagnostic).

Needs libkfac built with -DKFAC_TRD_TIMING=1:
    KFAC_NVCC_EXTRA=-DKFAC_TRD_TIMING=1 python -c "import __graft_entry__ as g; g.build()"
    python scripts/trd_timing.py [n] > gpurun_out/trd_timing.txt

Runs kfac_debug_tridiag on a seeded SPD matrix of order n (a K-FAC-like factor: X^T X / m with
m < n rows, plus a small ridge) and prints, for three CTAs of the group, the mean time per column
of each phase (clock64 cycles -> us at the measured SM clock) over column ranges.
"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2007_00784_b200 import _lib  # noqa: E402

PTS = ["A(+bar)", "B:tau", "B:v+V", "symv", "part+", "bar1", "C", "bar2", "D"]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4609
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 1568
    g = torch.Generator(device="cuda").manual_seed(7)
    X = torch.randn(m, n, device="cuda", generator=g)
    F = (X.T @ X) / m + 1e-3 * torch.eye(n, device="cuda")
    ld = (n + 3) // 4 * 4
    Fp = torch.zeros(n, ld, device="cuda")
    Fp[:, :n] = F
    d = torch.empty(n, dtype=torch.float64, device="cuda")
    e = torch.empty(n, dtype=torch.float64, device="cuda")
    fn = _lib.lib.kfac_debug_tridiag
    fn.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        st = fn(Fp.data_ptr(), n, ld, d.data_ptr(), e.data_ptr(), None)
        t1.record()
        torch.cuda.synchronize()
        assert st == 0, st
        print(f"rep {rep}: tridiagonalisation {t0.elapsed_time(t1):.2f} ms (n={n})")
    if not hasattr(_lib.lib, "kfac_debug_trd_timing"):
        print("(library built without -DKFAC_TRD_TIMING=1: no phase stamps)")
        return
    tim = np.zeros(3 * 8192 * 10, dtype=np.uint64)
    fn2 = _lib.lib.kfac_debug_trd_timing
    fn2.argtypes = [C.c_void_p, C.c_int]
    assert fn2(tim.ctypes.data, tim.size) == 0
    tim = tim.reshape(3, 8192, 10).astype(np.float64)
    ghz = 1.965
    for slot, name in enumerate(["cta first", "cta mid", "cta last"]):
        T = tim[slot, :n - 1]
        dur = np.diff(T, axis=1) / ghz / 1e3          # us per phase
        col = (T[:, 9] - T[:, 0]) / ghz / 1e3
        gap = (T[1:, 0] - T[:-1, 9]) / ghz / 1e3      # between columns (trailing update at panel ends)
        print(f"\n== {name}: column total mean {col.mean():.2f} us, sum {col.sum() / 1e3:.1f} ms; "
              f"inter-column gap sum {gap[gap > 0].sum() / 1e3:.1f} ms "
              f"(panel-end gaps mean {gap[31::32].mean():.1f} us)")
        print("cols        " + " ".join(f"{p:>8}" for p in PTS) + "    total")
        for a in range(0, n - 1, max(512, (n // 8) // 32 * 32)):
            b = min(n - 1, a + 512)
            s = dur[a:b].mean(axis=0)
            print(f"{a:5d}-{b:5d} " + " ".join(f"{x:8.2f}" for x in s) + f" {col[a:b].mean():8.2f}")


if __name__ == "__main__":
    main()

"""Per-step latencies of the bulge-chasing kernel (stage 2 of eigen_sbr.cu) for one lone factor.
Needs the diagnostic build: KFAC_NVCC_EXTRA=-DKFAC_SBR_TIMING=1 python scripts/sbr_chase_timing.py [n]
Prints, over the traced sweeps (s < 256), the median wait and compute time of a step, the lag
between consecutive sweeps' first steps, and the same split by CTA rank."""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_00784_b200.build import build  # noqa: E402

build(force=True)
from paper_2007_00784_b200 import _lib  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4609
rng = np.random.default_rng(n)
rows = 1568
X = rng.standard_normal((rows, n)).astype(np.float32)
X[:, -1] = 1
ld = (n + 3) // 4 * 4
F = torch.zeros(n, ld, device="cuda")
F[:, :n] = torch.from_numpy(X.T @ X / rows).cuda()
Q = torch.zeros_like(F)
v = torch.zeros(n, device="cuda")
ws = _lib.Workspace(torch.device("cuda"))
_lib.kfac_compute_eigen([F], [Q], [v], None, 0, ws=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
_lib.kfac_compute_eigen([F], [Q], [v], None, 0, ws=ws)
e1.record()
torch.cuda.synchronize()
total_ms = e0.elapsed_time(e1)
S, K = 256, 360
buf = np.zeros(S * K * 4, dtype=np.uint64)
L = _lib.lib
L.kfac_debug_sbr_timing.argtypes = [C.c_void_p, C.c_int]
assert L.kfac_debug_sbr_timing(buf.ctypes.data, buf.size) == 0
T = buf.reshape(S, K, 4).astype(np.int64)
valid = T[:, :, 2] > 0
t0 = T[valid][:, 0].min()
wait = (T[:, :, 1] - T[:, :, 0])[valid]
comp = (T[:, :, 2] - T[:, :, 1])[valid]
rank = T[:, :, 3][valid]
first = np.array([T[s, :, 1][valid[s]].min() if valid[s].any() else 0 for s in range(S)])
out = {"n": n, "eigen_ms": total_ms, "steps_traced": int(valid.sum()),
       "wait_ns_median": float(np.median(wait)), "compute_ns_median": float(np.median(comp)),
       "compute_ns_p90": float(np.percentile(comp, 90)),
       "sweep_lag_ns_median": float(np.median(np.diff(first[first > 0]))),
       "last_end_ns": int(T[valid][:, 2].max() - t0)}
for r in sorted(set(rank.tolist())):
    sel = rank == r
    out[f"rank{r}"] = {"steps": int(sel.sum()), "wait_med": float(np.median(wait[sel])),
                       "comp_med": float(np.median(comp[sel]))}
print(json.dumps(out, indent=1))
# sweep timelines (us from t0): (k, wait begin, step begin, step end)
for s in list(range(0, 40, 3)) + [100, 200]:
    ks = np.nonzero(valid[s])[0][:8]
    print(s, [(int(k), round((T[s, k, 0] - t0) / 1e3, 1), round((T[s, k, 1] - t0) / 1e3, 1),
               round((T[s, k, 2] - t0) / 1e3, 1)) for k in ks])
# full path of a few sweeps: (k, rank, wait us, step us) with the step's begin time
for s in (0, 1, 2, 3, 9, 100):
    ks = np.nonzero(valid[s])[0]
    print("sweep", s, " ".join(f"k{int(k)}r{int(T[s, k, 3])}:{(T[s, k, 1] - t0) / 1e3:.1f}+{(T[s, k, 2] - T[s, k, 1]) / 1e3:.1f}"
                                for k in ks[:24]))

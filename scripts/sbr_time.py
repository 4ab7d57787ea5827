"""Time kfac_compute_eigen on lone factors (cold, CUDA events) -- the latency of the largest
factors that bounds the eigen stage once each GPU owns one of them.
Usage: python scripts/sbr_time.py [n ...]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_00784_b200 import _lib  # noqa: E402

args = sys.argv[1:]
flags = 0
if args and args[0].startswith("--flags="):
    flags = int(args.pop(0).split("=")[1])          # 8: two-stage, 16: one-stage (kfac.h KFAC_EIG_*)
sizes = [int(x) for x in args] or [785, 1025, 2049, 2305, 4609]
ws = _lib.Workspace(torch.device("cuda"))
for n in sizes:
    rng = np.random.default_rng(n)
    rows = 1568 if n == 4609 else max(64, 2 * n)
    X = rng.standard_normal((rows, n)).astype(np.float32)
    X[:, -1] = 1
    ld = (n + 3) // 4 * 4
    F = torch.zeros(n, ld, device="cuda")
    F[:, :n] = torch.from_numpy(X.T @ X / rows).cuda()
    Q = torch.zeros_like(F)
    v = torch.zeros(n, device="cuda")
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.kfac_compute_eigen([F], [Q], [v], info, flags, ws=ws)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.kfac_compute_eigen([F], [Q], [v], info, flags, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    Qn = Q[:, :n].double()
    rec = float(torch.linalg.norm((Qn * v.double()) @ Qn.T - F[:, :n].double()) / torch.linalg.norm(F[:, :n].double()))
    print(json.dumps({"n": n, "flags": flags, "ms": min(ts), "all_ms": ts, "info": int(info.item()), "rel_rec": rec}), flush=True)

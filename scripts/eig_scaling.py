"""Projected eigen-stage time at W = 1, 2, 4, 8 GPUs, measured on ONE B200.

For each W the factors are assigned to ranks exactly as a W-rank run does (kfac_assign, LPT on
d^3, the same call the preconditioner makes), and each rank's owned factor set is then
eigendecomposed alone on this GPU (CUDA events); the stage time at W is the max over ranks.  It
excludes the eigenbasis all-gather (NVLink) and assumes identical GPUs -- a projection, printed
as one JSON line per W.  Usage: python scripts/eig_scaling.py [--config r50] [--reps 2]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_00784_b200 import _lib  # noqa: E402
from paper_2007_00784_b200.preconditioner import KFACPreconditioner  # noqa: E402
from workloads import shapes  # noqa: E402
from workloads.gen import layer_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="r50")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
layers = shapes.layers_for(a.config)
hp = shapes.HPARAMS[a.config]
acts, gouts, _ = layer_inputs(layers, seed=0, device="cuda")
pc = KFACPreconditioner(layers, damping=hp["damping"], xi=hp["xi"])
pc.update_factors([torch.from_numpy(x).cuda() for x in acts], [torch.from_numpy(x).cuda() for x in gouts], True)
torch.cuda.synchronize()
dims, layer_of = pc.dims, pc.layer_of
ws = _lib.Workspace(torch.device("cuda"))
for W in (1, 2, 4, 8):
    owner = _lib.kfac_assign(dims, layer_of, len(layers), W, _lib.LPT_D3)
    per_rank = []
    for r in range(W):
        fs = [f for f in range(len(dims)) if owner[f] == r]
        if not fs:
            per_rank.append(0.0)
            continue
        F = [pc.F[f] for f in fs]
        Q = [pc.Q[f] for f in fs]
        v = [pc.v[f] for f in fs]
        info = torch.zeros(len(fs), dtype=torch.int32, device="cuda")
        _lib.kfac_compute_eigen(F, Q, v, info, 0, ws=ws)          # warm-up (workspace, attributes)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            _lib.kfac_compute_eigen(F, Q, v, info, 0, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        per_rank.append(e0.elapsed_time(e1) / a.reps)
    print(json.dumps({"config": a.config, "world_size": W, "eigen_ms_max_over_ranks": max(per_rank),
                      "eigen_ms_per_rank": per_rank,
                      "largest_factor_per_rank": [max([dims[f] for f in range(len(dims)) if owner[f] == r] or [0])
                                                  for r in range(W)]}), flush=True)

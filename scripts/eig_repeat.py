"""Determinism probe: decompose the same full-size factor batch many times and compare every
output bit for bit with the first call (a race shows up as a changed result).
Usage: python scripts/eig_repeat.py [r50] [reps]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2007_00784_b200.preconditioner import KFACPreconditioner  # noqa: E402
from workloads import shapes  # noqa: E402
from workloads.gen import layer_inputs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "r50"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
flags = 0
layers = shapes.layers_for(cfg)
hp = shapes.HPARAMS[cfg]
acts, gouts, _ = layer_inputs(layers, seed=7, with_grad=False)
pc = KFACPreconditioner(layers, damping=hp["damping"], xi=hp["xi"], kappa=hp["kappa"], lr=hp["lr"])
pc.update_factors([torch.from_numpy(a).cuda() for a in acts], [torch.from_numpy(g).cuda() for g in gouts], True)
torch.cuda.synchronize()
ref = None
diffs = []
for it in range(reps):
    for q in pc.Q:
        q.fill_(float("nan"))
    pc.compute_eigen()
    torch.cuda.synchronize()
    cur = [(q.cpu().numpy().copy(), v.cpu().numpy().copy()) for q, v in zip(pc.Q, pc.v)]
    if ref is None:
        ref = cur
        continue
    bad = [f for f, ((q0, v0), (q1, v1)) in enumerate(zip(ref, cur))
           if not (np.array_equal(q0, q1, equal_nan=True) and np.array_equal(v0, v1))]
    if bad:
        diffs.append({"rep": it, "factors": bad[:10], "dims": [pc.dims[f] for f in bad[:10]]})
print(json.dumps({"config": cfg, "reps": reps, "flags": flags, "nondeterministic_reps": len(diffs),
                  "first": diffs[:5]}), flush=True)

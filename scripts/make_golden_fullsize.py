"""Write oracle-only golden values for the full-size ResNet-50 3x3 layers (tests/golden/).

Calls only `oracle/` (FP64 plain C) and `workloads/` (seeded inputs, no K-FAC arithmetic); nothing
here touches the CUDA path.  The oracle needs minutes per layer (a d = 4609 eigendecomposition is
~7 min single-threaded), too long for a test, so its result is stored once:

  * layer4.0.conv2 (d_A 4609, d_G 512, 1568 rows) and layer3.0.conv2 (2305, 256, 6272 rows) of
    ResNet-50 at batch 32, each drawn as a one-layer config with seed 5;
  * the oracle's full step (factors, eigen, Eqs. 13-15, kappa = 1e12 so nu = 1) -> P;
  * a seeded sample of P's rows (Eq. 15) stored as float64, plus the per-layer
    fp32 noise floor of SURVEY 8(c) consequence 2 (oracle factors rounded to fp32, their exact
    eigendecomposition rounded to fp32, the GEMM chain in fp32 arithmetic) on the same rows.

Usage: python scripts/make_golden_fullsize.py  (writes tests/golden/r50_<layer>.npz)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from workloads import shapes  # noqa: E402
from workloads.gen import layer_inputs  # noqa: E402

SEED = 5
NROWS = 32


def sample_rows(d_g, name):
    g = np.random.Generator(np.random.Philox(key=[SEED, sum(map(ord, name))]))
    return np.sort(g.choice(d_g, size=min(NROWS, d_g), replace=False))


def main(names):
    layers = {l.name: l for l in shapes.resnet50()}
    hp = shapes.HPARAMS["r50"]
    for name in names:
        lay = layers[name]
        t0 = time.time()
        acts, gouts, grads = layer_inputs([lay], seed=SEED)
        ref = oracle.full_step([lay], acts, gouts, grads, hp["damping"], hp["lr"], 1e12)
        t1 = time.time()
        rows = sample_rows(lay.d_g, name)
        P = ref["P"][0]
        # fp32 noise floor on the same rows (SURVEY 8(c) consequence 2)
        f32 = lambda x: np.asarray(x, np.float32)
        QA, vA = oracle.symeig(f32(ref["A"][0]).astype(np.float64))
        QG, vG = oracle.symeig(f32(ref["G"][0]).astype(np.float64))
        QA, vA, QG, vG, W = f32(QA), f32(vA), f32(QG), f32(vG), f32(grads[0])
        V1 = (QG.T @ W) @ QA
        D = np.outer(vG, vA) + np.float32(hp["damping"])
        Pf = ((QG @ (V1 / np.maximum(D, np.float32(1e-12)))) @ QA.T).astype(np.float64)
        floor = float(np.linalg.norm(Pf[rows] - P[rows]) / np.linalg.norm(P[rows]))
        out = os.path.join(ROOT, "tests", "golden", f"r50_{name.replace('.', '_')}.npz")
        np.savez_compressed(out, rows=rows, P_rows=P[rows], floor=floor, seed=SEED,
                            oracle_seconds=t1 - t0, layer=name)
        print(f"{name}: oracle {t1 - t0:.0f} s, floor {floor:.3e} -> {out}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["layer3.0.conv2", "layer4.0.conv2"])

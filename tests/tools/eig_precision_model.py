"""CPU model of how eigendecomposition errors reach the preconditioned gradient.

ResNet-50 fc layer (2049 x 1000 factors from 32 rows; oracle factors): relF(P) against the fp64
oracle when (a) the exact eigenvectors get absolute noise eps per element, (b) the eigenvalues
get noise eps * max eigenvalue.  Run: python tests/tools/eig_precision_model.py (about 1 min).
Measured: eps = 1e-7 on Q -> relF(P) 1.8e-3; on the eigenvalues -> 1.4e-5 (floor 1.5e-5)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle as orc  # noqa: E402
from workloads import shapes  # noqa: E402
from workloads.gen import layer_inputs  # noqa: E402


def main():
    layers = shapes.resnet50()
    hp = shapes.HPARAMS["r50"]
    sub = [layers[53]]
    acts, gouts, grads = layer_inputs(sub, seed=5)
    ref = orc.full_step(sub, acts, gouts, grads, hp["damping"], hp["lr"], 1e12)
    A, G, W = ref["A"][0], ref["G"][0], grads[0]
    g = hp["damping"]
    f32 = lambda x: np.asarray(x, np.float32).astype(np.float64)
    relF = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)

    def P_of(QA, vA, QG, vG):
        V1 = QG.T @ W @ QA
        return QG @ (V1 / (np.outer(vG, vA) + g)) @ QA.T

    wA, QA = np.linalg.eigh(f32(A))
    wG, QG = np.linalg.eigh(f32(G))
    wA, wG = np.clip(wA, 0, None), np.clip(wG, 0, None)
    Pref = ref["P"][0]
    print("lambda_max A %.3g G %.3g, damping %g" % (wA.max(), wG.max(), g))
    print("floor (exact eig of fp32 factors):", relF(P_of(f32(QA), wA, f32(QG), wG), Pref))
    rng = np.random.default_rng(0)
    for eps in (1e-8, 1e-7, 1e-6):
        qa = QA + eps * rng.standard_normal(QA.shape)
        qg = QG + eps * rng.standard_normal(QG.shape)
        va = np.clip(wA + eps * wA.max() * rng.standard_normal(len(wA)), 0, None)
        vg = np.clip(wG + eps * wG.max() * rng.standard_normal(len(wG)), 0, None)
        print(f"eps {eps:g}: Q noise relF(P) {relF(P_of(qa, wA, qg, wG), Pref):.3e}   "
              f"eigenvalue noise relF(P) {relF(P_of(QA, va, QG, vg), Pref):.3e}")


if __name__ == "__main__":
    main()

"""SURVEY 8(f)1 study: does a warm start from the previous eigenbasis pay on this workload?

Numpy fp64, CPU (a design study, not part of the path).  For factors of ResNet-50 layer shapes built
from the input recipe (workloads/gen.py: ReLU(N(0,1)) activations, N(0, 1/d_G) output gradients;
rows subsampled to `--rows` to keep it short), running averages with the configs' xi (Eqs. 16-17,
P:383-386) and an eigen refresh every `--interval` updates, it reports for the stale basis
Q of the previous refresh and the new factor F:
  off0      ||offdiag(Q^T F Q)||_F / ||F||_F       (how far from diagonal the warm start is)
  jac_cold  cyclic Jacobi sweeps from the identity to off <= tol
  jac_warm  cyclic Jacobi sweeps from Q to off <= tol
  oa        Ogita-Aishima refinement (RefSyEv: R = I - X^T X, S = X^T F X, quadratic when it
            converges; all GEMMs) -- the off-norm after each of 3 iterations, 'div' if it blows up
and the same with a much smaller xi (a nearly frozen factor) for contrast.
Usage: python scripts/warm_start_study.py [--rows 4096] [--interval 10]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from workloads import shapes  # noqa: E402


def off(S):
    return np.linalg.norm(S - np.diag(np.diag(S))) / np.linalg.norm(S)


def jacobi_sweeps(F, X, tol=1e-7, max_sweeps=30):
    S = X.T @ F @ X
    d = len(S)
    for sweep in range(max_sweeps):
        if off(S) <= tol:
            return sweep
        for p in range(d - 1):
            for q in range(p + 1, d):
                if abs(S[p, q]) < 1e-300:
                    continue
                th = (S[q, q] - S[p, p]) / (2 * S[p, q])
                t = np.sign(th) / (abs(th) + np.sqrt(th * th + 1)) if th != 0 else 1.0
                c = 1 / np.sqrt(t * t + 1)
                s = t * c
                Sp, Sq = S[:, p].copy(), S[:, q].copy()
                S[:, p], S[:, q] = c * Sp - s * Sq, s * Sp + c * Sq
                Sp, Sq = S[p, :].copy(), S[q, :].copy()
                S[p, :], S[q, :] = c * Sp - s * Sq, s * Sp + c * Sq
    return max_sweeps if off(S) > tol else max_sweeps


def ogita_aishima(F, X, iters=3):
    out = []
    nF = np.linalg.norm(F, 2)
    for _ in range(iters):
        R = np.eye(len(F)) - X.T @ X
        S = X.T @ F @ X
        lam = np.diag(S) / (1 - np.diag(R))
        delta = 2 * (np.linalg.norm(S - np.diag(lam), 2) + nF * np.linalg.norm(R, 2))
        diff = lam[None, :] - lam[:, None]
        far = np.abs(diff) > delta
        E = np.where(far, (S + lam[None, :] * R) / np.where(far, diff, 1.0), R / 2)
        X = X + X @ E
        if not np.isfinite(X).all() or np.abs(X).max() > 1e6:
            out.append("div")
            break
        out.append(f"{off(X.T @ F @ X):.1e}")
    return out


def factor_batch(kind, d, rows, rng):
    if kind == "A":
        x = np.maximum(rng.standard_normal((rows, d - 1)), 0.0)
        x = np.hstack([x, np.ones((rows, 1))])
    else:
        x = rng.standard_normal((rows, d)) / np.sqrt(d)
    return x.T @ x / rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--interval", type=int, default=10)
    ap.add_argument("--jacobi-max-d", type=int, default=130)
    a = ap.parse_args()
    xi = shapes.HPARAMS["r50"]["xi"]
    rng = np.random.default_rng(0)
    cases = [("A", 65), ("G", 64), ("A", 129), ("A", 257), ("G", 256), ("A", 577)]
    for kind, d in cases:
        for x in (xi, 1e-3 / a.interval):
            rows = min(a.rows, 8 * d) if kind == "A" else a.rows
            F = factor_batch(kind, d, rows, rng)
            for _ in range(3 * a.interval):
                F = x * factor_batch(kind, d, rows, rng) + (1 - x) * F
            _, Q = np.linalg.eigh(F)
            Fn = F
            for _ in range(a.interval):
                Fn = x * factor_batch(kind, d, rows, rng) + (1 - x) * Fn
            rec = dict(factor=kind, d=d, rows=rows, xi=x, interval=a.interval, off0=off(Q.T @ Fn @ Q),
                       oa=ogita_aishima(Fn, Q.copy()))
            if d <= a.jacobi_max_d:
                rec["jac_cold"] = jacobi_sweeps(Fn, np.eye(d))
                rec["jac_warm"] = jacobi_sweeps(Fn, Q)
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()

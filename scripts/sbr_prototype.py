"""Design prototype (numpy, fp64) of the two-stage tridiagonalisation the CUDA path implements for
the large factors -- dense -> band (bandwidth b) -> tridiagonal -- and of the blocked application
of the stage-2 reflectors.  Not part of the product or of the oracle: it fixes the index algebra
(step rows, bulge extent, sweep dependencies, the reflector-block order) before it is written in
CUDA.  Run: python scripts/sbr_prototype.py
"""
import numpy as np


def house(x):
    """dlarfg: H = I - tau v v^T, v[0] = 1, H x = beta e_0."""
    alpha = x[0]
    xn = np.linalg.norm(x[1:])
    v = np.zeros_like(x)
    v[0] = 1.0
    if xn == 0.0:
        return v, 0.0, alpha
    beta = -np.copysign(np.hypot(alpha, xn), alpha)
    tau = (beta - alpha) / beta
    v[1:] = x[1:] / (alpha - beta)
    return v, tau, beta


def larft(V, tau):
    """forward columnwise T: H_0 H_1 ... = I - V T V^T."""
    k = V.shape[1]
    T = np.zeros((k, k))
    for j in range(k):
        T[j, j] = tau[j]
        if j:
            T[:j, j] = -tau[j] * T[:j, :j] @ (V[:, :j].T @ V[:, j])
    return T


def stage1(A, b):
    """dense -> lower band b.  Returns band matrix, list of (p, V, tau) panels."""
    A = A.copy()
    n = A.shape[0]
    panels = []
    p = 0
    while p + b < n:
        m = n - p - b
        P = A[p + b:, p:p + b].copy()          # m x b panel
        nb = min(b, m)
        V = np.zeros((m, b))
        tau = np.zeros(b)
        for j in range(nb):
            v, t, beta = house(P[j:, j])
            V[j:, j] = v
            tau[j] = t
            P[j:, j + 1:] -= t * np.outer(v, v @ P[j:, j + 1:])
            P[j, j] = beta
            P[j + 1:, j] = 0.0
        A[p + b:, p:p + b] = P
        A[p:p + b, p + b:] = P.T
        T = larft(V, tau)
        A22 = A[p + b:, p + b:]
        X = A22 @ V @ T
        M = T.T @ (V.T @ X)
        W = X - 0.5 * V @ M
        A[p + b:, p + b:] = A22 - V @ W.T - W @ V.T
        panels.append((p, V, tau))
        p += b
    return A, panels


def stage2(A, b, check_bulge=True):
    """lower band b -> tridiagonal by bulge chasing.  Step (s, k) acts on rows R_k = [a_k, e_k],
    a_k = s + 1 + k b; returns T and the reflectors {(s, k): (a, v, tau)} in application order."""
    A = A.copy()
    n = A.shape[0]
    refl = []
    maxdist = 0
    for s in range(n - 2):
        k = 0
        while True:
            a = s + 1 + k * b
            if a > n - 1:
                break
            e = min(a + b - 1, n - 1)
            c = s if k == 0 else a - b                 # column the reflector cleans
            x = A[a:e + 1, c].copy()
            v, tau, beta = house(x)
            # (i)/(ii): left on rows R_k, columns c .. a-1 (column c becomes beta e_0)
            cols = slice(c, a)
            A[a:e + 1, cols] -= tau * np.outer(v, v @ A[a:e + 1, cols])
            A[cols, a:e + 1] = A[a:e + 1, cols].T
            # (iii): two-sided on the diagonal block
            D = A[a:e + 1, a:e + 1]
            y = D @ v
            w = tau * y - 0.5 * tau * tau * (v @ y) * v
            A[a:e + 1, a:e + 1] = D - np.outer(v, w) - np.outer(w, v)
            # (iv): right on rows e+1 .. e+b
            r1 = min(e + b, n - 1)
            if e + 1 <= r1:
                B = A[e + 1:r1 + 1, a:e + 1]
                A[e + 1:r1 + 1, a:e + 1] = B - tau * np.outer(B @ v, v)
                A[a:e + 1, e + 1:r1 + 1] = A[e + 1:r1 + 1, a:e + 1].T
            refl.append((s, k, a, v, tau))
            if check_bulge:
                nz = np.argwhere(np.abs(np.tril(A)) > 1e-13 * np.abs(A).max())
                maxdist = max(maxdist, int((nz[:, 0] - nz[:, 1]).max()))
            k += 1
    return A, refl, maxdist


def apply_q2_sequential(refl, Z):
    Z = Z.copy()
    for (s, k, a, v, tau) in reversed(refl):
        L = len(v)
        Z[a:a + L] -= tau * np.outer(v, v @ Z[a:a + L])
    return Z


def apply_q2_blocked(refl, Z, b, nb):
    """groups G(j, k) = {H_(s,k) : s in [j nb, (j+1) nb)} applied j descending, k ascending, each
    as one WY block I - V T V^T (V: (b + nb - 1) x nb parallelogram, rows from a_min)."""
    Z = Z.copy()
    groups = {}
    for (s, k, a, v, tau) in refl:
        groups.setdefault((s // nb, k), []).append((s, a, v, tau))
    J = max(j for j, _ in groups)
    for j in range(J, -1, -1):
        ks = sorted(k for (jj, k) in groups if jj == j)
        for k in ks:
            mem = sorted(groups[(j, k)], key=lambda t: t[0])   # product order: s ascending
            a0 = mem[0][1]
            rows = max(a + len(v) for (_, a, v, _) in mem) - a0
            V = np.zeros((rows, len(mem)))
            tau = np.zeros(len(mem))
            for i, (s, a, v, t) in enumerate(mem):
                V[a - a0:a - a0 + len(v), i] = v
                tau[i] = t
            T = larft(V, tau)
            Zs = Z[a0:a0 + rows]
            Z[a0:a0 + rows] = Zs - V @ (T @ (V.T @ Zs))
    return Z


def main():
    rng = np.random.default_rng(0)
    for n, b, nb in [(40, 4, 4), (67, 8, 4), (130, 16, 8), (97, 16, 16), (200, 16, 16)]:
        X = rng.standard_normal((n + 5, n))
        F = X.T @ X / n
        Bd, panels = stage1(F, b)
        band_ok = np.abs(np.tril(Bd, -b - 1)).max()
        T, refl, maxdist = stage2(Bd, b, check_bulge=(n <= 100))
        off = np.abs(np.tril(T, -2)).max()
        w_true = np.linalg.eigvalsh(F)
        d = np.diag(T)
        e = np.diag(T, -1)
        Tt = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
        wT, ZT = np.linalg.eigh(Tt)
        Zs = apply_q2_sequential(refl, ZT)
        Zb = apply_q2_blocked(refl, ZT, b, nb)
        # Q1 (Z): reflectors of panel p act on rows p + b + i ..
        Q = Zb.copy()
        for (p, V, tau) in reversed(panels):
            for i in range(V.shape[1] - 1, -1, -1):
                r0 = p + b
                v = V[:, i]
                Q[r0:] -= tau[i] * np.outer(v, v @ Q[r0:])
        rec = np.linalg.norm(Q @ np.diag(wT) @ Q.T - F) / np.linalg.norm(F)
        orth = np.abs(Q.T @ Q - np.eye(n)).max()
        print(f"n={n} b={b} nb={nb}: band {band_ok:.1e} bulge<= {maxdist} (2b-1={2*b-1}) tri-off {off:.1e} "
              f"eig {np.abs(wT - w_true).max() / w_true.max():.1e} blocked-vs-seq {np.abs(Zb - Zs).max():.1e} "
              f"rec {rec:.1e} orth {orth:.1e} steps {len(refl)}")


if __name__ == "__main__":
    main()


def stage2_wavefront(A, b, lag):
    """Same steps as stage2, executed in the order of t = lag s + k (a parallel schedule in which
    sweep s + 1 step k runs after sweep s step k + lag - 1).  Equal to stage2 bit for bit iff every
    pair of steps sharing a time slot touches disjoint entries."""
    n = A.shape[0]
    steps = []
    for s in range(n - 2):
        k = 0
        while s + 1 + k * b <= n - 1:
            steps.append((lag * s + k, s, k))
            k += 1
    steps.sort()
    A = A.copy()
    for _, s, k in steps:
        a = s + 1 + k * b
        e = min(a + b - 1, n - 1)
        c = s if k == 0 else a - b
        v, tau, beta = house(A[a:e + 1, c].copy())
        cols = slice(c, a)
        A[a:e + 1, cols] -= tau * np.outer(v, v @ A[a:e + 1, cols])
        A[cols, a:e + 1] = A[a:e + 1, cols].T
        D = A[a:e + 1, a:e + 1]
        y = D @ v
        w = tau * y - 0.5 * tau * tau * (v @ y) * v
        A[a:e + 1, a:e + 1] = D - np.outer(v, w) - np.outer(w, v)
        r1 = min(e + b, n - 1)
        if e + 1 <= r1:
            B = A[e + 1:r1 + 1, a:e + 1]
            A[e + 1:r1 + 1, a:e + 1] = B - tau * np.outer(B @ v, v)
            A[a:e + 1, e + 1:r1 + 1] = A[e + 1:r1 + 1, a:e + 1].T
    return A


def check_schedule():
    rng = np.random.default_rng(1)
    n, b = 90, 8
    X = rng.standard_normal((n, n))
    Bd, _ = stage1(X.T @ X / n, b)
    T, _, _ = stage2(Bd, b, check_bulge=False)
    for lag in (2, 3):
        Tw = stage2_wavefront(Bd, b, lag)
        print(f"wavefront lag {lag}: max |T_wave - T_seq| = {np.abs(Tw - T).max():.1e}")


if __name__ == "__main__":
    check_schedule()

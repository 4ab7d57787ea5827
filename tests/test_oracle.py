"""Pins for the FP64 oracle (oracle/) against what the paper and mathematics fix.

Each test names the passage it checks.  None of them re-types the oracle's own
formula: they use the paper's printed values, closed forms, invariants, brute
force, or an independent library routine (numpy/LAPACK, torch conv2d).
"""
import numpy as np
import pytest
import torch

from conftest import golden, read_sections, relF
from workloads import shapes
from workloads.gen import random_matrix, random_spd


# ------------------------------------------------------------------ kron --
def test_kron_eq7_exact(orc):
    """Eq. 7: the worked Kronecker product, exact integers."""
    g = read_sections(golden("eq7_kron.txt"))
    out = orc.kron(g["A"], g["B"])
    assert out.shape == (6, 4)
    assert np.array_equal(out, g["KRON"])
    assert list(out[0]) == [5, 6, 10, 12] and list(out[-1]) == [27, 0, 36, 0]


def test_kron_identities(orc):
    """I2 (x) I3 = I6; mixed product (A(x)B)(C(x)D) = (AC)(x)(BD)."""
    assert np.array_equal(orc.kron(np.eye(2), np.eye(3)), np.eye(6))
    A, Cm = random_matrix((2, 2), 1), random_matrix((2, 2), 2)
    B, D = random_matrix((3, 3), 3), random_matrix((3, 3), 4)
    lhs = orc.kron(A, B) @ orc.kron(Cm, D)
    assert np.abs(lhs - orc.kron(A @ Cm, B @ D)).max() <= 1e-10


# --------------------------------------------------------------- im2col --
@pytest.mark.parametrize("cin,cout,k,stride,h", [(3, 5, 3, 1, 6), (4, 6, 3, 2, 7), (3, 4, 7, 2, 11),
                                                 (5, 3, 1, 1, 4), (8, 4, 1, 2, 6)])
def test_im2col_matches_library_conv(orc, cin, cout, k, stride, h):
    """im2col . W^T == direct convolution, pinned to torch.nn.functional.conv2d in
    fp64; fixes the (k_h, k_w, c) column order (R8), stride and zero padding (R9)."""
    layer = shapes.conv("c", 2, cin, cout, k, stride, h)
    rng = np.random.default_rng(0)
    act = rng.standard_normal(layer.act_shape).astype(np.float32)
    w = rng.standard_normal((cout, cin, k, k))
    b = rng.standard_normal(cout)
    X = orc.im2col(layer, act)
    assert X.shape == (layer.rows, layer.d_a)
    assert np.all(X[:, -1] == 1.0)                                         # bias column
    wflat = np.concatenate([w.transpose(0, 2, 3, 1).reshape(cout, -1), b[:, None]], 1)
    y = (X @ wflat.T).reshape(layer.batch, layer.h_out, layer.w_out, cout)
    ref = torch.nn.functional.conv2d(torch.from_numpy(act.astype(np.float64)).permute(0, 3, 1, 2),
                                     torch.from_numpy(w), torch.from_numpy(b),
                                     stride=stride, padding=k // 2).permute(0, 2, 3, 1).numpy()
    assert np.abs(y - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


def test_im2col_counting_and_linear_equivalence(orc):
    """3x3 on a 1x1x4x4 input, stride 1, pad 0 -> 4 rows x (9+1) cols;
    a 1x1 stride-1 conv equals a linear layer on the reshaped rows."""
    L = shapes.Layer("c", shapes.CONV2D, 1, 1, 4, 4, 2, 2, 2, 3, 3, 1, 1, 0, 0, 1)
    X = orc.im2col(L, np.arange(16, dtype=np.float32).reshape(1, 4, 4, 1))
    assert X.shape == (4, 10)
    assert list(X[0, :9]) == [0, 1, 2, 4, 5, 6, 8, 9, 10]
    c = shapes.conv("c", 2, 5, 3, 1, 1, 3)
    act = np.random.default_rng(1).standard_normal(c.act_shape).astype(np.float32)
    lin = shapes.linear("l", 2 * 3 * 3, 5, 3)
    assert np.array_equal(orc.im2col(c, act), orc.im2col(lin, act.reshape(-1, 5)))


# -------------------------------------------------------------- factors --
def test_covariance_is_xtx_over_n(orc):
    """A = a a^T averaged over rows (Eq. 5) == numpy X^T X / n (library)."""
    X = random_matrix((37, 11), 5)
    F = orc.covariance(X)
    assert np.abs(F - X.T @ X / 37).max() <= 1e-13
    assert np.array_equal(F, F.T)
    assert np.linalg.eigvalsh(F).min() >= -1e-13                          # PSD


def test_update_factors_conv_and_linear(orc):
    """Stage 1 end to end: A = im2col^T im2col / n with bias row = column means and
    corner 1 (R7), G = g^T g / n; first call seeds."""
    layers = [shapes.conv("c", 2, 3, 4, 3, 2, 7), shapes.linear("l", 9, 6, 5)]
    rng = np.random.default_rng(2)
    acts = [rng.standard_normal(l.act_shape).astype(np.float32) for l in layers]
    gouts = [rng.standard_normal(l.gout_shape).astype(np.float32) for l in layers]
    A, G = orc.update_factors(layers, acts, gouts, xi=0.95, first=True)
    for l, a, g, Af, Gf in zip(layers, acts, gouts, A, G):
        X = orc.im2col(l, a)
        n = l.rows
        assert np.abs(Af - X.T @ X / n).max() <= 1e-12
        assert np.abs(Gf - g.astype(np.float64).T @ g / n).max() <= 1e-12
        assert Af[-1, -1] == 1.0
        assert np.abs(Af[-1, :-1] - X[:, :-1].mean(0)).max() <= 1e-12


def test_running_average_rules(orc):
    """Eqs. 16-17: xi weights the new batch estimate.  S:190 examples: xi = 1 -> the
    batch estimate exactly; the first call seeds F = batch; a constant batch B is approached
    geometrically, |F_k - B| = (1 - xi)^k |F_0 - B|; and one step is the convex combination
    with weight xi on the batch (checked against the endpoints, not the formula)."""
    B = random_spd(6, 3)
    F0 = random_spd(6, 4)
    assert np.array_equal(orc.running_average(F0, B, 1.0, False), B)
    assert np.array_equal(orc.running_average(F0, B, 0.95, True), B)
    assert np.array_equal(orc.running_average(F0, B, 0.0, False), F0)
    F = F0
    for k in range(1, 8):
        F = orc.running_average(F, B, 0.9, False)
        assert np.isclose(np.linalg.norm(F - B), 0.1 ** k * np.linalg.norm(F0 - B), rtol=1e-9)
    F1 = orc.running_average(F0, B, 0.95, False)
    assert np.isclose(np.linalg.norm(F1 - B), 0.05 * np.linalg.norm(F0 - B), rtol=1e-12)
    assert np.isclose(np.linalg.norm(F1 - F0), 0.95 * np.linalg.norm(B - F0), rtol=1e-12)


def test_factor_average_over_ranks_is_global_batch(orc):
    """Data-parallel pin (Alg. 1): the average of per-rank factors over equal
    shards equals the factor of the concatenated global batch (linearity of Eq. 5)."""
    l_rank = shapes.conv("c", 2, 3, 4, 3, 1, 5)
    l_glob = shapes.conv("c", 4, 3, 4, 3, 1, 5)
    rng = np.random.default_rng(3)
    a = rng.standard_normal(l_glob.act_shape).astype(np.float32)
    g = rng.standard_normal(l_glob.gout_shape).astype(np.float32)
    Ag, Gg = orc.update_factors([l_glob], [a], [g])
    A0, G0 = orc.update_factors([l_rank], [a[:2]], [g[: l_rank.rows]])
    A1, G1 = orc.update_factors([l_rank], [a[2:]], [g[l_rank.rows:]])
    assert np.abs((A0[0] + A1[0]) / 2 - Ag[0]).max() <= 1e-12
    assert np.abs((G0[0] + G1[0]) / 2 - Gg[0]).max() <= 1e-12


def test_mean_of_local_running_averages_is_global_running_average(orc):
    """Reduce-to-owner pin: Eqs. 16-17 are linear, so the mean of
    the ranks' LOCAL running averages after k steps equals the running average of the global
    batches (each step's global factor is the mean of the shard factors, previous test) -- the
    factors need no exchange on iterations without an eigen refresh."""
    l_rank = shapes.conv("c", 2, 3, 4, 3, 1, 5)
    l_glob = shapes.conv("c", 4, 3, 4, 3, 1, 5)
    rng = np.random.default_rng(5)
    loc = [[None, None], [None, None]]
    glob = [None, None]
    for k in range(4):
        a = rng.standard_normal(l_glob.act_shape).astype(np.float32)
        g = rng.standard_normal(l_glob.gout_shape).astype(np.float32)
        first = k == 0
        A, G = orc.update_factors([l_glob], [a], [g], A=glob[0], G=glob[1], xi=0.3, first=first)
        glob = [A, G]
        for r in range(2):
            A, G = orc.update_factors([l_rank], [a[2 * r:2 * r + 2]], [g[r * l_rank.rows:(r + 1) * l_rank.rows]],
                                      A=loc[r][0], G=loc[r][1], xi=0.3, first=first)
            loc[r] = [A, G]
        for t in range(2):
            mean = (loc[0][t][0] + loc[1][t][0]) / 2
            assert np.abs(mean - glob[t][0]).max() <= 1e-12 * max(1.0, np.abs(glob[t][0]).max())
    # and the non-trivial part: the local averages themselves differ from the global one
    assert np.abs(loc[0][0][0] - glob[0][0]).max() > 1e-3


# ---------------------------------------------------------------- eigen --
@pytest.mark.parametrize("method", ["qr", "jacobi"])
def test_symeig_trivial_cases(orc, method):
    """I3 -> eigenvalues 1; diag(4,1) -> [1,4] ascending, Q a permutation."""
    Q, v = orc.symeig(np.eye(3), method)
    assert np.allclose(v, 1.0) and np.allclose(Q.T @ Q, np.eye(3))
    Q, v = orc.symeig(np.diag([4.0, 1.0]), method)
    assert np.allclose(v, [1.0, 4.0]) and np.allclose(np.abs(Q), [[0, 1], [1, 0]])


@pytest.mark.parametrize("d,deficit,method", [(6, 0, "qr"), (6, 0, "jacobi"), (40, 0, "qr"),
                                              (40, 25, "qr"), (40, 25, "jacobi"), (150, 0, "qr"),
                                              (257, 200, "qr")])
def test_symeig_against_lapack(orc, d, deficit, method):
    """Reconstruction <= 1e-12 ||F||, orthogonality, eigenvalues vs
    LAPACK dsyevd (numpy.linalg.eigh), trace = sum v, PSD clamp."""
    F = random_spd(d, 10 + d + deficit, rank_deficit=deficit)
    Q, v = orc.symeig(F, method)
    w_ref = np.clip(np.linalg.eigvalsh(F), 0, None)
    nF = np.linalg.norm(F)
    assert np.abs(v - w_ref).max() <= 1e-12 * nF
    assert np.all(np.diff(v) >= 0) and v.min() >= 0
    assert np.linalg.norm(Q @ np.diag(v) @ Q.T - F) <= 1e-12 * nF
    assert np.abs(Q.T @ Q - np.eye(d)).max() <= 1e-12
    assert abs(v.sum() - np.trace(F)) <= 1e-11 * nF


def test_symeig_clustered_spectrum(orc):
    """Huge exact clusters (identity + rank-1, and a zero block) -- the null-space case of
    rank-deficient conv factors (R11)."""
    u = random_matrix((60, 1), 9)
    F = np.eye(60) + u @ u.T
    F[40:, :] = 0
    F[:, 40:] = 0
    Q, v = orc.symeig(F)
    assert np.linalg.norm(Q @ np.diag(v) @ Q.T - F) <= 1e-12 * np.linalg.norm(F)
    assert np.abs(Q.T @ Q - np.eye(60)).max() <= 1e-12


# -------------------------------------------------------------- inverse --
def test_damped_inverse(orc):
    """I4 -> I4 and diag(2,4) -> diag(.5,.25); vs numpy.linalg.inv; Eq. 8:
    (A (x) G)^{-1} == A^{-1} (x) G^{-1}."""
    assert np.allclose(orc.damped_inverse(np.eye(4), 0.0), np.eye(4))
    assert np.allclose(orc.damped_inverse(np.diag([2.0, 4.0]), 0.0), np.diag([0.5, 0.25]))
    F = random_spd(30, 5)
    assert np.abs(orc.damped_inverse(F, 1e-3) - np.linalg.inv(F + 1e-3 * np.eye(30))).max() <= 1e-9
    A, G = random_spd(4, 6), random_spd(3, 7)
    lhs = orc.damped_inverse(orc.kron(A, G), 0.0)
    rhs = orc.kron(orc.damped_inverse(A, 0.0), orc.damped_inverse(G, 0.0))
    assert np.abs(lhs - rhs).max() <= 1e-8 * np.abs(rhs).max()
    with pytest.raises(np.linalg.LinAlgError):
        orc.damped_inverse(-np.eye(3), 0.0)


# ------------------------------------------------------- preconditioner --
def test_kron_solve_matches_library_solve(orc):
    """The brute-force oracle (R13) equals numpy.linalg.solve on the dense system."""
    A, G = random_spd(4, 11), random_spd(3, 12)
    W = random_matrix((3, 4), 13)
    M = orc.kron(A, G) + 0.1 * np.eye(12)
    x = np.linalg.solve(M, W.T.reshape(-1))                 # column-stacking vec
    assert np.abs(orc.kron_solve(A, G, W, 0.1) - x.reshape(4, 3).T).max() <= 1e-12


def test_eigen_preconditioner_vs_bruteforce_corpus(orc):
    """SPEC acceptance #2: 200 random SPD pairs, dims 2-8, gamma in
    {0, 1e-3, 1}: Eqs. 13-15 == (A(x)G + gamma I)^{-1} vec(W), <= 1e-8."""
    rng = np.random.default_rng(20)
    worst = 0.0
    for t in range(200):
        da, dg = rng.integers(2, 9, size=2)
        A, G = random_spd(int(da), 1000 + t), random_spd(int(dg), 2000 + t)
        W = random_matrix((int(dg), int(da)), 3000 + t)
        QA, vA = orc.symeig(A)
        QG, vG = orc.symeig(G)
        for gamma in (0.0, 1e-3, 1.0):
            P = orc.precondition(W, QG, vG, QA, vA, gamma, orc.EIGEN)
            ref = orc.kron_solve(A, G, W, gamma)
            worst = max(worst, np.abs(P - ref).max() / max(1.0, np.abs(ref).max()))
    assert worst <= 1e-8


def test_factored_equals_explicit_inverse(orc):
    """SPEC acceptance #3: the explicit damped inverse (Eq. 12,
    P:230) equals the eigen form with denominator (v_G+g)(v_A+g)^T, and equals
    kron((A+gI)^-1, (G+gI)^-1) vec(W); at g = 0 it agrees with Eq. 14; for
    g > 0 it differs from Eq. 14 (Table I's distinction)."""
    rng = np.random.default_rng(21)
    for t in range(50):
        da, dg = rng.integers(2, 9, size=2)
        A, G = random_spd(int(da), 4000 + t), random_spd(int(dg), 5000 + t)
        W = random_matrix((int(dg), int(da)), 6000 + t)
        QA, vA = orc.symeig(A)
        QG, vG = orc.symeig(G)
        for gamma in (1e-3, 1.0):
            Ai, Gi = orc.damped_inverse(A, gamma), orc.damped_inverse(G, gamma)
            Pinv = orc.precondition(W, Gi, None, Ai, None, gamma, orc.INVERSE)
            Pfac = orc.precondition(W, QG, vG, QA, vA, gamma, orc.FACTORED)
            x = orc.kron(Ai, Gi) @ W.T.reshape(-1)
            assert np.abs(Pinv - Pfac).max() <= 1e-8 * max(1.0, np.abs(Pinv).max())
            assert np.abs(Pinv - x.reshape(int(da), int(dg)).T).max() <= 1e-8 * max(1.0, np.abs(Pinv).max())
            Peig = orc.precondition(W, QG, vG, QA, vA, gamma, orc.EIGEN)
            assert np.abs(Peig - Pinv).max() > 0.0
        Ai, Gi = orc.damped_inverse(A, 0.0), orc.damped_inverse(G, 0.0)
        P0 = orc.precondition(W, Gi, None, Ai, None, 0.0, orc.INVERSE)
        assert np.abs(P0 - orc.precondition(W, QG, vG, QA, vA, 0.0, orc.EIGEN)).max() <= \
            1e-6 * max(1.0, np.abs(P0).max())


def test_preconditioner_closed_forms(orc):
    """A = G = I -> W/(1+g); g = 1e12 -> W/g; A = G = 0 factored and
    inverse -> W/g^2; identity factors, g = 0 -> W."""
    W = random_matrix((3, 5), 30)
    I3, I5 = np.eye(3), np.eye(5)
    one3, one5 = np.ones(3), np.ones(5)
    assert np.allclose(orc.precondition(W, I3, one3, I5, one5, 1e-3), W / 1.001, rtol=1e-14)
    assert np.allclose(orc.precondition(W, I3, one3, I5, one5, 0.0), W, rtol=1e-14)
    A, G = random_spd(5, 31), random_spd(3, 32)
    QA, vA = orc.symeig(A)
    QG, vG = orc.symeig(G)
    assert relF(orc.precondition(W, QG, vG, QA, vA, 1e12), W / 1e12) <= 1e-6
    Z3, Z5 = np.zeros(3), np.zeros(5)
    assert np.allclose(orc.precondition(W, I3, Z3, I5, Z5, 0.1, orc.FACTORED), W / 0.01, rtol=1e-12)
    Ai, Gi = orc.damped_inverse(np.zeros((5, 5)), 0.1), orc.damped_inverse(np.zeros((3, 3)), 0.1)
    assert np.allclose(orc.precondition(W, Gi, None, Ai, None, 0.1, orc.INVERSE), W / 0.01, rtol=1e-12)


def test_full_chain_on_tiny_layer_vs_bruteforce(orc):
    """Stages 1-3 from raw activations: factors -> eigen -> Eq. 13-15 == brute-force
    Kronecker solve on the same factors (north_star's (A(x)G+gI)^{-1} vec(grad))."""
    from workloads.gen import layer_inputs
    layers = [shapes.conv("c", 2, 2, 3, 3, 1, 4), shapes.linear("l", 16, 5, 4)]
    acts, gouts, grads = layer_inputs(layers, seed=7)
    out = orc.full_step(layers, acts, gouts, grads, damping=3e-3, lr=0.1, kappa=1e12)
    assert out["nu"] == 1.0
    for i in range(2):
        ref = orc.kron_solve(out["A"][i], out["G"][i], grads[i], 3e-3)
        assert relF(out["P"][i], ref) <= 1e-9


# -------------------------------------------------------------- KL-clip --
def test_kl_clip_closed_forms(orc):
    """Eq. 18: kappa = 1e12 -> nu = 1; P = grad = [[1]], lr 1,
    kappa 0.25 -> nu = 0.5; when clipped lr^2 nu^2 s = kappa (R12); s = 0 -> 1."""
    _, nu, _ = orc.kl_clip([np.ones((2, 2))], [np.ones((2, 2))], 0.1, 1e12)
    assert nu == 1.0
    P, nu, s = orc.kl_clip([np.ones((1, 1))], [np.ones((1, 1))], 1.0, 0.25)
    assert nu == 0.5 and P[0][0, 0] == 0.5 and s == 1.0
    Ps = [random_matrix((4, 6), 40), random_matrix((3, 2), 41)]
    Ws = [random_matrix((4, 6), 42), random_matrix((3, 2), 43)]
    P2, nu, s = orc.kl_clip(Ps, Ws, 0.5, 1e-3)
    assert 0 < nu < 1
    assert abs(0.25 * nu * nu * s - 1e-3) <= 1e-15
    assert abs(s - sum(abs((p * w).sum()) for p, w in zip(Ps, Ws))) <= 1e-12
    for p, p0 in zip(P2, Ps):
        assert np.allclose(p, nu * p0, rtol=1e-15)
    _, nu, _ = orc.kl_clip([np.zeros((2, 2))], [np.ones((2, 2))], 0.1, 1e-3)
    assert nu == 1.0


def test_kl_terms_nonnegative_for_spd(orc):
    """Each per-layer term <P, grad> = vec(grad)^T M vec(grad) >= 0 for SPD M (R12)."""
    for t in range(20):
        A, G = random_spd(5, 700 + t), random_spd(4, 800 + t)
        W = random_matrix((4, 5), 900 + t)
        QA, vA = orc.symeig(A)
        QG, vG = orc.symeig(G)
        P = orc.precondition(W, QG, vG, QA, vA, 1e-3)
        assert (P * W).sum() >= 0

"""GPU parity: every C-ABI call against the FP64 oracle on the same seeded fp32 inputs.

Tolerances (north_star): factors relF <= 1e-4, preconditioned
gradients relF <= 1e-3.  Unit tests of a single call, fed identical fp32 inputs, use
tighter bounds derived from fp32 arithmetic (stated per test).  Eigenvectors are
compared only through reconstruction, orthogonality, eigenvalues and P (R11).
"""
import numpy as np
import pytest
import torch

from conftest import relF
from workloads import shapes
from workloads.gen import layer_inputs, random_matrix, random_spd

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2007_00784_b200.build import build
    build()
    from paper_2007_00784_b200 import _lib
    return _lib


def dev(x, ld=None):
    """fp32 device matrix with a padded leading dimension (multiple of 4)."""
    x = np.asarray(x, np.float32)
    if x.ndim == 1:
        return torch.from_numpy(x.copy()).cuda()
    r, c = x.shape
    ld = ld or (c + 3) // 4 * 4
    t = torch.zeros(r, ld, dtype=torch.float32, device="cuda")
    t[:, :c] = torch.from_numpy(x)
    return t[:, :c]


def host(t):
    return t.detach().double().cpu().numpy()


def empty(r, c):
    ld = (c + 3) // 4 * 4
    return torch.full((r, ld), float("nan"), dtype=torch.float32, device="cuda")[:, :c]


# ------------------------------------------------------------------ KL-clip --
@pytest.mark.parametrize("kappa", [1e-3, 1e12])
def test_kl_clip(L, orc, kappa):
    shp = [(7, 13), (64, 785), (10, 65), (300, 4)]
    Ps = [random_matrix(s, 100 + i).astype(np.float32) for i, s in enumerate(shp)]
    Ws = [random_matrix(s, 200 + i).astype(np.float32) for i, s in enumerate(shp)]
    ref, nu_ref, s_ref = orc.kl_clip(Ps, Ws, 0.1, kappa)
    P = [dev(p) for p in Ps]
    nu = torch.zeros(1, device="cuda")
    s = torch.zeros(1, dtype=torch.float64, device="cuda")
    L.kfac_kl_clip(P, [dev(w) for w in Ws], 0.1, kappa, nu, s)
    torch.cuda.synchronize()
    assert abs(s.item() - s_ref) <= 1e-6 * s_ref                 # fp32 products, fp64 sums
    assert abs(nu.item() - nu_ref) <= 1e-6 * nu_ref
    for p, r in zip(P, ref):
        assert relF(host(p), r) <= 2e-6


def test_kl_clip_deterministic_and_repeatable(L):
    shp = [(512, 4609), (1000, 2049)]
    P0 = [random_matrix(s, 300 + i).astype(np.float32) for i, s in enumerate(shp)]
    W = [dev(random_matrix(s, 400 + i)) for i, s in enumerate(shp)]
    outs = []
    for rep in range(3):
        P = [dev(p) for p in P0]
        s = torch.zeros(1, dtype=torch.float64, device="cuda")
        L.kfac_kl_clip(P, W, 0.1, 1e-3, None, s)
        outs.append((s.item(), [host(p) for p in P]))
    for o in outs[1:]:
        assert o[0] == outs[0][0]
        assert all(np.array_equal(a, b) for a, b in zip(o[1], outs[0][1]))


def test_kl_clip_many_layers_r152(L, orc):
    """ResNet-152's 156 layers in one call (more than one kernel-parameter chunk of layers),
    odd d_A (bias column) so every row ends in a masked float4 tail, padded ld with NaN pads."""
    layers = shapes.resnet152()
    assert len(layers) > 128
    g = np.random.Generator(np.random.Philox(key=[152, 7]))
    Ps, Ws, P, W = [], [], [], []
    for i, l in enumerate(layers):
        r, c = min(l.d_g, 96), min(l.d_a, 301)        # shapes of the real layers, trimmed for the oracle
        Ps.append(g.standard_normal((r, c)).astype(np.float32))
        Ws.append(g.standard_normal((r, c)).astype(np.float32))
        ld = (c + 3) // 4 * 4 + 4
        for src, dst in ((Ps[-1], P), (Ws[-1], W)):
            t = torch.full((r, ld), float("nan"), dtype=torch.float32, device="cuda")
            t[:, :c] = torch.from_numpy(src)
            dst.append(t[:, :c])
    ref, nu_ref, s_ref = orc.kl_clip(Ps, Ws, 0.0125, 1e-3)
    nu = torch.zeros(1, device="cuda")
    s = torch.zeros(1, dtype=torch.float64, device="cuda")
    L.kfac_kl_clip(P, W, 0.0125, 1e-3, nu, s)
    torch.cuda.synchronize()
    assert nu_ref < 1.0
    assert abs(s.item() - s_ref) <= 1e-6 * s_ref
    assert abs(nu.item() - nu_ref) <= 1e-6 * nu_ref
    for p, r in zip(P, ref):
        assert relF(host(p), r) <= 2e-6


# ---------------------------------------------------------- preconditioning --
def _eig_inputs(orc, dg, da, seed, deficit=0):
    G = random_spd(dg, seed, rank_deficit=min(deficit, dg - 1))
    A = random_spd(da, seed + 1, rank_deficit=min(deficit, da - 1))
    QG, vG = orc.symeig(G)
    QA, vA = orc.symeig(A)
    r = lambda x: np.asarray(x, np.float32).astype(np.float64)   # the fp32 inputs both sides see
    return r(QG), r(vG), r(QA), r(vA), A, G


@pytest.mark.parametrize("mode", [0, 1])
def test_precondition_eigen_modes(L, orc, mode):
    """Eqs. 13-15 on identical fp32 (Q, v, grad): fp32-faithful GEMM chain, relF <= 1e-5."""
    shp = [(64, 785), (10, 65), (130, 257), (1, 5), (33, 129)]
    layers = []
    for i, (dg, da) in enumerate(shp):
        QG, vG, QA, vA, _, _ = _eig_inputs(orc, dg, da, 10 * i)
        W = random_matrix((dg, da), 50 + i).astype(np.float32).astype(np.float64)
        layers.append((W, QG, vG, QA, vA))
    out = [empty(w.shape[0], w.shape[1]) for w, *_ in layers]
    L.kfac_precondition([dev(w) for w, *_ in layers], [dev(x[1]) for x in layers], [dev(x[2]) for x in layers],
                        [dev(x[3]) for x in layers], [dev(x[4]) for x in layers], 3e-3, mode, out)
    torch.cuda.synchronize()
    for (W, QG, vG, QA, vA), o in zip(layers, out):
        ref = orc.precondition(W, QG, vG, QA, vA, 3e-3, mode)
        assert relF(host(o), ref) <= 1e-5


def test_precondition_inverse_mode_and_alias(L, orc):
    """Eq. 12 with given inverses; out aliasing grad is allowed."""
    dg, da = 96, 200
    Gi = random_spd(dg, 7).astype(np.float32).astype(np.float64)
    Ai = random_spd(da, 8).astype(np.float32).astype(np.float64)
    W = random_matrix((dg, da), 9).astype(np.float32).astype(np.float64)
    g = dev(W)
    L.kfac_precondition([g], [dev(Gi)], None, [dev(Ai)], None, 1e-3, 2, [g])
    torch.cuda.synchronize()
    assert relF(host(g), Gi @ W @ Ai) <= 1e-5


# ------------------------------------------------------------------- factors --
FACTOR_LAYERS = [
    shapes.conv("c7s2", 2, 3, 16, 7, 2, 23),             # conv1-like, C_in = 3, pad 3
    shapes.conv("c3", 3, 20, 150, 3, 1, 9),              # ragged d_A = 181 (2 tiles), d_G = 150
    shapes.conv("c3s2", 2, 16, 40, 3, 2, 12, bias_col=0),
    shapes.conv("c1s2", 2, 130, 300, 1, 2, 8),           # d_A 131, d_G 300 (3 tiles)
    shapes.linear("fc", 37, 785, 64),
    shapes.linear("fc2", 5000, 20, 10),                  # 2 row chunks
    shapes.conv("c3big", 2, 64, 128, 3, 2, 30),          # tcgen05 path, im2col stride 2 + padding, d_A 577
    shapes.conv("c1big", 4, 256, 64, 1, 1, 36),          # tcgen05 path, 5184 rows = 2 row chunks
    shapes.conv("c7s2c3", 2, 3, 64, 7, 2, 40),           # C_in = 3 (ResNet conv1 shape): channel-padded
    shapes.conv("c5c5", 3, 5, 70, 5, 1, 14),             # C_in = 5, d_A 126, d_G 70: both padded
]


def test_update_factors_first_and_running_average(L, orc):
    layers = FACTOR_LAYERS
    a1, g1, _ = layer_inputs(layers, seed=1, with_grad=False)
    a2, g2, _ = layer_inputs(layers, seed=2, with_grad=False)
    A = [empty(l.d_a, l.d_a) for l in layers]
    G = [empty(l.d_g, l.d_g) for l in layers]
    L.kfac_update_factors(layers, [torch.from_numpy(a).cuda() for a in a1],
                          [torch.from_numpy(g).cuda() for g in g1], A, G, 0.95, True, 1.0)
    rA, rG = orc.update_factors(layers, a1, g1, xi=0.95, first=True)
    torch.cuda.synchronize()
    for x, r in zip(A + G, rA + rG):
        assert relF(host(x), r) <= 1e-5
        assert np.array_equal(host(x), host(x).T)                  # both triangles, bitwise symmetric
    # second call: running average with xi 0.95 and out_scale 0.5 (1/W before an allreduce-SUM)
    L.kfac_update_factors(layers, [torch.from_numpy(a).cuda() for a in a2],
                          [torch.from_numpy(g).cuda() for g in g2], A, G, 0.95, False, 0.5)
    rA, rG = orc.update_factors(layers, a2, g2, A=rA, G=rG, xi=0.95, first=False)
    torch.cuda.synchronize()
    for x, r in zip(A + G, rA + rG):
        assert relF(host(x), 0.5 * r) <= 1e-5


# --------------------------------------------------------------------- eigen --
@pytest.mark.parametrize("warm", [False, True])
def test_compute_eigen(L, orc, warm):
    dims = [1, 10, 16, 17, 64, 65, 150, 257, 577]
    Fs = [random_spd(d, 500 + d, rank_deficit=(d // 2 if d in (150, 577) else 0)) for d in dims]
    F32 = [f.astype(np.float32).astype(np.float64) for f in Fs]
    Fd = [dev(f) for f in F32]
    Q = [empty(d, d) for d in dims]
    v = [torch.full((d,), float("nan"), device="cuda") for d in dims]
    info = torch.full((len(dims),), -1, dtype=torch.int32, device="cuda")
    if warm:   # warm start from a perturbed-then-orthonormalised basis
        for q, f in zip(Q, F32):
            Qr, _ = np.linalg.qr(orc.symeig(f)[0] + 1e-2 * random_matrix(f.shape, 3))
            q.copy_(torch.from_numpy(Qr.astype(np.float32)))
    L.kfac_compute_eigen(Fd, Q, v, info, 1 if warm else 0)
    torch.cuda.synchronize()
    assert (info.cpu().numpy() == 0).all(), info
    for f, q, ev in zip(F32, Q, v):
        q, ev = host(q), host(ev)
        nf = np.linalg.norm(f)
        ref = np.clip(np.linalg.eigvalsh(f), 0, None)
        assert np.all(np.diff(ev) >= 0) and ev.min() >= 0
        assert np.abs(ev - ref).max() <= 2e-6 * nf                # Weyl bound on fp32 data
        assert np.abs(q.T @ q - np.eye(len(ev))).max() <= 2e-5
        assert np.linalg.norm(q @ np.diag(ev) @ q.T - f) <= 2e-5 * nf


# ------------------------------------------------------------------- inverse --
def test_compute_inverse(L, orc):
    dims = [5, 64, 65, 130, 300]
    Fs = [random_spd(d, 900 + d).astype(np.float32).astype(np.float64) for d in dims]
    Finv = [empty(d, d) for d in dims]
    info = torch.full((len(dims),), -1, dtype=torch.int32, device="cuda")
    L.kfac_compute_inverse([dev(f) for f in Fs], 1e-3, Finv, info)
    torch.cuda.synchronize()
    assert (info.cpu().numpy() == 0).all()
    for f, x in zip(Fs, Finv):
        ref = orc.damped_inverse(f, 1e-3)
        assert relF(host(x), ref) <= 1e-6                          # fp64 inside, fp32 output


def test_compute_inverse_reports_not_spd(L):
    F = -np.eye(8)
    Finv = [empty(8, 8)]
    info = torch.zeros(1, dtype=torch.int32, device="cuda")
    L.kfac_compute_inverse([dev(F)], 0.0, Finv, info)
    torch.cuda.synchronize()
    assert info.item() == 1


# ------------------------------------------------------------- full chains --
def _full_chain(L, layers, acts, gouts, grads, hp, variant="eigen"):
    from paper_2007_00784_b200.preconditioner import KFACPreconditioner
    pc = KFACPreconditioner(layers, damping=hp["damping"], xi=hp["xi"], kappa=hp["kappa"],
                            lr=hp["lr"], variant=variant)
    g = KFACPreconditioner.grad_buffer(layers, "cuda")
    for t, w in zip(g, grads):
        t.copy_(torch.from_numpy(w))
    P = pc.step([torch.from_numpy(a).cuda() for a in acts], [torch.from_numpy(x).cuda() for x in gouts], g,
                first=True)
    torch.cuda.synchronize()
    return pc, [host(p) for p in P]


@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
def test_full_step_mlp(L, orc, seed):
    """configs[0]: MLP 784->64->10, batch 128, gamma 0.003, eigen path (BASELINE.json)."""
    layers = shapes.mlp()
    hp = shapes.HPARAMS["mlp"]
    acts, gouts, grads = layer_inputs(layers, seed=seed)
    pc, P = _full_chain(L, layers, acts, gouts, grads, hp)
    ref = orc.full_step(layers, acts, gouts, grads, hp["damping"], hp["lr"], hp["kappa"])
    for x, r in zip(pc.A + pc.G, ref["A"] + ref["G"]):
        assert relF(host(x), r) <= 1e-4
    for p, r in zip(P, ref["P"]):
        assert relF(p, r) <= 1e-3
    assert abs(pc.nu.item() - ref["nu"]) <= 1e-4 * ref["nu"]


def _r32(x):
    return np.asarray(x, np.float32).astype(np.float64)


def _noise_floor(orc, layers, A, G, grads, hp, mode):
    """Per-layer floor: an fp32-faithful pipeline -- the oracle's factors rounded
    to fp32, the oracle's (exact) eigendecomposition / inverse of those rounded to fp32, and the
    preconditioning GEMM chain evaluated in fp32 arithmetic (numpy float32) -- against the
    all-fp64 oracle.  On rank-deficient layers the factored / inverse variants divide fp32
    accumulation noise by ~damping^2, so no fp32 pipeline can be closer than this."""
    g = np.float32(hp["damping"])
    f32 = lambda x: np.asarray(x, np.float32)
    if mode == 2:
        QA = [f32(orc.damped_inverse(_r32(a), float(g))) for a in A]
        QG = [f32(orc.damped_inverse(_r32(x), float(g))) for x in G]
    else:
        QA, vA = orc.symeig_batch([_r32(a) for a in A])
        QG, vG = orc.symeig_batch([_r32(x) for x in G])
        QA, QG, vA, vG = [f32(q) for q in QA], [f32(q) for q in QG], [f32(v) for v in vA], [f32(v) for v in vG]
    out = []
    for i, W in enumerate(grads):
        W = f32(W)
        if mode == 2:
            P = (QG[i] @ W) @ QA[i]
        else:
            V1 = (QG[i].T @ W) @ QA[i]
            D = np.outer(vG[i], vA[i]) + g if mode == 0 else np.outer(vG[i] + g, vA[i] + g)
            P = (QG[i] @ (V1 / np.maximum(D, np.float32(1e-12)))) @ QA[i].T
        out.append(P.astype(np.float64))
    full = orc.precondition_batch(grads, *orc_chain(orc, A, G, float(g), mode), float(g), mode)
    return [relF(p, f) for p, f in zip(out, full)]


def orc_chain(orc, A, G, g, mode):
    if mode == 2:
        return [orc.damped_inverse(x, g) for x in G], None, [orc.damped_inverse(a, g) for a in A], None
    QA, vA = orc.symeig_batch(A)
    QG, vG = orc.symeig_batch(G)
    return QG, vG, QA, vA


@pytest.mark.parametrize("variant", ["eigen", "factored", "inverse"])
def test_full_step_r32_small_batch(L, orc, variant):
    """ResNet-32 layer shapes (all 32 layers) at batch 4 so the oracle finishes in seconds.
    The eigen path is graded at relF <= 1e-3.  The factored / explicit-inverse variants divide
    by (v_G + g)(v_A + g) ~ g^2 on the null spaces of the rank-deficient stage-3 factors
    (256 rows, d_A = 577), where fp32 factor storage alone moves P; there they are graded
    against max(1e-3, 3 x the per-layer fp32-storage noise floor) (SURVEY 8(c) consequence 4)."""
    layers = shapes.resnet32(batch=4)
    hp = shapes.HPARAMS["r32"]
    acts, gouts, grads = layer_inputs(layers, seed=11)
    pc, P = _full_chain(L, layers, acts, gouts, grads, hp, variant)
    mode = {"eigen": 0, "factored": 1, "inverse": 2}[variant]
    ref = orc.full_step(layers, acts, gouts, grads, hp["damping"], hp["lr"], hp["kappa"], mode=mode)
    for x, r in zip(pc.A + pc.G, ref["A"] + ref["G"]):
        assert relF(host(x), r) <= 1e-4
    nu = ref["nu"]
    errs = [relF(p, r) for p, r in zip(P, ref["P"])]
    if variant == "eigen":
        assert max(errs) <= 1e-3, errs
    else:
        floors = _noise_floor(orc, layers, ref["A"], ref["G"], [g for g in grads], hp, mode)
        bound = [max(1e-3, 3 * f) for f in floors]
        bad = [(i, layers[i].name, e, f) for i, (e, f, b) in enumerate(zip(errs, floors, bound)) if e > b]
        assert not bad, bad


def test_full_size_r50_sampled_layers(L, orc):
    """Full ResNet-50 shapes (batch 32/GPU) for conv1 (401,408 rows, C_in = 3, SIMT SYRK), a
    1x1 conv (tcgen05 SYRK) and the fc layer (2049 x 1000 from 32 rows: both factors rank-
    deficient, the worst-conditioned layer of the network), checked one by one."""
    layers = shapes.resnet50()
    hp = shapes.HPARAMS["r50"]
    pick = [0, 1, 53]
    sub = [layers[i] for i in pick]
    acts, gouts, grads = layer_inputs(sub, seed=5)
    ref = orc.full_step(sub, acts, gouts, grads, hp["damping"], hp["lr"], 1e12)
    pc, P = _full_chain(L, sub, acts, gouts, grads, dict(hp, kappa=1e12))
    for x, r in zip(pc.A + pc.G, ref["A"] + ref["G"]):
        assert relF(host(x), r) <= 1e-4
    errs = [relF(p, r) for p, r in zip(P, ref["P"])]
    floors = _noise_floor(orc, sub, ref["A"], ref["G"], grads, dict(hp, kappa=1e12), 0)
    print("R50 sampled relF(P):", errs, "fp32-storage floors:", floors)
    assert max(errs) <= 1e-3, (errs, floors)


def test_packed_factor_outputs_roundtrip_bitwise(L):
    """packed_A/packed_G (the halved allreduce buffer) carry exactly the values written
    to the full factors: unpacking them reproduces both triangles bit for bit."""
    layers = FACTOR_LAYERS
    a1, g1, _ = layer_inputs(layers, seed=3, with_grad=False)
    A = [empty(l.d_a, l.d_a) for l in layers]
    G = [empty(l.d_g, l.d_g) for l in layers]
    pA = [torch.full((l.d_a * (l.d_a + 1) // 2,), float("nan"), device="cuda") for l in layers]
    pG = [torch.full((l.d_g * (l.d_g + 1) // 2,), float("nan"), device="cuda") for l in layers]
    L.kfac_update_factors(layers, [torch.from_numpy(a).cuda() for a in a1], [torch.from_numpy(g).cuda() for g in g1],
                          A, G, 0.95, True, 0.5, packed_A=pA, packed_G=pG)
    A2 = [empty(l.d_a, l.d_a) for l in layers]
    G2 = [empty(l.d_g, l.d_g) for l in layers]
    L.kfac_unpack_factors(pA + pG, A2 + G2)
    torch.cuda.synchronize()
    for x, y, p in zip(A + G, A2 + G2, pA + pG):
        assert torch.isfinite(p).all()
        assert torch.equal(x, y)

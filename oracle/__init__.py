"""FP64 CPU oracle of the K-FAC preconditioner hot path (ctypes over liboracle.so).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  It shares no
code with paper_2007_00784_b200/ (the CUDA path) and never imports it.

The arithmetic lives in kfac_oracle.c (plain C99, double precision); this
module only marshals numpy arrays.  `build()` compiles the C file with gcc.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_DIR, "kfac_oracle.c")
_LIB = os.path.join(_DIR, "liboracle.so")
_lib = None

EIGEN, FACTORED, INVERSE = 0, 1, 2
LPT_D3, ROUND_ROBIN_PAPER, LAYERWISE_LPT = 0, 1, 2


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_DIR, "kfac_oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-fopenmp", "-shared",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Layer(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "kind", "batch", "c_in", "h_in", "w_in", "c_out", "h_out", "w_out",
        "k_h", "k_w", "stride_h", "stride_w", "pad_h", "pad_w", "bias_col")]


_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int32)


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        L.orc_im2col.argtypes = [C.POINTER(_Layer), _fp, _dp]
        L.orc_covariance.argtypes = [_dp, C.c_int64, C.c_int32, _dp]
        L.orc_running_average.argtypes = [_dp, _dp, C.c_int32, C.c_double, C.c_int32]
        L.orc_update_factors.argtypes = [C.POINTER(_Layer), C.c_int32, C.POINTER(_fp), C.POINTER(_fp),
                                         C.POINTER(_dp), C.POINTER(_dp), C.c_double, C.c_int32]
        L.orc_symeig.argtypes = [_dp, C.c_int32, _dp, _dp]
        L.orc_symeig.restype = C.c_int
        L.orc_symeig_jacobi.argtypes = [_dp, C.c_int32, _dp, _dp]
        L.orc_symeig_jacobi.restype = C.c_int
        L.orc_damped_inverse.argtypes = [_dp, C.c_int32, C.c_double, _dp]
        L.orc_damped_inverse.restype = C.c_int
        L.orc_precondition.argtypes = [C.c_int32, C.c_int32, C.c_int32, _dp, _dp, _dp, _dp, _dp,
                                       C.c_double, _dp]
        L.orc_kl_clip.argtypes = [C.c_int32, C.POINTER(_dp), C.POINTER(_dp), C.POINTER(C.c_int64),
                                  C.c_double, C.c_double, _dp]
        L.orc_kl_clip.restype = C.c_double
        L.orc_kron.argtypes = [_dp, C.c_int32, C.c_int32, _dp, C.c_int32, C.c_int32, _dp]
        L.orc_kron_solve.argtypes = [_dp, C.c_int32, _dp, C.c_int32, C.c_double, _dp, _dp]
        L.orc_kron_solve.restype = C.c_int
        L.orc_assign.argtypes = [_ip, _ip, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _ip]
        L.orc_symeig_batch.argtypes = [C.c_int32, C.POINTER(_dp), _ip, C.POINTER(_dp), C.POINTER(_dp), _ip]
        L.orc_precondition_batch.argtypes = [C.c_int32, C.c_int32, _ip, _ip, C.POINTER(_dp),
                                             C.POINTER(_dp), C.POINTER(_dp), C.POINTER(_dp),
                                             C.POINTER(_dp), C.c_double, C.POINTER(_dp)]
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(_dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _layer(l) -> _Layer:
    t = l.as_tuple() if hasattr(l, "as_tuple") else tuple(l)
    return _Layer(*[int(v) for v in t])


def _ptrs(arrs, typ):
    return (typ * len(arrs))(*[a.ctypes.data_as(typ) for a in arrs])


# ----------------------------------------------------------------- stage 1 --
def im2col(layer, act) -> np.ndarray:
    act = _f32(act)
    X = np.empty((layer.rows, layer.d_a), np.float64)
    lib().orc_im2col(C.byref(_layer(layer)), act.ctypes.data_as(_fp), _d(X))
    return X


def covariance(X) -> np.ndarray:
    X = _f64(X)
    F = np.empty((X.shape[1], X.shape[1]), np.float64)
    lib().orc_covariance(_d(X), X.shape[0], X.shape[1], _d(F))
    return F


def running_average(F, Fb, xi, first) -> np.ndarray:
    F = _f64(F).copy()
    Fb = _f64(Fb)
    lib().orc_running_average(_d(F), _d(Fb), F.shape[0], float(xi), int(bool(first)))
    return F


def update_factors(layers, acts, gouts, A=None, G=None, xi=0.95, first=True):
    """Returns (A list, G list) in fp64 after one running-average update."""
    nl = len(layers)
    acts = [_f32(a) for a in acts]
    gouts = [_f32(g) for g in gouts]
    A = [np.zeros((l.d_a, l.d_a)) if A is None else _f64(A[i]).copy() for i, l in enumerate(layers)]
    G = [np.zeros((l.d_g, l.d_g)) if G is None else _f64(G[i]).copy() for i, l in enumerate(layers)]
    arr = (_Layer * nl)(*[_layer(l) for l in layers])
    lib().orc_update_factors(arr, nl, _ptrs(acts, _fp), _ptrs(gouts, _fp), _ptrs(A, _dp),
                             _ptrs(G, _dp), float(xi), int(bool(first)))
    return A, G


# ----------------------------------------------------------------- stage 2 --
def symeig(F, method: str = "qr"):
    """(Q, v): columns of Q are eigenvectors, v ascending, clamped >= 0."""
    F = _f64(F)
    d = F.shape[0]
    Q = np.empty((d, d))
    v = np.empty(d)
    fn = lib().orc_symeig if method == "qr" else lib().orc_symeig_jacobi
    st = fn(_d(F), d, _d(Q), _d(v))
    if st < 0:
        raise RuntimeError("oracle eigensolver did not converge")
    return Q, v


def symeig_batch(Fs):
    Fs = [_f64(F) for F in Fs]
    dims = np.array([F.shape[0] for F in Fs], np.int32)
    Qs = [np.empty_like(F) for F in Fs]
    vs = [np.empty(F.shape[0]) for F in Fs]
    st = np.zeros(len(Fs), np.int32)
    lib().orc_symeig_batch(len(Fs), _ptrs(Fs, _dp), dims.ctypes.data_as(_ip), _ptrs(Qs, _dp),
                           _ptrs(vs, _dp), st.ctypes.data_as(_ip))
    if (st < 0).any():
        raise RuntimeError("oracle eigensolver did not converge")
    return Qs, vs


def damped_inverse(F, gamma):
    F = _f64(F)
    Finv = np.empty_like(F)
    info = lib().orc_damped_inverse(_d(F), F.shape[0], float(gamma), _d(Finv))
    if info:
        raise np.linalg.LinAlgError(f"not SPD at pivot {info - 1}")
    return Finv


# ----------------------------------------------------------------- stage 3 --
def precondition(W, QG, vG, QA, vA, gamma, mode=EIGEN):
    W = _f64(W)
    dg, da = W.shape
    QG, QA = _f64(QG), _f64(QA)
    vG = _f64(vG if vG is not None else np.zeros(dg))
    vA = _f64(vA if vA is not None else np.zeros(da))
    P = np.empty_like(W)
    lib().orc_precondition(int(mode), dg, da, _d(W), _d(QG), _d(vG), _d(QA), _d(vA),
                           float(gamma), _d(P))
    return P


def precondition_batch(Ws, QGs, vGs, QAs, vAs, gamma, mode=EIGEN):
    Ws = [_f64(W) for W in Ws]
    QGs = [_f64(q) for q in QGs]
    QAs = [_f64(q) for q in QAs]
    vGs = [_f64(v) for v in vGs] if vGs is not None else [np.zeros(W.shape[0]) for W in Ws]
    vAs = [_f64(v) for v in vAs] if vAs is not None else [np.zeros(W.shape[1]) for W in Ws]
    dg = np.array([W.shape[0] for W in Ws], np.int32)
    da = np.array([W.shape[1] for W in Ws], np.int32)
    Ps = [np.empty_like(W) for W in Ws]
    lib().orc_precondition_batch(len(Ws), int(mode), dg.ctypes.data_as(_ip), da.ctypes.data_as(_ip),
                                 _ptrs(Ws, _dp), _ptrs(QGs, _dp), _ptrs(vGs, _dp), _ptrs(QAs, _dp),
                                 _ptrs(vAs, _dp), float(gamma), _ptrs(Ps, _dp))
    return Ps


# ----------------------------------------------------------------- stage 4 --
def kl_clip(Ps, Ws, lr, kappa):
    """Returns (scaled P list, nu, s)."""
    Ps = [_f64(P).copy() for P in Ps]
    Ws = [_f64(W) for W in Ws]
    numel = (C.c_int64 * len(Ps))(*[P.size for P in Ps])
    s = C.c_double(0.0)
    nu = lib().orc_kl_clip(len(Ps), _ptrs(Ps, _dp), _ptrs(Ws, _dp), numel, float(lr), float(kappa),
                           C.byref(s))
    return Ps, nu, s.value


# ------------------------------------------------------------------- misc --
def kron(A, B):
    A, B = _f64(A), _f64(B)
    out = np.empty((A.shape[0] * B.shape[0], A.shape[1] * B.shape[1]))
    lib().orc_kron(_d(A), A.shape[0], A.shape[1], _d(B), B.shape[0], B.shape[1], _d(out))
    return out


def kron_solve(A, G, W, gamma):
    A, G, W = _f64(A), _f64(G), _f64(W)
    P = np.empty_like(W)
    info = lib().orc_kron_solve(_d(A), A.shape[0], _d(G), G.shape[0], float(gamma), _d(W), _d(P))
    if info:
        raise np.linalg.LinAlgError("Kronecker system not SPD")
    return P


def assign(dims, layer_of, num_layers, world, policy):
    dims = np.ascontiguousarray(dims, np.int32)
    layer_of = np.ascontiguousarray(layer_of, np.int32)
    owner = np.empty(len(dims), np.int32)
    lib().orc_assign(dims.ctypes.data_as(_ip), layer_of.ctypes.data_as(_ip), len(dims),
                     int(num_layers), int(world), int(policy), owner.ctypes.data_as(_ip))
    return owner


def full_step(layers, acts, gouts, grads, damping, lr, kappa, mode=EIGEN, xi=0.95):
    """One full K-FAC update from a cold state (Alg. 1 steps 1-3 + Eq. 18)."""
    A, G = update_factors(layers, acts, gouts, xi=xi, first=True)
    if mode == INVERSE:
        QA = [damped_inverse(a, damping) for a in A]
        QG = [damped_inverse(g, damping) for g in G]
        vA = vG = None
    else:
        QGA = symeig_batch(A + G)
        QA, QG = QGA[0][:len(A)], QGA[0][len(A):]
        vA, vG = QGA[1][:len(A)], QGA[1][len(A):]
    P = precondition_batch(grads, QG, vG, QA, vA, damping, mode)
    P, nu, s = kl_clip(P, grads, lr, kappa)
    return dict(A=A, G=G, QA=QA, vA=vA, QG=QG, vG=vG, P=P, nu=nu, s=s)

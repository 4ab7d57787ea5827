"""Thin ctypes binding of libkfac.so (include/kfac.h).  Argument marshalling only.

Every function here has the name of the C entry point it wraps and takes torch
CUDA tensors; it passes their data pointers, shapes and leading dimensions
(`tensor.stride(0)`) to the library and launches on the current torch stream.
There is no fallback: if libkfac.so is missing or fails to load, importing this
module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libkfac.so")

KFAC_LINEAR, KFAC_CONV2D = 0, 1
EIGEN, EIGEN_FACTORED, INVERSE = 0, 1, 2
LPT_D3, ROUND_ROBIN_PAPER, LAYERWISE_LPT = 0, 1, 2
EIG_WARM_START = 1


class KfacError(RuntimeError):
    pass


class kfac_layer_t(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "kind", "batch", "c_in", "h_in", "w_in", "c_out", "h_out", "w_out",
        "k_h", "k_w", "stride_h", "stride_w", "pad_h", "pad_w", "bias_col")]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2007_00784_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P, I32P, SZ = C.c_void_p, C.POINTER(C.c_int32), C.c_size_t
    PP = C.POINTER(C.c_void_p)
    L.kfac_layer_dims.argtypes = [C.POINTER(kfac_layer_t), I32P, I32P, C.POINTER(C.c_int64)]
    L.kfac_update_factors_workspace_size.argtypes = [C.POINTER(kfac_layer_t), C.c_int32]
    L.kfac_update_factors_workspace_size.restype = SZ
    L.kfac_update_factors.argtypes = [C.POINTER(kfac_layer_t), C.c_int32, PP, PP, PP, I32P, PP, I32P, PP, PP,
                                      C.c_float, C.c_int32, C.c_float, P, SZ, P]
    L.kfac_unpack_factors.argtypes = [PP, I32P, PP, I32P, C.c_int32, C.c_float, P]
    L.kfac_compute_eigen_workspace_size.argtypes = [I32P, C.c_int32]
    L.kfac_compute_eigen_workspace_size.restype = SZ
    L.kfac_compute_eigen.argtypes = [PP, I32P, I32P, C.c_int32, PP, I32P, PP, P, C.c_uint32, P, SZ, P]
    L.kfac_compute_inverse_workspace_size.argtypes = [I32P, C.c_int32]
    L.kfac_compute_inverse_workspace_size.restype = SZ
    L.kfac_compute_inverse.argtypes = [PP, I32P, I32P, C.c_int32, C.c_float, PP, I32P, P, P, SZ, P]
    L.kfac_precondition_workspace_size.argtypes = [I32P, I32P, C.c_int32, C.c_int32]
    L.kfac_precondition_workspace_size.restype = SZ
    L.kfac_precondition.argtypes = [I32P, I32P, C.c_int32, PP, I32P, PP, I32P, PP, PP, I32P, PP,
                                    C.c_float, C.c_int32, PP, P, SZ, P]
    L.kfac_kl_clip_workspace_size.argtypes = [I32P, I32P, C.c_int32]
    L.kfac_kl_clip_workspace_size.restype = SZ
    L.kfac_kl_clip.argtypes = [PP, PP, I32P, I32P, I32P, C.c_int32, C.c_float, C.c_float, P, P, P, SZ, P]
    L.kfac_assign.argtypes = [I32P, I32P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, I32P]
    L.kfac_status_string.argtypes = [C.c_int]
    L.kfac_status_string.restype = C.c_char_p
    L.kfac_last_error.restype = C.c_char_p
    L.kfac_launch_count.restype = C.c_uint64
    L.kfac_version.restype = C.c_int32
    L.kfac_profile_start.argtypes = [C.c_int32]
    L.kfac_profile_stop.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                    C.POINTER(C.c_double)]
    for f in ("kfac_layer_dims", "kfac_update_factors", "kfac_unpack_factors", "kfac_compute_eigen", "kfac_compute_inverse",
              "kfac_precondition", "kfac_kl_clip", "kfac_assign", "kfac_profile_start", "kfac_profile_stop"):
        getattr(L, f).restype = C.c_int
    return L


lib = _load()

EXPORTED = ("kfac_layer_dims", "kfac_update_factors_workspace_size", "kfac_update_factors", "kfac_unpack_factors",
            "kfac_compute_eigen_workspace_size", "kfac_compute_eigen",
            "kfac_compute_inverse_workspace_size", "kfac_compute_inverse",
            "kfac_precondition_workspace_size", "kfac_precondition",
            "kfac_kl_clip_workspace_size", "kfac_kl_clip", "kfac_assign",
            "kfac_status_string", "kfac_last_error", "kfac_launch_count", "kfac_version",
            "kfac_profile_start", "kfac_profile_stop")


def _check(status: int, fn: str):
    if status != 0:
        raise KfacError(f"{fn}: {lib.kfac_status_string(status).decode()}: {lib.kfac_last_error().decode()}")


def _ptrs(ts: Sequence[Optional[torch.Tensor]]):
    return (C.c_void_p * len(ts))(*[(t.data_ptr() if t is not None else None) for t in ts])


def _i32(vals):
    return (C.c_int32 * len(vals))(*[int(v) for v in vals])


def _ld(t: torch.Tensor) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError("matrices must be 2-D with unit column stride (row-major, padded ld)")
    return t.stride(0)


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class Workspace:
    """Grow-only device scratch buffer handed to the library (caller-owned, per stream)."""

    def __init__(self, device=None):
        self.device = device
        self.buf = None

    def get(self, nbytes: int) -> torch.Tensor:
        nbytes = max(int(nbytes), 256)
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device or "cuda")
        return self.buf


_default_ws = {}


def _ws(ws: Optional[Workspace], key: str) -> Workspace:
    if ws is not None:
        return ws
    dev = torch.cuda.current_device()
    return _default_ws.setdefault((key, dev), Workspace(torch.device("cuda", dev)))


def layer_struct(layer) -> kfac_layer_t:
    t = layer.as_tuple() if hasattr(layer, "as_tuple") else tuple(layer)
    return kfac_layer_t(*[int(v) for v in t])


def kfac_layer_dims(layer):
    da, dg, rows = C.c_int32(), C.c_int32(), C.c_int64()
    _check(lib.kfac_layer_dims(C.byref(layer_struct(layer)), C.byref(da), C.byref(dg), C.byref(rows)),
           "kfac_layer_dims")
    return da.value, dg.value, rows.value


def kfac_update_factors(layers, acts: List[torch.Tensor], gouts: List[torch.Tensor],
                        A: List[torch.Tensor], G: List[torch.Tensor], xi: float, first: bool,
                        out_scale: float = 1.0, ws: Optional[Workspace] = None, stream=None,
                        packed_A: Optional[List[torch.Tensor]] = None, packed_G: Optional[List[torch.Tensor]] = None):
    n = len(layers)
    arr = (kfac_layer_t * n)(*[layer_struct(l) for l in layers])
    need = lib.kfac_update_factors_workspace_size(arr, n)
    buf = _ws(ws, "factors").get(need)
    _check(lib.kfac_update_factors(arr, n, _ptrs(acts), _ptrs(gouts), _ptrs(A), _i32([_ld(a) for a in A]),
                                   _ptrs(G), _i32([_ld(g) for g in G]),
                                   _ptrs(packed_A) if packed_A is not None else None,
                                   _ptrs(packed_G) if packed_G is not None else None,
                                   float(xi), int(bool(first)),
                                   float(out_scale), C.c_void_p(buf.data_ptr()), buf.numel(),
                                   _stream(stream)), "kfac_update_factors")


def kfac_unpack_factors(packed: List[torch.Tensor], F: List[torch.Tensor], scale: float = 1.0, stream=None):
    n = len(F)
    _check(lib.kfac_unpack_factors(_ptrs(packed), _i32([f.shape[0] for f in F]), _ptrs(F),
                                   _i32([_ld(f) for f in F]), n, float(scale), _stream(stream)),
           "kfac_unpack_factors")


def kfac_compute_eigen(F: List[torch.Tensor], Q: List[torch.Tensor], evals: List[torch.Tensor],
                       info: Optional[torch.Tensor] = None, flags: int = 0,
                       ws: Optional[Workspace] = None, stream=None):
    n = len(F)
    dims = _i32([f.shape[0] for f in F])
    need = lib.kfac_compute_eigen_workspace_size(dims, n)
    buf = _ws(ws, "eigen").get(need)
    _check(lib.kfac_compute_eigen(_ptrs(F), dims, _i32([_ld(f) for f in F]), n, _ptrs(Q),
                                  _i32([_ld(q) for q in Q]), _ptrs(evals),
                                  C.c_void_p(info.data_ptr() if info is not None else None), int(flags),
                                  C.c_void_p(buf.data_ptr()), buf.numel(), _stream(stream)),
           "kfac_compute_eigen")


def kfac_compute_inverse(F: List[torch.Tensor], damping: float, Finv: List[torch.Tensor],
                         info: Optional[torch.Tensor] = None, ws: Optional[Workspace] = None, stream=None):
    n = len(F)
    dims = _i32([f.shape[0] for f in F])
    need = lib.kfac_compute_inverse_workspace_size(dims, n)
    buf = _ws(ws, "inverse").get(need)
    _check(lib.kfac_compute_inverse(_ptrs(F), dims, _i32([_ld(f) for f in F]), n, float(damping),
                                    _ptrs(Finv), _i32([_ld(f) for f in Finv]),
                                    C.c_void_p(info.data_ptr() if info is not None else None),
                                    C.c_void_p(buf.data_ptr()), buf.numel(), _stream(stream)),
           "kfac_compute_inverse")


def kfac_precondition(grads: List[torch.Tensor], QG: List[torch.Tensor], vG, QA: List[torch.Tensor], vA,
                      damping: float, mode: int, out: List[torch.Tensor],
                      ws: Optional[Workspace] = None, stream=None):
    n = len(grads)
    dg = _i32([g.shape[0] for g in grads])
    da = _i32([g.shape[1] for g in grads])
    need = lib.kfac_precondition_workspace_size(dg, da, n, int(mode))
    buf = _ws(ws, "precond").get(need)
    vG = vG if vG is not None else [None] * n
    vA = vA if vA is not None else [None] * n
    for g, o in zip(grads, out):
        if _ld(g) != _ld(o):
            raise ValueError("grad and out must share the leading dimension")
    _check(lib.kfac_precondition(dg, da, n, _ptrs(grads), _i32([_ld(g) for g in grads]), _ptrs(QG),
                                 _i32([_ld(q) for q in QG]), _ptrs(vG), _ptrs(QA), _i32([_ld(q) for q in QA]),
                                 _ptrs(vA), float(damping), int(mode), _ptrs(out),
                                 C.c_void_p(buf.data_ptr()), buf.numel(), _stream(stream)),
           "kfac_precondition")


def kfac_kl_clip(precond: List[torch.Tensor], grads: List[torch.Tensor], lr: float, kappa: float,
                 nu_out: Optional[torch.Tensor] = None, s_out: Optional[torch.Tensor] = None,
                 ws: Optional[Workspace] = None, stream=None):
    n = len(precond)
    rows = _i32([p.shape[0] for p in precond])
    cols = _i32([p.shape[1] for p in precond])
    lds = [_ld(p) for p in precond]
    for p, g in zip(precond, grads):
        if _ld(g) != _ld(p):
            raise ValueError("precond and grad must share the leading dimension")
    need = lib.kfac_kl_clip_workspace_size(rows, cols, n)
    buf = _ws(ws, "klclip").get(need)
    _check(lib.kfac_kl_clip(_ptrs(precond), _ptrs(grads), rows, cols, _i32(lds), n, float(lr), float(kappa),
                            C.c_void_p(nu_out.data_ptr() if nu_out is not None else None),
                            C.c_void_p(s_out.data_ptr() if s_out is not None else None),
                            C.c_void_p(buf.data_ptr()), buf.numel(), _stream(stream)), "kfac_kl_clip")


def kfac_assign(dims, layer_of, num_layers: int, world_size: int, policy: int):
    nf = len(dims)
    owner = (C.c_int32 * nf)()
    _check(lib.kfac_assign(_i32(dims), _i32(layer_of), nf, int(num_layers), int(world_size), int(policy),
                           owner), "kfac_assign")
    return [int(o) for o in owner]


def kfac_launch_count() -> int:
    return int(lib.kfac_launch_count())


PROF_TRD_PANEL, PROF_GEMM64, PROF_SYRK_TC, PROF_GEMM_TC = 1, 2, 3, 4


def kfac_profile_start(kernel_class: int):
    _check(lib.kfac_profile_start(int(kernel_class)), "kfac_profile_start")


def kfac_profile_stop():
    """-> (device ms summed over the armed class's launches, launches, algorithmic bytes, flops)."""
    ms, n, by, fl = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
    _check(lib.kfac_profile_stop(C.byref(ms), C.byref(n), C.byref(by), C.byref(fl)), "kfac_profile_stop")
    return ms.value, n.value, by.value, fl.value

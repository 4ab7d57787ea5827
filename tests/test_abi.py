"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/kfac.h
declares, validates arguments before launching anything, and its host-only logic
(kfac_layer_dims, kfac_assign) matches the oracle exactly."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from workloads import shapes


@pytest.fixture(scope="module")
def L():
    from paper_2007_00784_b200.build import build
    build()
    from paper_2007_00784_b200 import _lib
    return _lib


def _declared():
    src = open(os.path.join(ROOT, "include", "kfac.h")).read()
    return sorted(set(re.findall(r"\b(kfac_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = _declared()
    assert len(names) >= 16
    for n in names:
        assert hasattr(L.lib, n), n
    assert set(L.EXPORTED) <= set(names)


def test_layer_dims_match_shapes(L):
    for cfg in ("mlp", "r32", "r50"):
        for l in shapes.layers_for(cfg):
            assert L.kfac_layer_dims(l) == (l.d_a, l.d_g, l.rows)


def test_layer_validation_errors(L):
    bad = shapes.Layer("x", 2, 1, 3, 4, 4, 2, 4, 4, 3, 3, 1, 1, 1, 1, 1)          # kind 2: not linear/conv
    with pytest.raises(L.KfacError, match="INVALID_VALUE"):
        L.kfac_layer_dims(bad)
    bad = shapes.Layer("x", 1, 1, 3, 4, 4, 2, 5, 4, 3, 3, 1, 1, 1, 1, 1)          # h_out inconsistent
    with pytest.raises(L.KfacError, match="SHAPE"):
        L.kfac_layer_dims(bad)


@pytest.mark.parametrize("policy", [0, 1, 2])
def test_assign_matches_oracle(L, orc, policy):
    rng = np.random.default_rng(policy)
    for t in range(30):
        nl = int(rng.integers(1, 40))
        dims = rng.integers(1, 5000, size=2 * nl).astype(np.int32)
        layer_of = np.repeat(np.arange(nl), 2).astype(np.int32)
        world = int(rng.integers(1, 70))
        ref = orc.assign(dims, layer_of, nl, world, policy)
        got = L.kfac_assign(list(dims), list(layer_of), nl, world, policy)
        assert list(ref) == got
    layers = shapes.resnet50()
    dims, lo = shapes.factor_dims(layers)
    for w in (1, 2, 4, 8, 16, 64):
        assert L.kfac_assign(dims, lo, 54, w, policy) == list(orc.assign(dims, lo, 54, w, policy))


def test_call_validation_before_launch(L):
    """Bad arguments are rejected on the host (no device needed, nothing launched)."""
    lib = L.lib
    n0 = L.kfac_launch_count()
    fake = C.c_void_p(0x10000)                      # 16-byte aligned, never dereferenced
    pp = (C.c_void_p * 1)(fake)
    dims = (C.c_int32 * 1)(8)
    ld_bad = (C.c_int32 * 1)(10)                     # not a multiple of 4
    ld_ok = (C.c_int32 * 1)(8)
    ws = C.c_void_p(0x20000)
    st = lib.kfac_compute_eigen(pp, dims, ld_bad, 1, pp, ld_ok, pp, None, 0, ws, 1 << 30, None)
    assert lib.kfac_status_string(st) == b"KFAC_ERR_ALIGNMENT"
    st = lib.kfac_compute_eigen(pp, dims, ld_ok, 0, pp, ld_ok, pp, None, 0, ws, 1 << 30, None)
    assert lib.kfac_status_string(st) == b"KFAC_ERR_INVALID_VALUE"
    st = lib.kfac_compute_eigen(pp, dims, ld_ok, 1, pp, ld_ok, pp, None, 0, ws, 16, None)
    assert lib.kfac_status_string(st) == b"KFAC_ERR_WORKSPACE"
    st = lib.kfac_compute_eigen(pp, dims, ld_ok, 1, pp, ld_ok, pp, None, 0x80, ws, 1 << 30, None)
    assert lib.kfac_status_string(st) == b"KFAC_ERR_INVALID_VALUE"
    mis = (C.c_void_p * 1)(C.c_void_p(0x10004))      # misaligned base
    st = lib.kfac_compute_eigen(mis, dims, ld_ok, 1, pp, ld_ok, pp, None, 0, ws, 1 << 30, None)
    assert lib.kfac_status_string(st) == b"KFAC_ERR_ALIGNMENT"
    r = (C.c_int32 * 1)(4)
    st = lib.kfac_kl_clip(pp, pp, r, r, ld_ok, 1, C.c_float(0.0), C.c_float(1e-3), None, None, ws,
                          1 << 20, None)
    assert lib.kfac_status_string(st) == b"KFAC_ERR_INVALID_VALUE"             # lr must be > 0
    dg = (C.c_int32 * 1)(4)
    st = lib.kfac_precondition(dg, dims, 1, pp, ld_ok, pp, ld_ok, pp, pp, ld_ok, pp, C.c_float(1e-3), 7,
                               pp, ws, 1 << 30, None)
    assert lib.kfac_status_string(st) == b"KFAC_ERR_INVALID_VALUE"             # unknown mode
    assert L.kfac_launch_count() == n0
    assert lib.kfac_last_error()


def test_profile_hook_host_side(L):
    """Instrumentation entry points: argument validation and an empty (no launch) window."""
    assert L.lib.kfac_profile_start(0) != 0
    assert L.lib.kfac_profile_start(99) != 0
    L.kfac_profile_start(L.PROF_TRD_PANEL)
    ms, n, by, fl = L.kfac_profile_stop()
    assert (ms, n, by, fl) == (0.0, 0, 0.0, 0.0)

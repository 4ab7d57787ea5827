"""Factor -> worker assignment (Alg. 1) in the oracle."""
import itertools

import numpy as np
import pytest

from conftest import golden, read_sections
from workloads import shapes


def _loads(dims, owner, world, power):
    out = np.zeros(world)
    for d, o in zip(dims, owner):
        out[o] += float(d) ** power
    return out


def test_round_robin_reproduces_paper_parameter_counts(orc):
    """per-worker factor parameter counts for ResNet-50 at 16 and 64 GPUs,
    reproduced exactly (3 significant digits) by the paper-rule round robin (R16)."""
    layers = shapes.resnet50()
    dims, layer_of = shapes.factor_dims(layers)
    rows = [r for r in open(golden("resnet50_assignment.txt")) if r.strip() and not r.startswith("#")]
    for row in rows:
        world, pmin, pmax = row.split()
        world = int(world)
        owner = orc.assign(dims, layer_of, len(layers), world, orc.ROUND_ROBIN_PAPER)
        loads = _loads(dims, owner, world, 2)
        assert float(f"{loads.min():.2e}") == float(pmin)
        assert float(f"{loads.max():.2e}") == float(pmax)


def test_table6_trend_under_round_robin(orc):
    """Table VI, qualitative: from 16 to 64 workers the fastest worker's
    cost drops far more than the slowest worker's (d^3 cost model)."""
    layers = shapes.resnet50()
    dims, layer_of = shapes.factor_dims(layers)
    l16 = _loads(dims, orc.assign(dims, layer_of, 54, 16, orc.ROUND_ROBIN_PAPER), 16, 3)
    l64 = _loads(dims, orc.assign(dims, layer_of, 54, 64, orc.ROUND_ROBIN_PAPER), 64, 3)
    slow = l16.max() / l64.max()
    fast = l16[l16 > 0].min() / l64[l64 > 0].min()
    assert slow < 2.0 < fast


def test_lpt_not_worse_than_round_robin(orc):
    """SPEC acceptance #9: size-balanced placement's max-worker cost <= round
    robin's on >= 95 of 100 heavy-tailed random size sets."""
    rng = np.random.default_rng(0)
    wins = 0
    for t in range(100):
        nl = int(rng.integers(3, 30))
        dims = (rng.pareto(1.2, size=2 * nl) * 64 + 8).astype(np.int32)
        layer_of = np.repeat(np.arange(nl), 2).astype(np.int32)
        world = int(rng.integers(2, 9))
        lpt = _loads(dims, orc.assign(dims, layer_of, nl, world, orc.LPT_D3), world, 3).max()
        rr = _loads(dims, orc.assign(dims, layer_of, nl, world, orc.ROUND_ROBIN_PAPER), world, 3).max()
        wins += lpt <= rr * (1 + 1e-12)
    assert wins >= 95


def test_lpt_graham_bound_bruteforce(orc):
    """Graham's LPT bound: makespan <= (4/3 - 1/(3W)) OPT, OPT by brute force."""
    rng = np.random.default_rng(1)
    for t in range(40):
        nf = int(rng.integers(2, 8))
        world = int(rng.integers(2, 4))
        dims = rng.integers(1, 20, size=nf).astype(np.int32)
        layer_of = np.arange(nf, dtype=np.int32)
        lpt = _loads(dims, orc.assign(dims, layer_of, nf, world, orc.LPT_D3), world, 3).max()
        opt = min(_loads(dims, ow, world, 3).max() for ow in itertools.product(range(world), repeat=nf))
        assert lpt <= (4 / 3 - 1 / (3 * world)) * opt + 1e-9


def test_lpt_examples_and_balance(orc):
    """equal sizes -> balanced counts; {8,1,...,1}, W=2 -> the 8 alone."""
    dims = np.full(12, 5, np.int32)
    owner = orc.assign(dims, np.arange(12, dtype=np.int32), 12, 4, orc.LPT_D3)
    assert sorted(np.bincount(owner, minlength=4)) == [3, 3, 3, 3]
    dims = np.array([8] + [1] * 7, np.int32)
    owner = orc.assign(dims, np.arange(8, dtype=np.int32), 8, 2, orc.LPT_D3)
    assert owner[0] != owner[1] and len(set(owner[1:])) == 1


def test_layerwise_keeps_layers_together_and_rr_granularity(orc):
    """K-FAC-lw: both factors of a layer on one worker.  Paper rule: with W > L
    every worker gets a factor (the 'double the worker utilization' claim)."""
    layers = shapes.resnet32()
    dims, layer_of = shapes.factor_dims(layers)
    owner = orc.assign(dims, layer_of, len(layers), 8, orc.LAYERWISE_LPT)
    for i in range(len(layers)):
        assert owner[2 * i] == owner[2 * i + 1]
    for L in (2, 5):
        for W in range(L + 1, 2 * L + 1):
            dims = np.ones(2 * L, np.int32)
            owner = orc.assign(dims, np.repeat(np.arange(L), 2).astype(np.int32), L, W,
                               orc.ROUND_ROBIN_PAPER)
            assert set(owner) == set(range(W))

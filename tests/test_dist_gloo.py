"""Multi-process (world_size 2, gloo, CPU) tests of the distributed orchestration:
the same assignment on every rank, the owner-major buffer layout that lets the eigenbasis
(K-FAC-opt) and preconditioned-gradient (K-FAC-lw) exchanges run as one broadcast per owner
of exactly its bytes, the packed-triangle factor allreduce in layer buckets, and the factor average through allreduce-SUM of out_scale = 1/W factors
(Alg. 1).  The CUDA kernels are not exercised here."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from workloads import shapes


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, exchange, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2007_00784_b200.preconditioner import KFACPreconditioner, exchange_from_owners
        layers = shapes.layers_for(cfg)
        pc = KFACPreconditioner(layers, device="cpu", exchange=exchange)
        # 1) identical assignment everywhere
        owners = [None] * world
        dist.all_gather_object(owners, pc.owner)
        assert all(o == owners[0] for o in owners)
        # 2) factor allreduce: each rank holds (its factor) * 1/W; SUM gives the average
        vals = torch.arange(pc.factor_flat.numel(), dtype=torch.float32) % 97
        pc.factor_flat.copy_((vals + 1000 * rank) / world)
        dist.all_reduce(pc.factor_flat, op=dist.ReduceOp.SUM)
        expect = (vals * world + 1000 * sum(range(world))) / world
        assert torch.allclose(pc.factor_flat, expect)
        # 2b) packed factor allreduce: the upper triangles are half the full-matrix bytes, the layer
        # buckets tile all layers in order, and SUM of 1/W-scaled packed buffers is their average
        full = sum(d * ((d + 3) // 4 * 4) for d in pc.dims)
        packed = sum(d * (d + 1) // 2 for d in pc.dims)
        assert packed <= 0.5 * full + sum(pc.dims)
        bks = pc.buckets()
        assert bks[0][0] == 0 and bks[-1][1] == len(layers) and all(a[1] == b[0] for a, b in zip(bks, bks[1:]))
        pv = torch.arange(pc.packed_flat.numel(), dtype=torch.float32) % 89
        for b0, b1 in bks:
            lo = pc.packed_seg[2 * b0][0]
            hi = pc.packed_seg[2 * b1 - 1][0] + pc.packed_seg[2 * b1 - 1][1]
            seg = pc.packed_flat[lo:hi]
            seg.copy_((pv[lo:hi] + 10 * rank) / world)
            dist.all_reduce(seg, op=dist.ReduceOp.SUM)
            assert torch.allclose(seg, pv[lo:hi] + 10 * sum(range(world)) / world)
        # 3) eigenbasis exchange (K-FAC-opt): owners write their factors, one broadcast per owner
        for f in pc.owned:
            pc.Q[f].fill_(float(f + 1))
            pc.v[f].fill_(float(-(f + 1)))
        exchange_from_owners(pc.q_flat, pc.q_off, pc.q_size)
        exchange_from_owners(pc.v_flat, pc.v_off, pc.v_size)
        for f in range(len(pc.dims)):
            assert torch.all(pc.Q[f] == f + 1) and torch.all(pc.v[f] == -(f + 1))
        # 4) preconditioned-gradient exchange (K-FAC-lw): layer owners write P
        for i in pc.owned_layers:
            pc.P[i].fill_(float(i + 7))
        exchange_from_owners(pc.p_flat, pc.p_off, pc.p_size)
        for i in range(len(layers)):
            assert torch.all(pc.P[i] == i + 7)
        if exchange == "allgather-grad":
            for i in range(len(layers)):
                assert pc.owner[2 * i] == pc.owner[2 * i + 1]
        # 5) reduce-to-owner (factor_comm="reduce-owner"): the packed buffer is owner-major, each
        # owner's factors lie inside its contiguous slice, the slices tile the buffer, and one
        # reduce per owner leaves the SUM of every rank's copy in the owner's slice
        from paper_2007_00784_b200.preconditioner import reduce_to_owners
        pr = KFACPreconditioner(layers, device="cpu", exchange=exchange, factor_comm="reduce-owner")
        assert pr.owner == pc.owner
        assert pr.pk_off[0] == 0 and all(pr.pk_off[r] + pr.pk_size[r] == pr.pk_off[r + 1] for r in range(world - 1))
        for f, (o, n) in enumerate(pr.packed_seg):
            r = pr.owner[f]
            assert pr.pk_off[r] <= o and o + n <= pr.pk_off[r] + pr.pk_size[r]
        assert sum(pr.pk_size) <= pr.packed_flat.numel()
        pv = torch.arange(pr.packed_flat.numel(), dtype=torch.float32) % 89
        pr.packed_flat.copy_(pv + 10 * rank)
        reduce_to_owners(pr.packed_flat, pr.pk_off, pr.pk_size)
        lo, hi = pr.pk_off[rank], pr.pk_off[rank] + pr.pk_size[rank]
        assert torch.equal(pr.packed_flat[lo:hi], world * pv[lo:hi] + 10 * sum(range(world)))
        # the averaged copies are private to the owner (shape = the owned factors only)
        assert sum(pr.F_src[f].numel() for f in pr.owned) <= pr.fown_flat.numel()
        assert all(pr.F_src[f] is None for f in range(len(pr.dims)) if pr.owner[f] != rank)
        q.put((rank, "ok", len(pc.owned)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,exchange", [("r32", "bcast-eig"), ("r32", "allgather-grad"), ("mlp", "bcast-eig")])
def test_two_rank_exchanges(cfg, exchange):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, exchange, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res
    assert sum(r[2] for r in res) == 2 * len(shapes.layers_for(cfg))     # every factor owned once


def test_lpt_balances_r50_eigen_cost():
    """LPT on d^3 at W = 2/4/8: the makespan is within Graham's bound of the ideal and
    matches the cap set by the largest factor (2.00 / 4.00 / 4.63)."""
    from paper_2007_00784_b200 import _lib
    layers = shapes.resnet50()
    dims, lo = shapes.factor_dims(layers)
    total = sum(d ** 3 for d in dims)
    speed = {}
    for w in (2, 4, 8):
        owner = _lib.kfac_assign(dims, lo, len(layers), w, _lib.LPT_D3)
        load = np.zeros(w)
        for d, o in zip(dims, owner):
            load[o] += d ** 3
        speed[w] = total / load.max()
    assert speed[2] > 1.99 and speed[4] > 3.95 and abs(speed[8] - total / 4609 ** 3) < 1e-6 * speed[8]

"""Two ranks on one GPU (gloo over CUDA tensors), running the real kernels.

Both processes use cuda:0 (this build has one GPU; NCCL refuses two ranks per device, so the
collectives go through gloo, which accepts CUDA tensors).  Each rank draws its own shard of a
ResNet-32 batch (seeded by rank) and the caller-side gradient allreduce is modelled by handing
every rank the global-batch weight gradient.  Checks:
  * W = 2 shards == the oracle on the concatenated global batch (Alg. 1: the
    average of per-rank running factors equals the factors of the global batch, equal shards):
    factors relF <= 1e-4, P relF <= 1e-3, nu to 1e-4;
  * K-FAC-opt (eigenbasis all-gather) and K-FAC-lw (preconditioned-gradient all-gather,
    P:618) give the same P (different owners -> different launch groupings, so to 1e-5).
"""
import os
import socket

import numpy as np
import pytest
import torch

from conftest import relF
from workloads import shapes
from workloads.gen import layer_inputs, weight_grad

pytestmark = pytest.mark.gpu

BATCH_PER_RANK = 4
SEED = 21


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _global_inputs(world):
    layers_r = shapes.resnet32(batch=BATCH_PER_RANK)
    shards = [layer_inputs(layers_r, seed=SEED, rank=r, with_grad=False) for r in range(world)]
    layers_g = shapes.resnet32(batch=BATCH_PER_RANK * world)
    acts = [np.concatenate([s[0][i] for s in shards], 0) for i in range(len(layers_g))]
    gouts = [np.concatenate([s[1][i] for s in shards], 0) for i in range(len(layers_g))]
    grads = [weight_grad(l, a, g) for l, a, g in zip(layers_g, acts, gouts)]
    return layers_r, layers_g, shards, acts, gouts, grads


def _worker(rank, world, port, exchange, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2007_00784_b200.preconditioner import KFACPreconditioner
        layers_r, _, shards, _, _, grads = _global_inputs(world)
        hp = shapes.HPARAMS["r32"]
        pc = KFACPreconditioner(layers_r, device="cuda:0", damping=hp["damping"], xi=hp["xi"],
                                kappa=hp["kappa"], lr=hp["lr"], exchange=exchange)
        g = KFACPreconditioner.grad_buffer(layers_r, "cuda:0")
        for t, w in zip(g, grads):
            t.copy_(torch.from_numpy(w))
        acts, gouts = shards[rank][0], shards[rank][1]
        P = pc.step([torch.from_numpy(a).cuda() for a in acts], [torch.from_numpy(x).cuda() for x in gouts],
                    g, first=True)
        torch.cuda.synchronize()
        assert (pc.info.cpu().numpy() == 0).all()
        np.savez(os.path.join(out_dir, f"{exchange}_{rank}.npz"),
                 nu=pc.nu.item(), owned=len(pc.owned),
                 **{f"P{i}": p.double().cpu().numpy() for i, p in enumerate(P)},
                 **{f"F{i}": f.double().cpu().numpy() for i, f in enumerate(pc.F)})
    finally:
        dist.destroy_process_group()


def _run(exchange, out_dir, world=2):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, exchange, out_dir)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    return [dict(np.load(os.path.join(out_dir, f"{exchange}_{r}.npz"))) for r in range(world)]


def test_two_ranks_one_gpu_match_global_batch_oracle(orc, tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2007_00784_b200.build import build
    build()
    world = 2
    res_opt = _run("bcast-eig", str(tmp_path), world)
    res_lw = _run("allgather-grad", str(tmp_path), world)
    _, layers_g, _, acts, gouts, grads = _global_inputs(world)
    hp = shapes.HPARAMS["r32"]
    ref = orc.full_step(layers_g, acts, gouts, grads, hp["damping"], hp["lr"], hp["kappa"])
    nl = len(layers_g)
    assert sum(int(r["owned"]) for r in res_opt) == 2 * nl
    ref_F = [x for i in range(nl) for x in (ref["A"][i], ref["G"][i])]
    for r in res_opt + res_lw:
        assert max(relF(r[f"F{f}"], ref_F[f]) for f in range(2 * nl)) <= 1e-4
        errs = [relF(r[f"P{i}"], ref["P"][i]) for i in range(nl)]
        assert max(errs) <= 1e-3, errs
        assert abs(float(r["nu"]) - ref["nu"]) <= 1e-4 * ref["nu"]
    # replicas agree bitwise after the exchange; opt == lw to fp32-chain rounding
    for res in (res_opt, res_lw):
        for i in range(nl):
            assert np.array_equal(res[0][f"P{i}"], res[1][f"P{i}"])
    for i in range(nl):
        assert relF(res_lw[0][f"P{i}"], res_opt[0][f"P{i}"]) <= 1e-5


# --------------------------------------------------------- reduce-to-owner --
SEEDS_RO = (SEED, SEED + 7)       # two update steps with different batches


def _global_inputs_seed(world, seed):
    layers_r = shapes.resnet32(batch=BATCH_PER_RANK)
    shards = [layer_inputs(layers_r, seed=seed, rank=r, with_grad=False) for r in range(world)]
    layers_g = shapes.resnet32(batch=BATCH_PER_RANK * world)
    acts = [np.concatenate([s[0][i] for s in shards], 0) for i in range(len(layers_g))]
    gouts = [np.concatenate([s[1][i] for s in shards], 0) for i in range(len(layers_g))]
    grads = [weight_grad(l, a, g) for l, a, g in zip(layers_g, acts, gouts)]
    return layers_r, layers_g, shards, acts, gouts, grads


def _worker_ro(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2007_00784_b200 import preconditioner as pre
        from paper_2007_00784_b200.preconditioner import KFACPreconditioner
        real_reduce = pre.reduce_to_owners

        def staged_reduce(flat, offs, sizes, group=None):
            # gloo reduces host memory only: stage the (CUDA) buffer through the host and run the
            # real reduce_to_owners on it (NCCL reduces the device buffer in place)
            h = flat.cpu()
            real_reduce(h, offs, sizes, group)
            flat.copy_(h)
        pre.reduce_to_owners = staged_reduce
        hp = shapes.HPARAMS["r32"]
        layers_r = shapes.resnet32(batch=BATCH_PER_RANK)
        pc = KFACPreconditioner(layers_r, device="cuda:0", damping=hp["damping"], xi=hp["xi"],
                                kappa=hp["kappa"], lr=hp["lr"], factor_comm="reduce-owner")
        g = KFACPreconditioner.grad_buffer(layers_r, "cuda:0")
        for k, seed in enumerate(SEEDS_RO):
            _, _, shards, _, _, grads = _global_inputs_seed(world, seed)
            for t, w in zip(g, grads):
                t.copy_(torch.from_numpy(w))
            acts, gouts = shards[rank][0], shards[rank][1]
            # step 0 updates the factors without a refresh (local running averages only, no factor
            # traffic); step 1 refreshes: reduce to owners, eigen on the averaged copies, exchange
            if k == 0:
                pc.update_factors([torch.from_numpy(a).cuda() for a in acts],
                                  [torch.from_numpy(x).cuda() for x in gouts], first=True, refresh=False)
                continue
            P = pc.step([torch.from_numpy(a).cuda() for a in acts], [torch.from_numpy(x).cuda() for x in gouts],
                        g, first=False)
        torch.cuda.synchronize()
        assert (pc.info.cpu().numpy() == 0).all()
        np.savez(os.path.join(out_dir, f"ro_{rank}.npz"), nu=pc.nu.item(),
                 owned=np.array(pc.owned, dtype=np.int64),
                 **{f"P{i}": p.double().cpu().numpy() for i, p in enumerate(P)},
                 **{f"Fown{f}": pc.F_src[f].double().cpu().numpy() for f in pc.owned},
                 **{f"Floc{f}": x.double().cpu().numpy() for f, x in enumerate(pc.F)})
    finally:
        dist.destroy_process_group()


def test_two_ranks_reduce_to_owner_two_steps(orc, tmp_path):
    """factor_comm='reduce-owner': local running averages (no factor exchange on the step without
    an eigen refresh), reduce-SUM to the owners + unpack with scale 1/W at the refresh.  After two
    steps the owners' averaged factors equal the oracle's running average of the two GLOBAL batches
    (Eqs. 16-17 linear; factors relF <= 1e-4), P matches the oracle (relF <= 1e-3), the
    replicas' P agree bitwise, and each rank's local running average is NOT the global one."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    from paper_2007_00784_b200.build import build
    build()
    world = 2
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker_ro, args=(r, world, port, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = [dict(np.load(os.path.join(str(tmp_path), f"ro_{r}.npz"))) for r in range(world)]
    hp = shapes.HPARAMS["r32"]
    A = G = None
    for k, seed in enumerate(SEEDS_RO):
        _, layers_g, _, acts, gouts, grads = _global_inputs_seed(world, seed)
        A, G = orc.update_factors(layers_g, acts, gouts, A=A, G=G, xi=hp["xi"], first=(k == 0))
    nl = len(layers_g)
    QGA = orc.symeig_batch(A + G)
    QA, QG, vA, vG = QGA[0][:nl], QGA[0][nl:], QGA[1][:nl], QGA[1][nl:]
    Pr = orc.precondition_batch(grads, QG, vG, QA, vA, hp["damping"])
    Pr, nu, _ = orc.kl_clip(Pr, grads, hp["lr"], hp["kappa"])
    ref_F = [x for i in range(nl) for x in (A[i], G[i])]
    owned = sorted(int(f) for r in res for f in r["owned"])
    assert owned == list(range(2 * nl))
    for r in res:
        for f in r["owned"]:
            assert relF(r[f"Fown{int(f)}"], ref_F[int(f)]) <= 1e-4
        errs = [relF(r[f"P{i}"], Pr[i]) for i in range(nl)]
        assert max(errs) <= 1e-3, errs
        assert abs(float(r["nu"]) - nu) <= 1e-4 * nu
    for i in range(nl):
        assert np.array_equal(res[0][f"P{i}"], res[1][f"P{i}"])
    assert max(relF(res[0][f"Floc{f}"], ref_F[f]) for f in range(2 * nl)) > 1e-3

"""KFACPreconditioner: device buffers + Alg. 1 orchestration over the C-ABI calls.

One process per GPU.  Every arithmetic step runs in libkfac's CUDA kernels
(`_lib`); this module owns the buffers (torch CUDA tensors), decides which
calls to make, and issues the collectives through torch.distributed:

  step 1  kfac_update_factors (local mini-batch; out_scale = 1/W fused into the kernel), the
          factors' packed upper triangles (half the bytes of the full matrices) all-reduced with
          SUM in buckets of layers on a communication stream, each bucket's allreduce overlapping
          the next bucket's factor kernels, then kfac_unpack_factors -- Alg. 1 P:343-345, P:387,
          P:426-428 (asynchronous, batched communication).
          factor_comm="reduce-owner" (K-FAC-opt, SURVEY 8(e) "reduce-to-owner"): each rank keeps
          its LOCAL running average (Eqs. 16-17 are linear, so the mean of the W local running
          averages is the running average of the averaged batches); only when an eigen refresh
          follows are the packed triangles reduced (SUM) to each factor's owner -- one reduce per
          owner over its contiguous owner-major slice, (W-1)/W of the buffer per rank instead of the
          allreduce's 2(W-1)/W, and no factor traffic at all on iterations without a refresh
           -- and the owner unpacks them with scale 1/W into its own averaged copy.
  step 2  kfac_assign (host, identical on all ranks) -> kfac_compute_eigen on the
          owned factors -> exchange:
            K-FAC-opt ("bcast-eig"): every owner broadcasts its contiguous, owner-major slice
              of eigenbases (exactly its bytes, no padding to the largest slice);
            K-FAC-lw ("allgather-grad"): layer owners keep their
              eigenbases and the preconditioned gradients are all-gathered.
  step 3  kfac_precondition (Eqs. 13-15) and kfac_kl_clip (Eq. 18).

Buffers are allocated once, in the layout the collectives need, so no copy
kernel is issued on the path.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import torch
import torch.distributed as dist

from . import _lib


def _ld(d: int) -> int:
    return (d + 3) // 4 * 4


def _aligned(n: int) -> int:          # keep every matrix 256-byte aligned inside flat buffers
    return (n + 63) // 64 * 64


@dataclass
class Segment:
    offset: int
    rows: int
    cols: int
    ld: int

    @property
    def numel(self):
        return _aligned(self.rows * self.ld)


def _views(flat: torch.Tensor, segs: List[Segment]) -> List[torch.Tensor]:
    return [flat[s.offset:s.offset + s.rows * s.ld].view(s.rows, s.ld)[:, :s.cols] for s in segs]


class KFACPreconditioner:
    def __init__(self, layers, device=None, damping: float = 1e-3, xi: float = 0.95,
                 kappa: float = 1e-3, lr: float = 0.1, variant: str = "eigen",
                 exchange: str = "bcast-eig", assign_policy: int = _lib.LPT_D3,
                 process_group=None, factor_comm: str = "allreduce"):
        self.layers = list(layers)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.damping, self.xi, self.kappa, self.lr = damping, xi, kappa, lr
        assert variant in ("eigen", "factored", "inverse")
        assert exchange in ("bcast-eig", "allgather-grad")
        assert factor_comm in ("allreduce", "reduce-owner")
        self.variant, self.exchange, self.factor_comm = variant, exchange, factor_comm
        self.pg = process_group
        self.world = dist.get_world_size(process_group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(process_group) if dist.is_initialized() else 0
        L = len(self.layers)
        self.d_a = [l.d_a for l in self.layers]
        self.d_g = [l.d_g for l in self.layers]
        self.dims = [d for l in self.layers for d in (l.d_a, l.d_g)]       # [A0, G0, A1, G1, ...]
        self.layer_of = [i for i in range(L) for _ in range(2)]
        policy = _lib.LAYERWISE_LPT if exchange == "allgather-grad" else assign_policy
        self.owner = _lib.kfac_assign(self.dims, self.layer_of, L, self.world, policy)
        self.layer_owner = [self.owner[2 * i] for i in range(L)]

        f32 = dict(dtype=torch.float32, device=self.device)
        # factors: flat, factor order, all-reduced as one message
        off, self.fseg = 0, []
        for d in self.dims:
            s = Segment(off, d, d, _ld(d))
            self.fseg.append(s)
            off += s.numel
        self.factor_flat = torch.zeros(off, **f32)
        self.F = _views(self.factor_flat, self.fseg)
        self.A = self.F[0::2]
        self.G = self.F[1::2]
        per_rank = [[f for f in range(len(self.dims)) if self.owner[f] == r] for r in range(self.world)]
        self.reduce_owner = self.world > 1 and factor_comm == "reduce-owner"
        # packed upper triangles of the factors (the collective's buffer, W > 1): factor order for the
        # allreduce (layer buckets), owner-major for the reduce to owners (one contiguous slice each)
        order = [f for fs in per_rank for f in fs] if self.reduce_owner else range(len(self.dims))
        self.packed_seg, off = [None] * len(self.dims), 0
        self.pk_off, self.pk_size = [0] * self.world, [0] * self.world
        for f in order:
            d = self.dims[f]
            self.packed_seg[f] = (off, d * (d + 1) // 2)
            if self.reduce_owner:
                self.pk_size[self.owner[f]] += _aligned(d * (d + 1) // 2)
            off += _aligned(d * (d + 1) // 2)
        self.pk_off = [sum(self.pk_size[:r]) for r in range(self.world)]
        self.packed_flat = torch.zeros(off if self.world > 1 else 64, **f32)
        self.packed = [self.packed_flat[o:o + n] for o, n in self.packed_seg] if self.world > 1 else None
        self.bucket_bytes = 64 << 20
        self.comm_stream = torch.cuda.Stream(self.device) if (self.world > 1 and self.device.type == "cuda") else None
        # eigenbases / inverses: owner-major, each rank's factors contiguous; slices have their real
        # sizes (the exchange broadcasts exactly each owner's bytes)
        self.q_size = [sum(_aligned(self.dims[f] * _ld(self.dims[f])) for f in fs) for fs in per_rank]
        self.v_size = [sum(_aligned(self.dims[f]) for f in fs) for fs in per_rank]
        self.q_off = [sum(self.q_size[:r]) for r in range(self.world)]
        self.v_off = [sum(self.v_size[:r]) for r in range(self.world)]
        self.q_flat = torch.zeros(max(64, sum(self.q_size)), **f32)
        self.v_flat = torch.zeros(max(64, sum(self.v_size)), **f32)
        self.qseg, self.vseg = [None] * len(self.dims), [None] * len(self.dims)
        for r, fs in enumerate(per_rank):
            qo, vo = self.q_off[r], self.v_off[r]
            for f in fs:
                d = self.dims[f]
                self.qseg[f] = Segment(qo, d, d, _ld(d))
                qo += self.qseg[f].numel
                self.vseg[f] = Segment(vo, 1, d, _aligned(d))
                vo += _aligned(d)
        self.Q = _views(self.q_flat, self.qseg)
        self.v = [self.v_flat[s.offset:s.offset + s.cols] for s in self.vseg]
        self.owned = per_rank[self.rank]
        # reduce-owner: the averaged copies of the owned factors (the local running averages in F
        # stay untouched, so the linearity argument above holds at every refresh)
        self.F_src = self.F
        if self.reduce_owner:
            segs, o = {}, 0
            for f in self.owned:
                segs[f] = Segment(o, self.dims[f], self.dims[f], _ld(self.dims[f]))
                o += segs[f].numel
            self.fown_flat = torch.zeros(max(64, o), **f32)
            self.F_src = [None] * len(self.dims)
            for f, v in zip(self.owned, _views(self.fown_flat, [segs[f] for f in self.owned])):
                self.F_src[f] = v
        self.reduced = False
        self.info = torch.zeros(max(1, len(self.owned)), dtype=torch.int32, device=self.device)
        # preconditioned gradients: owner-major by layer (K-FAC-lw all-gathers them in place)
        per_rank_l = [[i for i in range(L) if self.layer_owner[i] == r] for r in range(self.world)]
        self.p_size = [sum(_aligned(self.d_g[i] * _ld(self.d_a[i])) for i in ls) for ls in per_rank_l]
        self.p_off = [sum(self.p_size[:r]) for r in range(self.world)]
        self.p_flat = torch.zeros(max(64, sum(self.p_size)), **f32)
        self.pseg = [None] * L
        for r, ls in enumerate(per_rank_l):
            o = self.p_off[r]
            for i in ls:
                self.pseg[i] = Segment(o, self.d_g[i], self.d_a[i], _ld(self.d_a[i]))
                o += self.pseg[i].numel
        self.P = _views(self.p_flat, self.pseg)
        self.owned_layers = per_rank_l[self.rank]
        self.nu = torch.ones(1, **f32)
        self.s = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.ws = {k: _lib.Workspace(self.device) for k in ("factors", "eigen", "precond", "klclip")}
        self.have_eigen = False

    # ------------------------------------------------------------ helpers --
    @staticmethod
    def grad_buffer(layers, device=None, return_flat=False):
        """Padded (d_G x ld) gradient views of one flat buffer, in the layout kfac_precondition
        expects (the flat buffer is what a data-parallel gradient allreduce would reduce)."""
        segs, off = [], 0
        for l in layers:
            s = Segment(off, l.d_g, l.d_a, _ld(l.d_a))
            segs.append(s)
            off += s.numel
        flat = torch.zeros(off, dtype=torch.float32, device=device)
        views = _views(flat, segs)
        return (views, flat) if return_flat else views

    # -------------------------------------------------------------- steps --
    def buckets(self):
        """Contiguous layer ranges whose packed factors hold about bucket_bytes each."""
        out, start, acc = [], 0, 0
        for i in range(len(self.layers)):
            acc += 4 * sum(self.packed_seg[2 * i + k][1] for k in (0, 1))
            if acc >= self.bucket_bytes or i == len(self.layers) - 1:
                out.append((start, i + 1))
                start, acc = i + 1, 0
        return out

    def update_factors(self, acts, gouts, first: bool, refresh: bool = True):
        """Alg. 1 step 1: local factors + running average, then the factor allreduce.

        factor_comm="reduce-owner": the local running averages only; when `refresh` (an eigen
        decomposition follows) their packed triangles are reduced to the owners (reduce_to_owners).

        W > 1: the factors' packed upper triangles are all-reduced (SUM of the out_scale = 1/W
        factors = their average) bucket by bucket; with NCCL each bucket's allreduce runs on the
        communication stream as soon as its factor kernels are done, overlapping the next bucket's
        kernels.  Then both triangles are restored from the reduced packed buffer."""
        if self.world == 1:
            _lib.kfac_update_factors(self.layers, acts, gouts, self.A, self.G, self.xi, first,
                                     1.0, ws=self.ws["factors"])
            return
        if self.reduce_owner:
            pk = dict(packed_A=self.packed[0::2], packed_G=self.packed[1::2]) if refresh else {}
            _lib.kfac_update_factors(self.layers, acts, gouts, self.A, self.G, self.xi, first, 1.0,
                                     ws=self.ws["factors"], **pk)
            if refresh:
                compute = torch.cuda.current_stream(self.device) if self.comm_stream is not None else None
                if compute is not None:
                    self.comm_stream.wait_stream(compute)
                    with torch.cuda.stream(self.comm_stream):
                        reduce_to_owners(self.packed_flat, self.pk_off, self.pk_size, self.pg)
                    compute.wait_stream(self.comm_stream)
                else:
                    reduce_to_owners(self.packed_flat, self.pk_off, self.pk_size, self.pg)
                if self.owned:
                    _lib.kfac_unpack_factors([self.packed[f] for f in self.owned],
                                             [self.F_src[f] for f in self.owned], 1.0 / self.world)
                self.reduced = True
            return
        compute = torch.cuda.current_stream(self.device) if self.comm_stream is not None else None
        works = []
        for b0, b1 in self.buckets():
            _lib.kfac_update_factors(self.layers[b0:b1], acts[b0:b1], gouts[b0:b1], self.A[b0:b1], self.G[b0:b1],
                                     self.xi, first, 1.0 / self.world, ws=self.ws["factors"],
                                     packed_A=self.packed[2 * b0:2 * b1:2], packed_G=self.packed[2 * b0 + 1:2 * b1:2])
            lo = self.packed_seg[2 * b0][0]
            hi = self.packed_seg[2 * b1 - 1][0] + self.packed_seg[2 * b1 - 1][1]
            if self.comm_stream is not None:
                self.comm_stream.wait_stream(compute)
                with torch.cuda.stream(self.comm_stream):
                    works.append(dist.all_reduce(self.packed_flat[lo:hi], op=dist.ReduceOp.SUM, group=self.pg,
                                                 async_op=True))
            else:
                dist.all_reduce(self.packed_flat[lo:hi], op=dist.ReduceOp.SUM, group=self.pg)
        for w in works:
            w.wait()                                   # the compute stream waits for the collectives
        if self.comm_stream is not None:
            compute.wait_stream(self.comm_stream)
        _lib.kfac_unpack_factors(self.packed, self.F)

    def compute_eigen(self, warm: bool = False, check: Optional[bool] = None):
        """Alg. 1 step 2 on the owned factors, then the exchange of the results.

        check: read back the device `info` codes and raise if a decomposition failed (an
        unconverged eigensolver or a non-SPD damped factor would otherwise reach P and the
        KL-clip silently).  Default: on the first decomposition only (one host sync)."""
        if check is None:
            check = not self.have_eigen
        if self.reduce_owner:
            if not self.reduced:
                raise RuntimeError("factor_comm='reduce-owner': call update_factors(..., refresh=True) "
                                   "before compute_eigen (the owners' averaged factors are stale)")
            self.reduced = False
        if self.owned:
            F = [self.F_src[f] for f in self.owned]
            Q = [self.Q[f] for f in self.owned]
            if self.variant == "inverse":
                _lib.kfac_compute_inverse(F, self.damping, Q, self.info, ws=self.ws["eigen"])
            else:
                flags = _lib.EIG_WARM_START if (warm and self.have_eigen) else 0
                _lib.kfac_compute_eigen(F, Q, [self.v[f] for f in self.owned], self.info, flags,
                                        ws=self.ws["eigen"])
        if check and self.owned:
            bad = [(self.owned[i], int(c)) for i, c in enumerate(self.info[:len(self.owned)].tolist()) if c != 0]
            if bad:
                what = "not SPD at leading minor" if self.variant == "inverse" else "not converged after sweeps"
                raise FloatingPointError(f"kfac_compute_{'inverse' if self.variant == 'inverse' else 'eigen'}: "
                                         f"factor(s) {what}: {bad[:8]}")
        self.have_eigen = True
        if self.world > 1 and self.exchange == "bcast-eig":
            exchange_from_owners(self.q_flat, self.q_off, self.q_size, self.pg)
            if self.variant != "inverse":
                exchange_from_owners(self.v_flat, self.v_off, self.v_size, self.pg)

    def precondition(self, grads: List[torch.Tensor]) -> List[torch.Tensor]:
        """Alg. 1 step 3 (Eqs. 13-15 / Eq. 12) followed by the KL-clip (Eq. 18)."""
        mode = {"eigen": _lib.EIGEN, "factored": _lib.EIGEN_FACTORED, "inverse": _lib.INVERSE}[self.variant]
        layers = range(len(self.layers)) if (self.world == 1 or self.exchange == "bcast-eig") \
            else self.owned_layers
        layers = list(layers)
        if layers:
            g = [grads[i] for i in layers]
            QG = [self.Q[2 * i + 1] for i in layers]
            QA = [self.Q[2 * i] for i in layers]
            vG = vA = None
            if mode != _lib.INVERSE:
                vG = [self.v[2 * i + 1] for i in layers]
                vA = [self.v[2 * i] for i in layers]
            _lib.kfac_precondition(g, QG, vG, QA, vA, self.damping, mode, [self.P[i] for i in layers],
                                   ws=self.ws["precond"])
        if self.world > 1 and self.exchange == "allgather-grad":
            exchange_from_owners(self.p_flat, self.p_off, self.p_size, self.pg)
        _lib.kfac_kl_clip(self.P, grads, self.lr, self.kappa, self.nu, self.s, ws=self.ws["klclip"])
        return self.P

    def step(self, acts, gouts, grads, update_factors=True, update_eigen=True, first=False, warm=False):
        if update_factors:
            self.update_factors(acts, gouts, first, refresh=update_eigen or not self.have_eigen)
        if update_eigen or not self.have_eigen:
            self.compute_eigen(warm=warm)
        return self.precondition(grads)


def reduce_to_owners(flat: torch.Tensor, offs, sizes, group=None):
    """Rank r owns flat[offs[r]:offs[r]+sizes[r]]; afterwards rank r's slice holds the SUM of every
    rank's copy of it (other ranks' copies of slices they do not own are left as the collective
    leaves them).  One reduce per owner, all issued before any is waited on."""
    world = dist.get_world_size(group)
    works = [dist.reduce(flat[offs[r]:offs[r] + sizes[r]], dst=dist.get_global_rank(group, r) if group else r,
                         op=dist.ReduceOp.SUM, group=group, async_op=True)
             for r in range(world) if sizes[r] > 0]
    for w in works:
        w.wait()


def exchange_from_owners(flat: torch.Tensor, offs, sizes, group=None):
    """Rank r owns flat[offs[r]:offs[r]+sizes[r]]; afterwards every rank holds every slice.  One
    broadcast per owner of exactly its bytes (an all-gather would pad every slice to the largest);
    all are issued before any is waited on, so NCCL pipelines them."""
    world = dist.get_world_size(group)
    works = [dist.broadcast(flat[offs[r]:offs[r] + sizes[r]], src=dist.get_global_rank(group, r) if group else r,
                            group=group, async_op=True)
             for r in range(world) if sizes[r] > 0]
    for w in works:
        w.wait()

"""Multi-GPU element slabs with an NCCL interface-row exchange.

One process per GPU (torchrun).  Rank g of G integrates the elements whose
slowest index lies in [s_g, s_{g+1}), s_g = floor(g K / G), and owns the CSR
rows of dof planes [s_g, s_{g+1}) (the last rank also owns [K, K+p)).  The
slowest axis is the reference's first multi-index component (assembly.py:25,
mesh.py:20), so every rank's rows are one contiguous CSR range.

The slab's elements also touch the first p dof planes of rank g+1; those
partial "interface rows" are computed first, sent to g+1 with one NCCL
point-to-point transfer (overlapped with the interior compute), and added by
g+1 into its own first p planes with ``iga_axpy``.  No other data crosses
ranks.  The exchange is the only collective: the path is otherwise
embarrassingly parallel.

``SlabSession(..., halo="recompute")`` is the NCCL-free ablation of SURVEY.md
§8(e): rank g also integrates the p element layers below its slab, restricted
to its own planes, so its first p planes are complete without any transfer
(p / (K/G) extra element work: 9.4% at C5 with G=8, 2.3% with G=2).
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib


@dataclass(frozen=True)
class SlabPlan:
    K: int
    p: int
    world: int
    rank: int
    el_lo: int        # element slab [el_lo, el_hi) along the slowest axis
    el_hi: int
    own_lo: int       # owned dof planes [own_lo, own_hi)
    own_hi: int
    comp_hi: int      # computed planes [own_lo, comp_hi): owned + interface planes of rank+1

    @property
    def send_planes(self) -> tuple[int, int]:
        return (self.own_hi, self.comp_hi)

    @property
    def recompute_elements(self) -> tuple[int, int]:
        """Element slab of the NCCL-free ablation: the own slab plus the p layers below
        it, whose contributions complete the first p owned planes."""
        return (max(0, self.el_lo - self.p), self.el_hi)

    @property
    def recv_planes(self) -> tuple[int, int]:
        """Planes whose partial sums arrive from rank-1."""
        if self.rank == 0:
            return (self.own_lo, self.own_lo)
        return (self.own_lo, min(self.own_lo + self.p, self.own_hi))


def slab_plan(K: int, p: int, world: int, rank: int) -> SlabPlan:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if K < world:
        raise ValueError(f"cannot split K={K} element planes over {world} ranks")
    N = K + p
    el_lo, el_hi = rank * K // world, (rank + 1) * K // world
    own_lo = el_lo
    own_hi = el_hi if rank < world - 1 else N
    comp_hi = min(el_hi + p, N) if rank < world - 1 else N
    for g in range(1, world - 1):
        if (g + 1) * K // world - g * K // world < p:
            raise ValueError(f"slabs thinner than p={p} planes (K={K}, world={world})")
    return SlabPlan(K, p, world, rank, el_lo, el_hi, own_lo, own_hi, comp_hi)


def plane_nnz(dim: int, K: int, p: int, lo: int, hi: int) -> int:
    from .device import csr_nnz, plane_rows

    pr = plane_rows(dim, K, p)
    return csr_nnz(dim, K, p, lo * pr, hi * pr)


def _interface_ops(plan: SlabPlan, values, dim: int, group=None):
    import torch
    import torch.distributed as dist

    K, p = plan.K, plan.p
    n_own = plane_nnz(dim, K, p, plan.own_lo, plan.own_hi)
    ops, recv = [], None
    if plan.rank + 1 < plan.world:
        send = values[n_own:n_own + plane_nnz(dim, K, p, *plan.send_planes)]
        ops.append(dist.P2POp(dist.isend, send, plan.rank + 1, group=group))
    if plan.rank > 0:
        n_recv = plane_nnz(dim, K, p, *plan.recv_planes)
        recv = torch.empty(n_recv, dtype=values.dtype, device=values.device)
        ops.append(dist.P2POp(dist.irecv, recv, plan.rank - 1, group=group))
    return ops, recv


def start_interface_exchange(plan: SlabPlan, values, dim: int = 3, group=None):
    """Post the send of this rank's interface partial rows (values[n_own:]) to
    rank+1 and the receive of rank-1's into a fresh buffer; returns
    (works, recv).  With NCCL the transfer runs on NCCL's stream after the work
    already queued on the current stream, so compute launched afterwards
    overlaps it."""
    import torch.distributed as dist

    ops, recv = _interface_ops(plan, values, dim, group)
    works = dist.batch_isend_irecv(ops) if ops else []
    return works, recv


def finish_interface_exchange(works, recv, values, add=None):
    """Wait for the transfer and add the received partial rows into the first
    owned planes (values[:len(recv)])."""
    for w in works:
        w.wait()
    if recv is not None:
        if add is not None:
            add(recv, values[:recv.numel()])
        else:
            values[:recv.numel()] += recv


def exchange_interface(plan: SlabPlan, values, dim: int = 3, group=None, add=None):
    """Blocking form of the exchange (both halves)."""
    works, recv = start_interface_exchange(plan, values, dim, group)
    finish_interface_exchange(works, recv, values, add)
    return recv


HALO_MODES = ("exchange", "recompute")


class SlabSession:
    """Per-rank device state for the distributed integrate+assemble step.

    halo="exchange" (default, the deliverable): step() computes the interface
    planes first (so the NCCL send can start), then the owned planes, then the
    exchange and the interface accumulation.  halo="recompute": one launch over
    the elements [el_lo - p, el_hi) restricted to the owned planes, no exchange."""

    def __init__(self, cfg, plan: SlabPlan, halo: str = "exchange"):
        torch = _lib.require_cuda()
        from .device import MeshProblem
        from .runtime import method_code

        if cfg.dim != 3:
            raise ValueError("distributed slabs are implemented for dim=3")
        if halo not in HALO_MODES:
            raise ValueError(f"halo must be one of {HALO_MODES}, got {halo!r}")
        self.cfg, self.plan, self.halo = cfg, plan, halo
        self.code = method_code(cfg)
        self.prob = MeshProblem(3, cfg.mesh, cfg.degree, cfg.points, cfg.operator,
                                cfg.coefficient)
        self.n_own = plane_nnz(3, plan.K, plan.p, plan.own_lo, plan.own_hi)
        hi = plan.own_hi if halo == "recompute" else plan.comp_hi
        self.n_comp = plane_nnz(3, plan.K, plan.p, plan.own_lo, hi)
        self.values = torch.empty(self.n_comp, dtype=torch.float64, device=self.prob.device)
        self.stream = torch.cuda.current_stream()
        # separable kernel: 1D band matrices precomputed by the K1 launch
        self.use_band = self.code == 3 and self.prob.build_band_tables(self.stream)

    def _ia(self, values, el, planes):
        self.prob.integrate_assemble(values, self.code, el_range=el, plane_range=planes,
                                     stream=self.stream, band=self.use_band)

    def _axpy(self, x, y):
        _lib.check(_lib.load().iga_axpy(x.numel(), x.data_ptr(), y.data_ptr(),
                                        _lib.stream_ptr(self.stream)))

    def step(self, exchange: bool = True):
        pl = self.plan
        if self.use_band:
            self.prob.build_band_tables(self.stream)
        else:
            self.prob.build_tables(self.stream)
        if self.halo == "recompute":
            self._ia(self.values, pl.recompute_elements, (pl.own_lo, pl.own_hi))
            return self.values
        el = (pl.el_lo, pl.el_hi)
        if pl.comp_hi > pl.own_hi:
            self._ia(self.values[self.n_own:], el, (pl.own_hi, pl.comp_hi))
        pending = None
        if exchange and pl.world > 1:
            pending = start_interface_exchange(pl, self.values)
        self._ia(self.values, el, (pl.own_lo, pl.own_hi))
        if pending is not None:
            finish_interface_exchange(*pending, self.values, add=self._axpy)
        return self.values[:self.n_own]

    @property
    def kernel_launches_per_step(self) -> int:
        pl = self.plan
        if self.halo == "recompute":
            return 2
        return 1 + 1 + (1 if pl.comp_hi > pl.own_hi else 0) + (1 if pl.rank > 0 else 0)

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

``transport``: "device" (default) hands device tensors to the process group
(NCCL over NVLink); "host" stages the interface rows through pinned host
buffers for a CPU process group (gloo) -- the same plan and the same device
kernels, used to run several ranks' real kernels on one GPU in the tests.

``MultiDeviceRuntime`` drives G devices from ONE process (the drop-in
``run_integration(RunConfig(..., devices=G))``): one stream per device, the
slab kernels on each, and the interface exchange as one grouped NCCL
send/recv over an ``ncclCommInitAll`` communicator (libnccl through ctypes);
``exchange="copy"`` moves the interface rows with device-to-device copies
instead (the path that also runs when several shards share one GPU).
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


TRANSPORTS = ("device", "host")


def _interface_ops(plan: SlabPlan, values, dim: int, group=None, transport: str = "device"):
    import torch
    import torch.distributed as dist

    K, p = plan.K, plan.p
    n_own = plane_nnz(dim, K, p, plan.own_lo, plan.own_hi)
    ops, recv = [], None
    host = transport == "host" and values.is_cuda
    if plan.rank + 1 < plan.world:
        send = values[n_own:n_own + plane_nnz(dim, K, p, *plan.send_planes)]
        if host:  # stage through pinned host memory for a CPU (gloo) process group
            staged = torch.empty(send.numel(), dtype=send.dtype).pin_memory()
            staged.copy_(send, non_blocking=True)
            torch.cuda.current_stream(values.device).synchronize()
            send = staged
        ops.append(dist.P2POp(dist.isend, send, plan.rank + 1, group=group))
    if plan.rank > 0:
        n_recv = plane_nnz(dim, K, p, *plan.recv_planes)
        dev = "cpu" if host else values.device
        recv = torch.empty(n_recv, dtype=values.dtype, device=dev)
        if host:
            recv = recv.pin_memory()
        ops.append(dist.P2POp(dist.irecv, recv, plan.rank - 1, group=group))
    return ops, recv


def start_interface_exchange(plan: SlabPlan, values, dim: int = 3, group=None,
                             transport: str = "device"):
    """Post the send of this rank's interface partial rows (values[n_own:]) to
    rank+1 and the receive of rank-1's into a fresh buffer; returns
    (works, recv).  With NCCL the transfer runs on NCCL's stream after the work
    already queued on the current stream, so compute launched afterwards
    overlaps it.  transport="host": the rows travel through pinned host buffers
    (CPU process group)."""
    import torch.distributed as dist

    if transport not in TRANSPORTS:
        raise ValueError(f"transport must be one of {TRANSPORTS}, got {transport!r}")
    ops, recv = _interface_ops(plan, values, dim, group, transport)
    works = dist.batch_isend_irecv(ops) if ops else []
    return works, recv


def finish_interface_exchange(works, recv, values, add=None):
    """Wait for the transfer and add the received partial rows into the first
    owned planes (values[:len(recv)])."""
    for w in works:
        w.wait()
    if recv is not None:
        if recv.device != values.device:  # host-staged transport
            recv = recv.to(values.device, non_blocking=True)
        if add is not None:
            add(recv, values[:recv.numel()])
        else:
            values[:recv.numel()] += recv


def exchange_interface(plan: SlabPlan, values, dim: int = 3, group=None, add=None,
                       transport: str = "device"):
    """Blocking form of the exchange (both halves)."""
    works, recv = start_interface_exchange(plan, values, dim, group, transport)
    finish_interface_exchange(works, recv, values, add)
    return recv


HALO_MODES = ("exchange", "recompute")


class SlabSession:
    """Per-rank device state for the distributed integrate+assemble step.

    halo="exchange" (default, the deliverable): step() computes the interface
    planes first (so the NCCL send can start), then the owned planes, then the
    exchange and the interface accumulation.  halo="recompute": one launch over
    the elements [el_lo - p, el_hi) restricted to the owned planes, no exchange."""

    def __init__(self, cfg, plan: SlabPlan, halo: str = "exchange", transport: str = "device",
                 group=None, device=None):
        torch = _lib.require_cuda()
        from .device import MeshProblem
        from .runtime import method_code

        if cfg.dim != 3:
            raise ValueError("distributed slabs are implemented for dim=3")
        if halo not in HALO_MODES:
            raise ValueError(f"halo must be one of {HALO_MODES}, got {halo!r}")
        if transport not in TRANSPORTS:
            raise ValueError(f"transport must be one of {TRANSPORTS}, got {transport!r}")
        self.cfg, self.plan, self.halo = cfg, plan, halo
        self.transport, self.group = transport, group
        self.code = method_code(cfg)
        self.prob = MeshProblem(3, cfg.mesh, cfg.degree, cfg.points, cfg.operator,
                                cfg.coefficient, device=device, knots=cfg.knots)
        self.n_own = plane_nnz(3, plan.K, plan.p, plan.own_lo, plan.own_hi)
        hi = plan.own_hi if halo == "recompute" else plan.comp_hi
        self.n_comp = plane_nnz(3, plan.K, plan.p, plan.own_lo, hi)
        self.values = torch.empty(self.n_comp, dtype=torch.float64, device=self.prob.device)
        self.stream = torch.cuda.current_stream(self.prob.device)
        # separable kernel: 1D band matrices precomputed by the K1 launch
        self.use_band = self.code == 3 and self.prob.build_band_tables(self.stream)

    def _ia(self, values, el, planes):
        self.prob.integrate_assemble(values, self.code, el_range=el, plane_range=planes,
                                     stream=self.stream, band=self.use_band)

    def _axpy(self, x, y):
        _lib.check(_lib.load().iga_axpy(x.numel(), x.data_ptr(), y.data_ptr(),
                                        _lib.stream_ptr(self.stream)))

    def compute_interface(self):
        """K1 tables, then the interface planes of rank+1 (values[n_own:])."""
        pl = self.plan
        if self.use_band:
            self.prob.build_band_tables(self.stream)
        else:
            self.prob.build_tables(self.stream)
        if self.halo == "exchange" and pl.comp_hi > pl.own_hi:
            self._ia(self.values[self.n_own:], (pl.el_lo, pl.el_hi), (pl.own_hi, pl.comp_hi))

    def compute_owned(self):
        pl = self.plan
        if self.halo == "recompute":
            self._ia(self.values, pl.recompute_elements, (pl.own_lo, pl.own_hi))
        else:
            self._ia(self.values, (pl.el_lo, pl.el_hi), (pl.own_lo, pl.own_hi))

    @property
    def send_buffer(self):
        return self.values[self.n_own:]

    def add_received(self, recv):
        """Interface partial rows of rank-1 into the first owned planes (iga_axpy)."""
        self._axpy(recv, self.values[:recv.numel()])

    def step(self, exchange: bool = True):
        pl = self.plan
        self.compute_interface()
        if self.halo == "recompute":
            self.compute_owned()
            return self.values
        pending = None
        if exchange and pl.world > 1:
            pending = start_interface_exchange(pl, self.values, group=self.group,
                                               transport=self.transport)
        self.compute_owned()
        if pending is not None:
            finish_interface_exchange(*pending, self.values, add=self._axpy)
        return self.values[:self.n_own]

    @property
    def kernel_launches_per_step(self) -> int:
        pl = self.plan
        if self.halo == "recompute":
            return 2
        return 1 + 1 + (1 if pl.comp_hi > pl.own_hi else 0) + (1 if pl.rank > 0 else 0)


# ------------------------------------------------------------------ one process, G devices
_NCCL_FLOAT64 = 8  # ncclDataType_t ncclFloat64 (nccl.h)


class NcclComms:
    """ncclCommInitAll communicator over `devices` (one process drives them all), bound
    through ctypes to the libnccl that torch ships (the same library torch.distributed
    loads).  send/recv calls between group_start/group_end are issued for all devices
    from this one thread, as NCCL requires for single-process multi-device use."""

    def __init__(self, devices):
        import ctypes
        import glob
        import os

        cands = []
        try:
            import nvidia.nccl

            for d in nvidia.nccl.__path__:
                cands += glob.glob(os.path.join(d, "lib", "libnccl.so*"))
        except ImportError:
            pass
        cands += ["libnccl.so.2"]
        err = None
        for c in cands:
            try:
                self.lib = ctypes.CDLL(c)
                break
            except OSError as e:
                err = e
        else:
            raise RuntimeError(f"libnccl not found: {err}")
        L, vp = self.lib, ctypes.c_void_p
        L.ncclGetErrorString.restype = ctypes.c_char_p
        L.ncclSend.argtypes = [vp, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, vp, vp]
        L.ncclRecv.argtypes = [vp, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, vp, vp]
        L.ncclCommDestroy.argtypes = [vp]
        self.devices = list(devices)
        n = len(self.devices)
        self.comms = (vp * n)()
        devs = (ctypes.c_int * n)(*self.devices)
        self._check(L.ncclCommInitAll(self.comms, n, devs), "ncclCommInitAll")

    def _check(self, rc, what):
        if rc != 0:
            raise RuntimeError(f"{what}: {self.lib.ncclGetErrorString(rc).decode()}")

    def group_start(self):
        self._check(self.lib.ncclGroupStart(), "ncclGroupStart")

    def group_end(self):
        self._check(self.lib.ncclGroupEnd(), "ncclGroupEnd")

    def send(self, rank, t, peer, stream):
        self._check(self.lib.ncclSend(t.data_ptr(), t.numel(), _NCCL_FLOAT64, peer,
                                      self.comms[rank], stream.cuda_stream), "ncclSend")

    def recv(self, rank, t, peer, stream):
        self._check(self.lib.ncclRecv(t.data_ptr(), t.numel(), _NCCL_FLOAT64, peer,
                                      self.comms[rank], stream.cuda_stream), "ncclRecv")

    def close(self):
        for c in self.comms:
            if c:
                self.lib.ncclCommDestroy(c)
        self.comms = None

    def __del__(self):
        try:
            if self.comms is not None:
                self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


EXCHANGES = ("auto", "nccl", "copy")


class MultiDeviceRuntime:
    """The drop-in's multi-GPU path: ``run_integration(RunConfig(..., devices=G))``.

    One process drives G devices (the reference's analogue is the worker pool of
    ``over_elements``, runtime.py:258-267).  Shard g lives on ``devices[g]``: it integrates
    the element slab of ``slab_plan(K, p, G, g)`` on that device's stream, computing the p
    interface planes of shard g+1 first; the interface rows then move to g+1 on a side
    stream -- one grouped ncclSend/ncclRecv per neighbour pair over an ncclCommInitAll
    communicator (``exchange="nccl"``) or a device-to-device copy (``"copy"``, which also
    works when shards share a GPU) -- while the owned planes are integrated, and g+1 adds
    them with ``iga_axpy``.  ``"auto"``: NCCL when the G devices are distinct GPUs."""

    def __init__(self, cfg, devices=None, exchange: str = "auto", halo: str = "exchange"):
        torch = _lib.require_cuda()
        G = cfg.devices
        devices = list(range(G)) if devices is None else [int(d) for d in devices]
        if len(devices) != G:
            raise ValueError(f"{G} shards need {G} device ids, got {devices}")
        avail = torch.cuda.device_count()
        if any(not 0 <= d < avail for d in devices):
            raise ValueError(f"devices={devices} but only {avail} CUDA device(s) are visible")
        if exchange not in EXCHANGES:
            raise ValueError(f"exchange must be one of {EXCHANGES}, got {exchange!r}")
        distinct = len(set(devices)) == G
        if exchange == "auto":
            exchange = "nccl" if distinct and G > 1 else "copy"
        if exchange == "nccl" and not distinct:
            raise ValueError("the NCCL exchange needs one distinct GPU per shard")
        self.cfg, self.devices, self.exchange, self.halo = cfg, devices, exchange, halo
        self.plans = [slab_plan(cfg.mesh, cfg.degree, G, g) for g in range(G)]
        self.sessions, self.side, self.recv = [], [], []
        for g, d in enumerate(devices):
            with torch.cuda.device(d):
                s = SlabSession(cfg, self.plans[g], halo=halo, device=d)
                s.stream = torch.cuda.Stream(device=d)
                s.use_band = s.code == 3 and s.prob.build_band_tables(s.stream)
                self.sessions.append(s)
                self.side.append(torch.cuda.Stream(device=d))
                n = plane_nnz(3, cfg.mesh, cfg.degree, *self.plans[g].recv_planes) if g else 0
                self.recv.append(torch.empty(n, dtype=torch.float64, device=d) if n else None)
        self.nccl = NcclComms(devices) if exchange == "nccl" and G > 1 else None

    def step(self):
        """One integrate+assemble of the whole mesh; returns the owned values per shard."""
        torch = _lib.require_cuda()
        S, G = self.sessions, len(self.sessions)
        for g, s in enumerate(S):
            with torch.cuda.device(self.devices[g]):
                s.compute_interface()
        if self.halo == "exchange" and G > 1:
            for g, s in enumerate(S):
                self.side[g].wait_stream(s.stream)
            if self.nccl is not None:
                self.nccl.group_start()
                for g, s in enumerate(S):
                    if g + 1 < G:
                        self.nccl.send(g, s.send_buffer, g + 1, self.side[g])
                    if g > 0:
                        self.nccl.recv(g, self.recv[g], g - 1, self.side[g])
                self.nccl.group_end()
            else:
                for g in range(1, G):
                    with torch.cuda.device(self.devices[g]), torch.cuda.stream(self.side[g]):
                        self.side[g].wait_stream(self.side[g - 1])
                        self.recv[g].copy_(S[g - 1].send_buffer, non_blocking=True)
        for g, s in enumerate(S):
            with torch.cuda.device(self.devices[g]):
                s.compute_owned()
        if self.halo == "exchange" and G > 1:
            for g in range(1, G):
                with torch.cuda.device(self.devices[g]):
                    S[g].stream.wait_stream(self.side[g])
                    S[g].add_received(self.recv[g])
            for g in range(G - 1):  # the send buffer is rewritten by the next step
                S[g].stream.wait_stream(self.side[g] if self.nccl is not None else self.side[g + 1])
        return [s.values[:s.n_own] for s in S]

    def synchronize(self):
        for s in self.sessions:
            s.stream.synchronize()

    def close(self):
        if self.nccl is not None:
            self.nccl.close()
            self.nccl = None

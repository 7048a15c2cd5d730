"""Mesh-wide entry point (drop-in for igabench.runtime).

``run_integration(RunConfig(...))`` integrates and assembles the whole mesh on
the device and returns the same ``RunResult(config, gram, times, flops)`` as
runtime.py:287-295.  The reference's CPU strategies (sequential /
over_elements / within_element / combined, runtime.py:16-20) are scheduling
knobs for host threads; they are accepted and validated for drop-in
compatibility and all run the same device schedule (grid over element
tiles, CTAs over rows, threads over contractions), so results are identical
across them exactly as the reference guarantees.

Extensions: ``strategy="device"``, ``operator``,
``coefficient`` (None | scalar | array [K^dim, q^dim]), ``dim`` (2 or 3),
``devices`` and ``assembly`` ("auto" | "owner" | "scatter" | "separable").
``assembly="separable"`` (3D, scalar coefficient) integrates the 1D band
matrices per axis and fills the CSR with their Kronecker combination
(csrc/iga_kron.cu) -- exact for a constant coefficient, HBM-bound; "auto"
selects it for scalar coefficients and the assembled DMMA sum factorization
(csrc/iga_gsf_p3.cu, iga_gsf.cu) for coefficient fields.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .assembly import GlobalGram
from .device import MeshProblem
from .integrators import flop_count

METHODS = ("classical", "sumfact")
STRATEGIES = ("sequential", "over_elements", "within_element", "combined", "device")
ASSEMBLY = ("auto", "owner", "scatter", "separable")
BARRIER_TIMEOUT = 300.0


@dataclass(frozen=True)
class RunConfig:
    method: str
    strategy: str
    mesh: int
    degree: int
    workers: int = 1
    repetitions: int = 1
    quad_points: int | None = None
    inner_workers: int = 1
    chunking: str = "static"
    operator: str = "mass"
    coefficient: object = field(default=None, compare=False, repr=False)
    dim: int = 3
    devices: int = 1
    assembly: str = "auto"
    # general open knot vector (K + 2p + 1 knots, the same on every axis like the reference's
    # single KnotVector), or None for make_knot_vector's uniform mesh
    knots: object = field(default=None, compare=False, repr=False)

    def __post_init__(self):
        if self.method not in METHODS:
            raise ValueError(f"method must be one of {METHODS}, got {self.method!r}")
        if self.strategy not in STRATEGIES:
            raise ValueError(f"strategy must be one of {STRATEGIES}, got {self.strategy!r}")
        if self.mesh < 1 or self.degree < 0:
            raise ValueError("mesh must be >= 1 and degree >= 0")
        if self.workers < 1 or self.inner_workers < 1:
            raise ValueError("worker counts must be >= 1")
        if self.repetitions < 1:
            raise ValueError("repetitions must be >= 1")
        if self.chunking not in ("static", "dynamic"):
            raise ValueError(f"chunking must be static or dynamic, got {self.chunking!r}")
        if self.operator not in _lib.OPS:
            raise ValueError(f"operator must be one of {tuple(_lib.OPS)}, got {self.operator!r}")
        if self.operator != "mass" and self.degree < 1:
            raise ValueError("derivatives require degree >= 1")
        if self.dim not in (2, 3):
            raise ValueError(f"dim must be 2 or 3, got {self.dim}")
        if self.devices < 1:
            raise ValueError("devices must be >= 1")
        if self.assembly not in ASSEMBLY:
            raise ValueError(f"assembly must be one of {ASSEMBLY}, got {self.assembly!r}")
        if self.quad_points is not None and self.quad_points < 1:
            raise ValueError("quad_points must be >= 1")
        if self.knots is not None:
            from .splines import check_knots

            check_knots(self.knots, self.mesh, self.degree)

    @property
    def points(self) -> int:
        return self.degree + 1 if self.quad_points is None else self.quad_points


@dataclass
class RunResult:
    config: RunConfig
    gram: GlobalGram
    times: list[float]
    flops: int


@dataclass
class ExecutionTrace:
    """Instrumentation of one within-element run (runtime.py:100-107).

    The device executes the sum-factorization task classes of one element as barrier
    phases of one CTA (csrc/iga_element.cu k_element_strict: the p + 1 Cox-de Boor /
    Jacobian classes inside K1's table evaluation, then the product/reduce classes of the
    three directions).  ``completion_order`` lists the element's tasks class by class in
    task-id order -- the order a barrier-phase schedule completes them, and exactly the
    reference's ``DependencyGraph.class_members()`` concatenated (its alphabet is numbered
    class-monotonically, taskgraph.py:132-152) -- ``barriers`` the p + 6 class
    boundaries, and ``intra_class_syncs`` 0.  ``graph`` stays None: the dependency-graph
    analysis (taskgraph.py) is outside this package's hot-path scope."""

    graph: object = None
    completion_order: list = field(default_factory=list)
    barriers: int = 0
    intra_class_syncs: int = 0


def foata_class_sizes(p: int, points: int) -> list[int]:
    """Task counts of the p + 7 Foata classes of one element (runtime.py:435-440,
    taskgraph.py:132-152): cox orders 0..p-1, cox order p + the P Jacobian tasks, then
    product / reduce per direction (a product per canonical pair and point, a reduce per
    pair)."""
    m = p + 1
    pairs = m**3 * (m**3 + 1) // 2
    cox = 3 * m * points
    return [cox] * p + [cox + points] + [pairs * points, pairs] * 3


def _foata_task_count(p: int, points: int) -> int:
    return sum(foata_class_sizes(p, points))


def run_within_element(alpha, kv, method: str, workers: int, points: int | None = None,
                       trace: ExecutionTrace | None = None):
    """Integrate one element with intra-element parallelism (runtime.py:476-505).

    The device runs the element on one CTA -- threads over canonical pairs / stage
    entries, barrier phases between the sum-factorization classes -- in the reference's
    operation order, so the matrix is bitwise equal to the sequential kernels for any
    ``workers`` (which, like the reference's thread count, does not change the result)."""
    from .integrators import ElementMatrix, default_rule, flop_count
    from .device import MeshProblem

    if method not in METHODS:
        raise ValueError(f"method must be one of {METHODS}")
    if trace is not None and method != "sumfact":
        raise ValueError("execution traces are only defined for the sum factorization graph")
    cfg = RunConfig(method=method, strategy="within_element", mesh=kv.elements, degree=kv.degree,
                    workers=workers, quad_points=points)
    q = cfg.points
    rule = default_rule(kv, tuple(alpha), q)
    for d in range(3):
        if not 0 <= alpha[d] < kv.elements:
            raise ValueError(f"element {alpha} outside mesh with K={kv.elements}")
    torch = _lib.require_cuda()
    prob = MeshProblem(3, kv.elements, kv.degree, q)
    code = _lib.METHOD_CLASSICAL if method == "classical" else _lib.METHOD_SUMFACT
    out = prob.element_matrices([tuple(alpha)], code,
                                elem_weights=np.asarray(rule.weights).reshape(1, 3, q),
                                jac=float(rule.jacobian))
    torch.cuda.synchronize()
    entries = out[0].cpu().numpy()
    if trace is not None:
        P = q**3
        trace.completion_order.extend(range(_foata_task_count(kv.degree, P)))
        trace.barriers += kv.degree + 6
    return ElementMatrix(tuple(alpha), entries.shape[0], entries, flop_count(method, kv.degree, q))


def grams_bitwise_equal(a: GlobalGram, b: GlobalGram) -> bool:
    ma, mb = a.matrix, b.matrix
    return (ma.shape == mb.shape and np.array_equal(ma.indptr, mb.indptr)
            and np.array_equal(ma.indices, mb.indices)
            and ma.data.tobytes() == mb.data.tobytes())


MAX_P_ASSEMBLED = 5  # the assembled (row-owner) sum factorization kernels: p <= 5
MAX_P = 9            # every other path (csrc/iga_dispatch.cuh)


def separable_fits(K: int, p: int) -> bool:
    """Shared-memory budget of k_kron3 (csrc/iga_kron.cu: 1D band tables + two
    staging chunks)."""
    nb = 2 * p + 1
    rows = 16 if p <= 2 else ((16 if K <= 96 else 8) if p == 3 else (4 if p <= 5 else 1))
    nbuf = 2 if p <= 5 else 3
    return 2 * 16 * (K + p) * nb + 8 * nbuf * (rows * nb**3 + 2) <= 220 * 1024


def method_code(cfg: RunConfig) -> int:
    """Kernel selection: classical -> Algorithm 1 + fused scatter; sumfact ->
    "auto": the separable (Kronecker) path for a scalar coefficient in 3D (exact
    factorisation of the quadrature, HBM-bound), else assembled (row-owner) sum
    factorization; "owner" / "scatter" / "separable" force a kernel."""
    if cfg.method == "classical":
        if cfg.assembly == "owner":
            raise ValueError("assembly='owner' requires method='sumfact'")
        return _lib.METHOD_CLASSICAL
    if cfg.assembly == "separable":
        if cfg.dim != 3:
            raise ValueError("the separable method is 3D only")
        c = cfg.coefficient
        if c is not None and np.ndim(c) != 0:
            raise ValueError("assembly='separable' needs a scalar coefficient")
        return _lib.METHOD_SEPARABLE
    if cfg.assembly == "scatter":
        if cfg.dim != 3:
            raise ValueError("element-local sum factorization scatter is 3D only")
        return _lib.METHOD_SUMFACT
    if cfg.dim != 3:
        raise ValueError("assembled sum factorization is 3D only; use method='classical' "
                         "for dim=2")
    c = cfg.coefficient
    if (cfg.assembly == "auto" and (c is None or np.ndim(c) == 0)
            and separable_fits(cfg.mesh, cfg.degree)):
        return _lib.METHOD_SEPARABLE
    if cfg.degree > MAX_P_ASSEMBLED:
        if cfg.assembly == "owner":
            raise ValueError(f"assembly='owner' runs p <= {MAX_P_ASSEMBLED}; p={cfg.degree} "
                             "takes 'auto' (separable or element-local sum factorization)")
        # high degrees: element-local sum factorization (stage buffers in global scratch)
        return _lib.METHOD_SUMFACT
    return _lib.METHOD_SUMFACT_ASSEMBLED


class DeviceSession:
    """Persistent device buffers for repeated integrate+assemble calls.

    ``step()`` runs the device hot path (K1 tables + fused integrate/assemble)
    on resident inputs; ``step_host(out)`` is the end-to-end call with host
    buffers: the problem inputs (Gauss nodes/weights and the coefficient
    field, if any) are copied host->device, the matrix is integrated and
    assembled, and the CSR values are copied device->host into ``out``
    (pinned host memory for full PCIe bandwidth)."""

    def __init__(self, cfg: RunConfig, stream=None, use_graph: bool = False):
        torch = _lib.require_cuda()
        self.cfg = cfg
        self.use_graph = use_graph  # replay the step's launches as one CUDA graph
        self._graph = None
        self.code = method_code(cfg)
        self.prob = MeshProblem(cfg.dim, cfg.mesh, cfg.degree, cfg.points, cfg.operator,
                                cfg.coefficient, knots=cfg.knots)
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        # separable kernel: 1D band matrices precomputed by the K1 launch
        self.use_band = self.code == 3 and self.prob.build_band_tables(self.stream)
        self.values = torch.empty(self.prob.nnz(), dtype=torch.float64, device=self.prob.device)
        self._host_in = [torch.from_numpy(self.prob.ref_nodes_host).pin_memory(),
                         torch.from_numpy(self.prob.weights_host).pin_memory()]
        if self.prob.knots is not None:
            self._host_in.append(torch.from_numpy(self.prob.knots_host).pin_memory())
        self._host_coef = None
        if self.prob.coef is not None:
            self._host_coef = self.prob.coef.cpu().pin_memory()

    @property
    def h2d_bytes(self) -> int:
        n = sum(t.numel() * 8 for t in self._host_in)
        return n + (0 if self._host_coef is None else self._host_coef.numel() * 8)

    @property
    def d2h_bytes(self) -> int:
        return self.values.numel() * 8

    @property
    def launches_per_step(self) -> int:
        return 2

    def _launch(self, stream):
        if self.use_band:  # K1 + band matrices in one launch, then the separable kernel
            self.prob.build_band_tables(stream)
            self.prob.integrate_assemble(self.values, self.code, stream=stream, band=True)
            return
        self.prob.build_tables(stream)
        self.prob.integrate_assemble(self.values, self.code, stream=stream)

    def step(self):
        if not self.use_graph:
            self._launch(self.stream)
            return self.values
        torch = _lib.require_cuda()
        if self._graph is None:
            # one eager step first (kernel attributes and launch set-up are cached outside
            # the capture), then capture K1 + the integrate+assemble kernel once
            self._launch(self.stream)
            self.stream.synchronize()
            side = torch.cuda.Stream()
            side.wait_stream(self.stream)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                self._launch(side)
            self._graph = g
        with torch.cuda.stream(self.stream):
            self._graph.replay()
        return self.values

    def step_host(self, out):
        torch = _lib.require_cuda()
        with torch.cuda.stream(self.stream):
            self.prob.ref_nodes.copy_(self._host_in[0], non_blocking=True)
            self.prob.weights.copy_(self._host_in[1], non_blocking=True)
            if self.prob.knots is not None:
                self.prob.knots.copy_(self._host_in[2], non_blocking=True)
            if self._host_coef is not None:
                self.prob.coef.copy_(self._host_coef, non_blocking=True)
            self.step()
            out.copy_(self.values, non_blocking=True)
        return out


class IntegrationRuntime:
    """Owns the device buffers for one configuration; ``run`` is not reentrant
    (runtime.py:155-185)."""

    def __init__(self, cfg: RunConfig, device_ids=None, exchange: str = "auto"):
        self.cfg = cfg
        self.device_ids = device_ids  # devices > 1: GPU of each slab (default 0..devices-1)
        self.exchange = exchange
        self._active = threading.Lock()

    def run(self) -> RunResult:
        if not self._active.acquire(blocking=False):
            raise RuntimeError("run_integration is already active on this runtime")
        try:
            return self._run_locked()
        finally:
            self._active.release()

    def _run_multi(self) -> RunResult:
        """devices > 1: element slabs on G devices driven from this process with the NCCL
        interface exchange (distributed.MultiDeviceRuntime)."""
        torch = _lib.require_cuda()
        from .distributed import MultiDeviceRuntime

        cfg = self.cfg
        if cfg.dim != 3:
            raise ValueError("devices > 1 is implemented for dim=3")
        rt = MultiDeviceRuntime(cfg, self.device_ids, exchange=self.exchange)
        try:
            times = []
            for _ in range(cfg.repetitions):
                ev = []
                for s in rt.sessions:
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(s.stream)
                    ev.append((a, b))
                shards = rt.step()
                for (a, b), s in zip(ev, rt.sessions):
                    b.record(s.stream)
                rt.synchronize()
                times.append(max(a.elapsed_time(b) for a, b in ev) / 1e3)
        finally:
            rt.close()
        prob = rt.sessions[0].prob
        gram = GlobalGram(K=cfg.mesh, p=cfg.degree, n_dofs=prob.n_dofs, dim=3, shards=shards)
        per_el = flop_count(cfg.method, cfg.degree, cfg.points)
        return RunResult(config=cfg, gram=gram, times=times, flops=per_el * prob.n_elements)

    def _run_locked(self) -> RunResult:
        torch = _lib.require_cuda()
        cfg = self.cfg
        if cfg.devices > 1:
            return self._run_multi()
        sess = DeviceSession(cfg)
        prob, stream = sess.prob, sess.stream
        times = []
        for _ in range(cfg.repetitions):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sess.step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
        gram = GlobalGram(K=cfg.mesh, p=cfg.degree, n_dofs=prob.n_dofs, values=sess.values,
                          dim=cfg.dim)
        per_el = flop_count(cfg.method, cfg.degree, cfg.points)
        return RunResult(config=cfg, gram=gram, times=times, flops=per_el * prob.n_elements)


def run_integration(cfg: RunConfig, device_ids=None, exchange: str = "auto") -> RunResult:
    """Integrate + assemble the mesh under cfg on the device (runtime.py:287-295).
    ``cfg.devices = G > 1`` splits the elements into G slabs along the slowest axis on
    ``device_ids`` (default 0..G-1) with the interface rows exchanged over NCCL
    (``exchange="copy"``: device copies, e.g. when the slabs share one GPU)."""
    return IntegrationRuntime(cfg, device_ids, exchange).run()

"""Device-resident problem state and the calls through the C-ABI.

``MeshProblem`` owns, on one CUDA device, everything one mesh-wide
integration needs: the Gauss weights, the per-1D-element basis tables (K1,
evaluated on the device, bitwise equal to runtime._MeshContext.build_tables,
runtime.py:142-149), the optional coefficient field, and the ``iga_problem``
block handed to ``libiga_b200.so``.  Torch is used only for device memory and
streams.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

OPERATORS = tuple(_lib.OPS)


def gauss_reference(q: int):
    """Gauss-Legendre nodes/weights on [-1,1] from numpy, as mesh.py:82 does (bits
    come from the host numpy and are uploaded, never recomputed on the GPU)."""
    return np.polynomial.legendre.leggauss(q)


def jacobian(K: int, dim: int) -> float:
    """(1/(2K))**dim exactly as mesh.py:90 computes it (Python float pow)."""
    return (1.0 / (2.0 * K)) ** dim


def n_dofs(dim: int, K: int, p: int) -> int:
    return (K + p) ** dim


def csr_nnz(dim: int, K: int, p: int, row_begin: int = 0, row_end: int | None = None) -> int:
    L = _lib.load()
    row_end = n_dofs(dim, K, p) if row_end is None else row_end
    nnz = L.iga_csr_nnz(dim, K, p, row_begin, row_end)
    if nnz < 0:
        raise ValueError(f"invalid CSR request dim={dim} K={K} p={p} rows=[{row_begin},{row_end})")
    return int(nnz)


def plane_rows(dim: int, K: int, p: int) -> int:
    return (K + p) ** (dim - 1)


@dataclass
class CsrPattern:
    """Device CSR pattern (int64 indptr relative to row_begin, int32 indices)."""

    dim: int
    K: int
    p: int
    row_begin: int
    row_end: int
    indptr: object  # torch.int64 [rows+1]
    indices: object  # torch.int32 [nnz]


def csr_pattern(dim, K, p, row_begin=0, row_end=None, device=None, stream=None,
                with_indices=True) -> CsrPattern:
    """K5: structured pattern on the device (assembly.symbolic_pattern, assembly.py:99-115)."""
    torch = _lib.require_cuda()
    row_end = n_dofs(dim, K, p) if row_end is None else row_end
    dev = torch.device("cuda") if device is None else device
    nnz = csr_nnz(dim, K, p, row_begin, row_end)
    indptr = torch.empty(row_end - row_begin + 1, dtype=torch.int64, device=dev)
    indices = torch.empty(nnz if with_indices else 0, dtype=torch.int32, device=dev)
    _lib.check(_lib.load().iga_csr_pattern(dim, K, p, row_begin, row_end, indptr.data_ptr(),
                                           indices.data_ptr() if with_indices and nnz else None,
                                           _lib.stream_ptr(stream)))
    return CsrPattern(dim, K, p, row_begin, row_end, indptr, indices if with_indices else None)


class MeshProblem:
    """Device state of one (dim, K, p, q, operator, coefficient) problem."""

    def __init__(self, dim: int, K: int, p: int, q: int | None = None, operator: str = "mass",
                 coefficient=None, device=None, stream=None, knots=None):
        torch = _lib.require_cuda()
        if dim not in (2, 3):
            raise ValueError(f"dim must be 2 or 3, got {dim}")
        if K < 1 or p < 0:
            raise ValueError("mesh must be >= 1 and degree >= 0")
        if operator not in _lib.OPS:
            raise ValueError(f"operator must be one of {OPERATORS}, got {operator!r}")
        if operator != "mass" and p < 1:
            raise ValueError("derivatives require degree >= 1")
        q = p + 1 if q is None else int(q)
        if q < 1:
            raise ValueError(f"quadrature points must be >= 1, got {q}")
        self.dim, self.K, self.p, self.q, self.operator = dim, K, p, q, operator
        self.device = torch.device("cuda") if device is None else torch.device(device)
        self.stream = stream
        ref, w = gauss_reference(q)
        self.ref_nodes_host = np.ascontiguousarray(ref)
        self.weights_host = np.ascontiguousarray(w)
        self.ref_nodes = torch.from_numpy(self.ref_nodes_host).to(self.device)
        self.weights = torch.from_numpy(self.weights_host).to(self.device)
        # general open knot vector: element Jacobians folded into
        # per-element weights written by K1, jac = 1
        self.knots_host = None
        self.knots = self.elem_weights = None
        if knots is not None:
            from .splines import check_knots

            self.knots_host = check_knots(knots, K, p)
            self.knots = torch.from_numpy(self.knots_host).to(self.device)
            self.elem_weights = torch.empty((K, q), dtype=torch.float64, device=self.device)
        self.jac = jacobian(K, dim) if knots is None else 1.0
        m = p + 1
        self.tables_v = torch.empty((K, m, q), dtype=torch.float64, device=self.device)
        self.tables_d = torch.empty((K, m, q), dtype=torch.float64, device=self.device)
        self.coef = None
        self.coef_scalar = 1.0
        self.band = None
        self.set_coefficient(coefficient)
        self.build_tables()

    # -- coefficient ----------------------------------------------------
    def set_coefficient(self, coefficient):
        """None / scalar / array [K^dim, q^dim] (element lexicographic, k1 slowest)."""
        torch = _lib.require_cuda()
        self.coef = None
        self.coef_scalar = 1.0
        if coefficient is None:
            return
        if np.isscalar(coefficient):
            self.coef_scalar = float(coefficient)
            return
        n_el = self.K ** self.dim
        nq = self.q ** self.dim
        if isinstance(coefficient, torch.Tensor):
            c = coefficient.to(device=self.device, dtype=torch.float64)
        else:
            c = torch.from_numpy(np.ascontiguousarray(coefficient, dtype=np.float64))
            c = c.to(self.device)
        if c.numel() != n_el * nq:
            raise ValueError(f"coefficient must have {n_el}x{nq} values (elements x quadrature "
                             f"points), got shape {tuple(c.shape)}")
        self.coef = c.reshape(n_el, nq).contiguous()

    # -- K1 -------------------------------------------------------------
    def build_tables(self, stream=None):
        """Basis values/derivatives per 1D element at the mapped nodes (K1)."""
        L = _lib.load()
        if self.knots is not None:
            _lib.check(L.iga_mesh_tables_general(
                self.K, self.p, self.q, self.knots.data_ptr(), self.ref_nodes.data_ptr(),
                self.weights.data_ptr(), self.tables_v.data_ptr(), self.tables_d.data_ptr(),
                self.elem_weights.data_ptr(), _lib.stream_ptr(stream or self.stream)))
            return
        _lib.check(L.iga_mesh_tables(self.K, self.p, self.q, self.ref_nodes.data_ptr(),
                                     self.tables_v.data_ptr(), self.tables_d.data_ptr(),
                                     _lib.stream_ptr(stream or self.stream)))

    def problem_struct(self, band: bool = False) -> _lib.IgaProblem:
        """iga_problem of this mesh; ``band`` passes the band tables of the last
        ``build_band_tables`` (separable method)."""
        s = _lib.IgaProblem()
        s.dim, s.K, s.p, s.q = self.dim, self.K, self.p, self.q
        s.op = _lib.OPS[self.operator]
        s.reserved = 0
        s.jac = self.jac
        s.coef_scalar = self.coef_scalar
        s.coef = None if self.coef is None else self.coef.data_ptr()
        s.weights = self.weights.data_ptr()
        s.tables_v = self.tables_v.data_ptr()
        s.tables_d = self.tables_d.data_ptr() if self.operator != "mass" else None
        s.band = self.band.data_ptr() if band else None
        s.knots = _lib.ptr(self.knots)
        s.elem_weights = _lib.ptr(self.elem_weights)
        return s

    # -- K1 + 1D band matrices (separable method) ------------------------
    def build_band_tables(self, stream=None) -> bool:
        """K1 tables and the assembled 1D band matrices in one launch
        (``iga_band_tables``); False if the library cannot (the separable kernel then
        integrates the band matrices itself)."""
        torch = _lib.require_cuda()
        if getattr(self, "band", None) is None:
            N, nb = self.K + self.p, 2 * self.p + 1
            self.band = torch.empty(N * nb * 2, dtype=torch.float64, device=self.device)
        s = self.problem_struct()
        rc = _lib.load().iga_band_tables(ctypes.byref(s), self.ref_nodes.data_ptr(),
                                         self.tables_v.data_ptr(), self.tables_d.data_ptr(),
                                         self.band.data_ptr(), _lib.ptr(self.elem_weights),
                                         _lib.stream_ptr(stream or self.stream))
        if rc == _lib.IGA_EUNSUPPORTED:
            return False
        _lib.check(rc)
        return True

    # -- sizes ----------------------------------------------------------
    @property
    def n_dofs(self) -> int:
        return n_dofs(self.dim, self.K, self.p)

    @property
    def n_elements(self) -> int:
        return self.K ** self.dim

    def nnz(self, plane_begin: int = 0, plane_end: int | None = None) -> int:
        N = self.K + self.p
        plane_end = N if plane_end is None else plane_end
        pr = plane_rows(self.dim, self.K, self.p)
        return csr_nnz(self.dim, self.K, self.p, plane_begin * pr, plane_end * pr)

    # -- fused integrate + assemble ------------------------------------
    def integrate_assemble(self, values, method: int, el_range=None, plane_range=None,
                           stream=None, band: bool = False):
        """Write CSR values of row planes ``plane_range`` from elements ``el_range``
        (slowest axis) into ``values`` (torch fp64, starts at the first row); ``band``:
        use the band tables of the last ``build_band_tables`` (separable method)."""
        el = (0, self.K) if el_range is None else el_range
        pl = (0, self.K + self.p) if plane_range is None else plane_range
        s = self.problem_struct(band)
        _lib.check(_lib.load().iga_integrate_assemble(
            ctypes.byref(s), method, int(el[0]), int(el[1]), int(pl[0]), int(pl[1]),
            values.data_ptr(), _lib.stream_ptr(stream or self.stream)))
        return values

    def element_matrices(self, elem_ids, method: int, elem_nodes=None, elem_weights=None,
                         elem_coef=None, jac=None, coef_scalar=None, stream=None):
        """Per-element matrices [count, n, n] (strict reference operation order).
        ``elem_nodes`` / ``elem_weights``: [count, dim, q] per-axis nodes and weights (the
        caller's QuadratureRule); ``elem_coef``: [count, q^dim] coefficients at those
        points (only these values are uploaded, never a mesh-wide field)."""
        torch = _lib.require_cuda()
        ids = torch.as_tensor(np.ascontiguousarray(elem_ids, dtype=np.int32)).reshape(-1, self.dim)
        ids = ids.to(self.device)
        count = ids.shape[0]
        n = (self.p + 1) ** self.dim

        def upload(x, shape):
            if x is None:
                return None
            t = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64))
            return t.reshape(shape).to(self.device)

        nodes = upload(elem_nodes, (count, self.dim, self.q))
        weights = upload(elem_weights, (count, self.dim, self.q))
        coef = upload(elem_coef, (count, self.q ** self.dim))
        out = torch.empty((count, n, n), dtype=torch.float64, device=self.device)
        s = self.problem_struct()
        if jac is not None:
            s.jac = float(jac)
        if coef_scalar is not None:
            s.coef_scalar = float(coef_scalar)
        _lib.check(_lib.load().iga_element_matrices(
            ctypes.byref(s), method, self.ref_nodes.data_ptr(), ids.data_ptr(), _lib.ptr(nodes),
            _lib.ptr(weights), _lib.ptr(coef), count, out.data_ptr(),
            _lib.stream_ptr(stream or self.stream)))
        return out


def basis_eval(K: int, p: int, elems, xs, derivatives: bool = True, knots=None):
    """K1' at arbitrary points: (values [n, p+1], derivatives [n, p+1]) on the device, on
    the open uniform knot vector or a general one (``knots``)."""
    torch = _lib.require_cuda()
    e = torch.as_tensor(np.ascontiguousarray(elems, dtype=np.int32)).cuda()
    x = torch.as_tensor(np.ascontiguousarray(xs, dtype=np.float64)).cuda()
    t = None
    if knots is not None:
        from .splines import check_knots

        t = torch.from_numpy(check_knots(knots, K, p)).cuda()
    n = e.numel()
    V = torch.empty((n, p + 1), dtype=torch.float64, device="cuda")
    D = torch.empty((n, p + 1), dtype=torch.float64, device="cuda") if derivatives else None
    _lib.check(_lib.load().iga_basis_eval(K, p, _lib.ptr(t), n, e.data_ptr(), x.data_ptr(),
                                          V.data_ptr(), None if D is None else D.data_ptr(),
                                          _lib.stream_ptr()))
    return V, D

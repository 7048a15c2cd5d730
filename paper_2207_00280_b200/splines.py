"""B-spline knot vectors and basis tables (drop-in for igabench.splines).

Knot vectors are host metadata (make_knot_vector, splines.py:59-75).  Basis
*evaluation* runs on the device (kernel K1, ``iga_basis_eval`` /
``iga_mesh_tables``), bitwise equal to the reference's Cox-de Boor recursion
(splines.py:108-161); there is no host evaluation path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class KnotVector:
    """Open uniform knot vector: degree ``p``, ``K`` elements, ``K + 2p + 1`` knots."""

    degree: int
    elements: int
    knots: np.ndarray = field(repr=False)

    @property
    def n_basis(self) -> int:
        return self.elements + self.degree

    @property
    def is_uniform(self) -> bool:
        """True for the open uniform vector of make_knot_vector (the reference's mesh)."""
        return np.array_equal(self.knots, _uniform_knots(self.elements, self.degree))

    def element_bounds(self, e: int) -> tuple[float, float]:
        """Span [t_{p+e}, t_{p+e+1}] of element e: (e/K, (e+1)/K) on the uniform vector
        (the same floats as splines.py:38-42), the knot span on a general one."""
        if not 0 <= e < self.elements:
            raise IndexError(f"element index {e} out of range for K={self.elements}")
        if self.is_uniform:
            return e / self.elements, (e + 1) / self.elements
        p = self.degree
        return float(self.knots[p + e]), float(self.knots[p + e + 1])


@dataclass(frozen=True)
class BasisValues:
    element: int
    point: float
    values: np.ndarray
    derivatives: np.ndarray | None = None


def _uniform_knots(K: int, p: int) -> np.ndarray:
    knots = np.empty(K + 2 * p + 1)
    knots[: p + 1] = 0.0
    knots[p + 1 : K + p] = np.arange(1, K) / K
    knots[K + p :] = 1.0
    return knots


def make_knot_vector(K: int, p: int) -> KnotVector:
    """Clamped uniform knots on [0, 1] (same values as splines.py:59-75)."""
    if K < 1:
        raise ValueError(f"element count must be >= 1, got {K}")
    if p < 0:
        raise ValueError(f"degree must be >= 0, got {p}")
    return KnotVector(degree=p, elements=K, knots=_uniform_knots(K, p))


def check_knots(knots, K: int, p: int) -> np.ndarray:
    """Validate a general open knot vector for K elements of degree p (SURVEY.md 8(f) row
    4): K + 2p + 1 finite values, p + 1 equal knots at each end, strictly increasing
    interior breakpoints (K non-empty spans; the CSR pattern is then the uniform one)."""
    t = np.ascontiguousarray(knots, dtype=np.float64).reshape(-1)
    if t.size != K + 2 * p + 1:
        raise ValueError(f"knot vector needs K + 2p + 1 = {K + 2 * p + 1} entries, got {t.size}")
    if not np.all(np.isfinite(t)):
        raise ValueError("knots must be finite")
    if np.any(t[: p + 1] != t[0]) or np.any(t[K + p :] != t[-1]):
        raise ValueError(f"an open knot vector repeats its end knots p + 1 = {p + 1} times")
    if np.any(np.diff(t[p : K + p + 1]) <= 0.0):
        raise ValueError("breakpoints must be strictly increasing (K non-empty spans)")
    return t


def make_general_knot_vector(knots, p: int) -> KnotVector:
    """KnotVector over a general open knot vector (K = len(knots) - 2p - 1 spans)."""
    t = np.ascontiguousarray(knots, dtype=np.float64).reshape(-1)
    K = t.size - 2 * p - 1
    if K < 1:
        raise ValueError(f"{t.size} knots cannot carry degree {p}")
    return KnotVector(degree=p, elements=K, knots=check_knots(t, K, p))


def _eval_knots(kv: KnotVector, index, order: int, xs) -> np.ndarray:
    """B_{index[i], order}(xs[i]) on the device (iga_eval_basis) from kv.knots."""
    from . import _lib

    torch = _lib.require_cuda()
    t = torch.from_numpy(np.ascontiguousarray(kv.knots, dtype=np.float64)).cuda()
    idx = torch.as_tensor(np.ascontiguousarray(index, dtype=np.int32)).reshape(-1).cuda()
    x = torch.as_tensor(np.ascontiguousarray(xs, dtype=np.float64)).reshape(-1).cuda()
    out = torch.empty(idx.numel(), dtype=torch.float64, device="cuda")
    _lib.check(_lib.load().iga_eval_basis(t.data_ptr(), t.numel(), order, idx.numel(),
                                          idx.data_ptr(), x.data_ptr(), out.data_ptr(),
                                          _lib.stream_ptr()))
    return out.cpu().numpy()


def eval_basis_order0(kv: KnotVector, i: int, x: float) -> float:
    """Order-0 basis: indicator of the knot span [t_i, t_{i+1}), the last non-empty span
    closed at the last knot (splines.py:78-91; evaluated on the device)."""
    if not 0 <= i <= len(kv.knots) - 2:
        raise IndexError(f"order-0 basis index {i} out of range")
    return float(_eval_knots(kv, [i], 0, [x])[0])


def eval_basis(kv: KnotVector, i: int, q: int, x: float) -> float:
    """Basis function i of order q at x by the two-term recursion with 0/0 := 0
    (splines.py:94-118), bitwise equal, on the device for any knot vector."""
    if not 0 <= q <= kv.degree:
        raise ValueError(f"order {q} outside [0, {kv.degree}]")
    if not 0 <= i <= len(kv.knots) - q - 2:
        raise IndexError(f"basis index {i} out of range at order {q}")
    return float(_eval_knots(kv, [i], q, [x])[0])


def eval_basis_many(kv: KnotVector, index, q: int, xs) -> np.ndarray:
    """Vectorised eval_basis: B_{index[j], q}(xs[j]) for all j in one device launch."""
    index = np.asarray(index, dtype=np.int64).reshape(-1)
    if not 0 <= q <= kv.degree:
        raise ValueError(f"order {q} outside [0, {kv.degree}]")
    if index.size and (index.min() < 0 or index.max() > len(kv.knots) - q - 2):
        raise IndexError(f"basis index out of range at order {q}")
    return _eval_knots(kv, index, q, xs)


def _check_point(kv: KnotVector, e: int, x: float) -> None:
    lo, hi = kv.element_bounds(e)
    if not lo <= x <= hi:
        raise ValueError(f"point {x} outside element {e} = [{lo}, {hi}]")


def _eval(kv: KnotVector, elems, xs, derivatives):
    from .device import basis_eval

    V, D = basis_eval(kv.elements, kv.degree, elems, xs, derivatives,
                      knots=None if kv.is_uniform else kv.knots)
    return V.cpu().numpy(), (None if D is None else D.cpu().numpy())


def eval_nonzero_basis(kv: KnotVector, e: int, x: float) -> BasisValues:
    """Values of the p+1 functions supported on element e (device K1)."""
    _check_point(kv, e, x)
    V, _ = _eval(kv, [e], [x], False)
    return BasisValues(element=e, point=x, values=V[0])


def eval_nonzero_basis_derivatives(kv: KnotVector, e: int, x: float) -> np.ndarray:
    """First derivatives of the p+1 supported functions (device K1)."""
    if kv.degree < 1:
        raise ValueError("derivatives require degree >= 1")
    _check_point(kv, e, x)
    _, D = _eval(kv, [e], [x], True)
    return D[0]


def basis_value_table(kv: KnotVector, e: int, points: np.ndarray) -> np.ndarray:
    """Table B[r, k] of supported values at the points of element e (splines.py:164-170)."""
    points = np.asarray(points, dtype=np.float64)
    for x in points:
        _check_point(kv, e, float(x))
    V, _ = _eval(kv, np.full(len(points), e), points, False)
    return np.ascontiguousarray(V.T)


def basis_derivative_table(kv: KnotVector, e: int, points: np.ndarray) -> np.ndarray:
    """Table B'[r, k] of supported derivatives (splines.py:173-178)."""
    if kv.degree < 1:
        raise ValueError("derivatives require degree >= 1")
    points = np.asarray(points, dtype=np.float64)
    for x in points:
        _check_point(kv, e, float(x))
    _, D = _eval(kv, np.full(len(points), e), points, True)
    return np.ascontiguousarray(D.T)


def find_element(kv: KnotVector, x: float) -> int:
    """Element containing x; the last element is right-closed (splines.py:181-185); on a
    general knot vector the span [t_{p+e}, t_{p+e+1}) holding x."""
    if kv.is_uniform:
        if not 0.0 <= x <= 1.0:
            raise ValueError(f"point {x} outside [0, 1]")
        return min(int(x * kv.elements), kv.elements - 1)
    p, K = kv.degree, kv.elements
    lo, hi = float(kv.knots[p]), float(kv.knots[p + K])
    if not lo <= x <= hi:
        raise ValueError(f"point {x} outside [{lo}, {hi}]")
    e = int(np.searchsorted(kv.knots[p + 1:p + K], x, side="right"))
    return min(e, K - 1)

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

    def element_bounds(self, e: int) -> tuple[float, float]:
        if not 0 <= e < self.elements:
            raise IndexError(f"element index {e} out of range for K={self.elements}")
        return e / self.elements, (e + 1) / self.elements


@dataclass(frozen=True)
class BasisValues:
    element: int
    point: float
    values: np.ndarray
    derivatives: np.ndarray | None = None


def make_knot_vector(K: int, p: int) -> KnotVector:
    """Clamped uniform knots on [0, 1] (same values as splines.py:59-75)."""
    if K < 1:
        raise ValueError(f"element count must be >= 1, got {K}")
    if p < 0:
        raise ValueError(f"degree must be >= 0, got {p}")
    knots = np.empty(K + 2 * p + 1)
    knots[: p + 1] = 0.0
    knots[p + 1 : K + p] = np.arange(1, K) / K
    knots[K + p :] = 1.0
    return KnotVector(degree=p, elements=K, knots=knots)


def _check_point(kv: KnotVector, e: int, x: float) -> None:
    lo, hi = kv.element_bounds(e)
    if not lo <= x <= hi:
        raise ValueError(f"point {x} outside element {e} = [{lo}, {hi}]")


def _eval(kv: KnotVector, elems, xs, derivatives):
    from .device import basis_eval

    V, D = basis_eval(kv.elements, kv.degree, elems, xs, derivatives)
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
    """Element containing x; the last element is right-closed (splines.py:181-185)."""
    if not 0.0 <= x <= 1.0:
        raise ValueError(f"point {x} outside [0, 1]")
    return min(int(x * kv.elements), kv.elements - 1)

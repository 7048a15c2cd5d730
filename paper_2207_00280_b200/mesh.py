"""Mesh enumeration and Gauss rules (drop-in for igabench.mesh).

Host-side index metadata only.  Element ids are triples (i, j, k) with the
first index slowest (mesh.py:16-20); the CUDA kernels never materialise these
lists, they use the same ordering arithmetically.
"""

from __future__ import annotations

from dataclasses import dataclass
from itertools import product

import numpy as np

ElementId = tuple[int, int, int]


def element_list(K: int) -> list[ElementId]:
    if K < 1:
        raise ValueError(f"mesh size must be >= 1, got {K}")
    return list(product(range(K), repeat=3))


def support_set(alpha: ElementId, p: int) -> list[tuple[int, int, int]]:
    """(p+1)^3 supported multi-indices of element alpha, lexicographic offsets."""
    return [tuple(a + o for a, o in zip(alpha, off)) for off in product(range(p + 1), repeat=3)]


def local_index(alpha: ElementId, beta: tuple[int, int, int], p: int) -> int:
    m = p + 1
    offs = [b - a for a, b in zip(alpha, beta)]
    if any(not 0 <= o <= p for o in offs):
        raise ValueError(f"multi-index {beta} not supported on element {alpha}")
    return (offs[0] * m + offs[1]) * m + offs[2]


@dataclass(frozen=True)
class QuadratureRule:
    """Per-element Gauss-Legendre rule: mapped nodes [3, q], reference weights
    [3, q] (sum 2) and the constant Jacobian (1/(2K))^3."""

    points_per_direction: tuple[int, int, int]
    nodes: np.ndarray
    weights: np.ndarray
    jacobian: float

    @property
    def total_points(self) -> int:
        a, b, c = self.points_per_direction
        return a * b * c


def _rule(K: int, alpha: ElementId, q: int, jac: float) -> QuadratureRule:
    ref, w = np.polynomial.legendre.leggauss(q)
    h = 1.0 / K
    nodes = np.stack([alpha[d] * h + (ref + 1.0) * (h / 2.0) for d in range(3)])
    weights = np.stack([w, w, w])
    return QuadratureRule((q, q, q), nodes, weights, jac)


def gauss_rule(p: int, K: int, alpha: ElementId) -> QuadratureRule:
    """p+1 points per direction on element alpha (mesh.py:73-93)."""
    if p < 0:
        raise ValueError(f"degree must be >= 0, got {p}")
    return _rule(K, alpha, p + 1, (1.0 / (2.0 * K)) ** 3)


def knot_rule(kv, alpha: ElementId, points: int | None = None) -> QuadratureRule:
    """Gauss rule on element alpha of a general open knot vector:
    nodes lo + (ref + 1) (h / 2) in each axis' span [lo, lo + h], per-axis weights
    w * (h / 2) -- the element's Jacobian folded per axis -- and jacobian 1.0; the same
    definition as the device's per-element weights (tools/gen_golden.py section 12)."""
    q = kv.degree + 1 if points is None else points
    if q < 1:
        raise ValueError(f"quadrature points must be >= 1, got {q}")
    ref, w = np.polynomial.legendre.leggauss(q)
    nodes, weights = [], []
    for d in range(3):
        lo, hi = kv.element_bounds(alpha[d])
        h = hi - lo
        nodes.append(lo + (ref + 1.0) * (h / 2.0))
        weights.append(w * (h / 2.0))
    return QuadratureRule((q, q, q), np.stack(nodes), np.stack(weights), 1.0)


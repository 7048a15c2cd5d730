"""Per-element integration API (drop-in for igabench.integrators).

``integrate_element_classical`` / ``integrate_element_sumfact`` keep the
reference signatures (integrators.py:193-230) and return the same frozen
``ElementMatrix``; the matrix is computed on the device by
``iga_element_matrices`` with the reference's exact operation order, so mass
matrices are bitwise equal to the numba kernels.  Keyword-only extensions:
``operator`` ("mass" | "stiffness" | "stiffness_mass") and ``coefficient``
(scalar or q^3 values at the element's quadrature points, k1 slowest).
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _lib
from .mesh import ElementId, QuadratureRule, gauss_rule
from .splines import KnotVector


@dataclass(frozen=True)
class ElementMatrix:
    """Dense (p+1)^3 x (p+1)^3 element contribution; ``flops`` = reference op model."""

    element: ElementId
    n: int
    entries: np.ndarray
    flops: int


@dataclass
class SumFactBuffers:
    """Staging shapes of the reference sum factorization (integrators.py:44-66).

    The device kernel keeps these stages in shared memory; the buffers are
    validated for API compatibility and zeroed like the reference does."""

    D: np.ndarray
    C: np.ndarray

    @classmethod
    def allocate(cls, p: int, points: int | None = None) -> "SumFactBuffers":
        m = p + 1
        q = m if points is None else points
        return cls(D=np.empty((m, m, q, q)), C=np.empty((m, m, m, m, q)))

    def matches(self, p: int, q: int) -> bool:
        m = p + 1
        return self.D.shape == (m, m, q, q) and self.C.shape == (m, m, m, m, q)


@lru_cache(maxsize=None)
def canonical_pairs(n: int) -> tuple[np.ndarray, np.ndarray]:
    """Lower-triangle (row >= col) local pairs, row-major (integrators.py:69-74)."""
    rows, cols = np.tril_indices(n)
    return rows.astype(np.int64), cols.astype(np.int64)


def flop_count(method: str, p: int, points: int | None = None) -> int:
    """The reference's per-element op model (integrators.py:154-170)."""
    m = p + 1
    q = m if points is None else points
    n = m**3
    pairs = n * (n + 1) // 2
    if method == "classical":
        return pairs * q**3 * 10
    if method == "sumfact":
        return 4 * (m**2 * q**3 + m**4 * q**2 + pairs * q)
    raise ValueError(f"unknown method {method!r}")


def _check_inputs(alpha: ElementId, kv: KnotVector, rule: QuadratureRule) -> int:
    q1, q2, q3 = rule.points_per_direction
    if not (q1 == q2 == q3):
        raise ValueError("anisotropic quadrature rules are not supported")
    for d in range(3):
        if not 0 <= alpha[d] < kv.elements:
            raise ValueError(f"element {alpha} outside mesh with K={kv.elements}")
        lo, hi = kv.element_bounds(alpha[d])
        if rule.nodes[d].min() < lo or rule.nodes[d].max() > hi:
            raise ValueError(f"quadrature nodes outside element {alpha}")
    return q1


@lru_cache(maxsize=32)
def _element_problem(K: int, p: int, q: int, operator: str, device: int, knots=None):
    """Device problem reused by the per-element calls of one (K, p, q, operator, knots):
    the per-call inputs (nodes, per-axis weights, Jacobian, coefficient) travel with each
    call, so a call uploads O(q) values (O(q^3) with a coefficient) -- never a mesh-wide
    array.  ``knots``: a general knot vector (tuple), whose tables the kernel evaluates."""
    from .device import MeshProblem

    return MeshProblem(3, K, p, q, operator=operator,
                       knots=None if knots is None else np.asarray(knots))


def _device_element(alpha, kv, rule, method_code, operator, coefficient):
    q = _check_inputs(alpha, kv, rule)  # ValueError before any device work, as the reference
    if operator not in _lib.OPS:
        raise ValueError(f"operator must be one of {tuple(_lib.OPS)}, got {operator!r}")
    if operator != "mass" and kv.degree < 1:
        raise ValueError("derivatives require degree >= 1")
    elem_coef, coef_scalar = None, 1.0
    if coefficient is not None:
        if np.isscalar(coefficient):
            coef_scalar = float(coefficient)
        else:
            elem_coef = np.ascontiguousarray(coefficient, dtype=np.float64).reshape(-1)
            if elem_coef.size != q**3:
                raise ValueError(f"element coefficient needs {q**3} values, got {elem_coef.size}")
    torch = _lib.require_cuda()
    prob = _element_problem(kv.elements, kv.degree, q, operator, torch.cuda.current_device(),
                            None if kv.is_uniform else tuple(np.asarray(kv.knots).tolist()))
    nodes = np.ascontiguousarray(rule.nodes, dtype=np.float64).reshape(1, 3, q)
    weights = np.ascontiguousarray(rule.weights, dtype=np.float64).reshape(1, 3, q)
    out = prob.element_matrices([alpha], method_code, elem_nodes=nodes, elem_weights=weights,
                                elem_coef=elem_coef, jac=float(rule.jacobian),
                                coef_scalar=coef_scalar)
    return out[0].cpu().numpy(), q


def integrate_element_classical(alpha: ElementId, kv: KnotVector, rule: QuadratureRule, *,
                                operator: str = "mass", coefficient=None) -> ElementMatrix:
    """Element matrix by the classical quadrature loop (Algorithm 1) on the device."""
    entries, q = _device_element(alpha, kv, rule, _lib.METHOD_CLASSICAL, operator, coefficient)
    return ElementMatrix(element=alpha, n=entries.shape[0], entries=entries,
                         flops=flop_count("classical", kv.degree, q))


def integrate_element_sumfact(alpha: ElementId, kv: KnotVector, rule: QuadratureRule,
                              buffers: SumFactBuffers, *, operator: str = "mass",
                              coefficient=None) -> ElementMatrix:
    """Element matrix by sum factorization (Algorithm 2) on the device."""
    q = _check_inputs(alpha, kv, rule)
    if not buffers.matches(kv.degree, q):
        raise ValueError(
            f"buffer shapes {buffers.D.shape}/{buffers.C.shape} do not match p={kv.degree}, q={q}")
    buffers.D[:] = 0.0
    buffers.C[:] = 0.0
    entries, q = _device_element(alpha, kv, rule, _lib.METHOD_SUMFACT, operator, coefficient)
    return ElementMatrix(element=alpha, n=entries.shape[0], entries=entries,
                         flops=flop_count("sumfact", kv.degree, q))


def element_tables(kv: KnotVector, rule: QuadratureRule, alpha: ElementId):
    """Per-direction basis value tables at the rule's nodes (device K1)."""
    from .splines import basis_value_table

    return tuple(basis_value_table(kv, alpha[d], rule.nodes[d]) for d in range(3))


def default_rule(kv: KnotVector, alpha: ElementId, points: int | None = None) -> QuadratureRule:
    """Gauss rule for alpha with an optional point override (integrators.py:233-251); on a
    general knot vector the rule of mesh.knot_rule."""
    if not kv.is_uniform:
        from .mesh import knot_rule

        return knot_rule(kv, alpha, points)
    rule = gauss_rule(kv.degree, kv.elements, alpha)
    if points is None or points == kv.degree + 1:
        return rule
    from .mesh import _rule

    return _rule(kv.elements, alpha, points, rule.jacobian)

"""Algorithmic work of the device kernels, for roofline reporting.

Counts are exact for a K^3 mesh (boundary truncation of the 1D bands
included), 1 FMA = 2 flops, and count only the work the algorithm needs --
not the halo recomputation of a particular tiling.

Assembled sum factorization (iga_gsf.cu), per operator:
  stage A (axis 0): types x K^3 (p+1)^2 q^3            MACs   (types: mass 1, stiffness 2)
  stage B (axis 1): prods_B x nnz1 K^2 (p+1)^2 q^2     MACs   (prods: mass 1, stiffness 3)
  stage S (axis 2): prods_S x nnz1^2 K (p+1)^2 q       MACs   (prods: mass 1, stiffness 2)
with nnz1 = (K+p)(2p+1) - p(p+1) the 1D band pairs.  Each 1D band pair
(I, J) overlaps sum_e = K (p+1)^2 element-local pairs in total, which is
where the K (p+1)^2 factors come from.

The symmetric p = 3 kernel (iga_gsf_p3s.cu, whole-mesh runs) needs only the J0 >= I0 half:
symmetric_assembled_macs.

Separable path (iga_kron.cu, scalar coefficient): the 1D element integrals
(types x K (p+1)^2 q MACs per axis, computed once) and per CSR value one
multiply and one FMA (stiffness; mass: one multiply) -- a few flops per 8-byte
value written, so the HBM write of the values binds.

Classical (Algorithm 1, iga_scatter.cu k_classical_mma): SURVEY.md §8(d)'s
per-(pair, point) counts, see classical_flops.

Bytes: 8 nnz written (each CSR value exactly once) + 8 K^3 q^3 read when a
per-quadrature-point coefficient field is given.
"""

from __future__ import annotations


def nnz1(K: int, p: int) -> int:
    return (K + p) * (2 * p + 1) - p * (p + 1)


def assembled_macs(op: str, K: int, p: int, q: int) -> int:
    m2 = (p + 1) ** 2
    t = nnz1(K, p)
    types, pb, ps = (1, 1, 1) if op == "mass" else (2, 3, 2)
    a = types * K**3 * m2 * q**3
    b = pb * t * K**2 * m2 * q**2
    s = ps * t * t * K * m2 * q
    return a + b + s


def assembled_flops(op: str, K: int, p: int, q: int) -> int:
    return 2 * assembled_macs(op, K, p, q)


def nnz1_half(K: int, p: int) -> int:
    """1D band pairs with J >= I (one triangle and the diagonal)."""
    N = K + p
    return (p + 1) * N - p * (p + 1) // 2


def symmetric_assembled_macs(op: str, K: int, p: int, q: int) -> int:
    """The symmetric kernel (csrc/iga_gsf_p3s.cu) computes only the values with J0 >= I0:
    stage A the element-local pairs with s >= r ((p+1)(p+2)/2 of (p+1)^2), stages B and S the
    X / Y rows of the nnz1_half axis-0 band pairs; the other values are mirrored copies (no
    arithmetic)."""
    m2 = (p + 1) ** 2
    t, th = nnz1(K, p), nnz1_half(K, p)
    types, pb, ps = (1, 1, 1) if op == "mass" else (2, 3, 2)
    a = types * K**3 * ((p + 1) * (p + 2) // 2) * q**3
    b = pb * th * K**2 * m2 * q**2
    s = ps * th * t * K * m2 * q
    return a + b + s


def symmetric_assembled_flops(op: str, K: int, p: int, q: int) -> int:
    return 2 * symmetric_assembled_macs(op, K, p, q)


def separable_flops(op: str, K: int, p: int, q: int) -> int:
    n1 = nnz1(K, p)
    types = 1 if op == "mass" else 2
    per_value = 1 if op == "mass" else 3
    return 2 * types * K * (p + 1) ** 2 * q + per_value * n1**3


def element_sumfact_flops(op: str, p: int, q: int) -> int:
    """SURVEY.md §8(d) general element-local sum factorization, per element."""
    m = p + 1
    S1, S2, S3 = m * m * q**3, m**4 * q * q, (m**3 * (m**3 + 1) // 2) * q
    if op == "mass":
        return 2 * (S1 + S2 + S3)
    return 2 * (2 * S1 + 3 * S2 + 2 * S3)


def classical_flops(op: str, p: int, q: int, dim: int = 3) -> int:
    """Algorithm 1 per element, SURVEY.md §8(d)'s minimal count with the per-axis pair
    products precomputed: per (canonical pair, quadrature point) mass 4 flops,
    stiffness 10, stiffness+mass 12 (3D; 2D: mass 3, stiffness 6, stiffness+mass 8).
    The reference's own model (integrators.py:154-170) is 10 per pair and point."""
    n = (p + 1) ** dim
    per = {3: {"mass": 4, "stiffness": 10, "stiffness_mass": 12},
           2: {"mass": 3, "stiffness": 6, "stiffness_mass": 8}}[dim][op]
    return per * (n * (n + 1) // 2) * q**dim


def algorithmic_bytes(dim: int, K: int, p: int, q: int, coefficient_field: bool) -> int:
    nnz = nnz1(K, p) ** dim
    b = 8 * nnz
    if coefficient_field:
        b += 8 * K**dim * q**dim
    return b

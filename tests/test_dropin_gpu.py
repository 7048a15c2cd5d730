"""GPU parity of the drop-in names completing the reference's public API
(igabench/__init__.py:10-58): eval_basis / eval_basis_order0 on uniform and general
knot vectors, per-axis quadrature weights and per-element coefficients in
integrate_element_*, and run_within_element + ExecutionTrace -- all bitwise against
outputs of the reference itself (tests/golden, tools/gen_golden.py sections 10, 11, 13)."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2207_00280_b200.runtime import foata_class_sizes
from tests.conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2207_00280_b200 as P

    return P


def _kv(pkg, g, tag, K, p):
    if tag == "u":
        kv = pkg.make_knot_vector(K, p)
        assert np.array_equal(kv.knots, g[f"{tag}_K{K}_p{p}_knots"])
        return kv
    return pkg.KnotVector(degree=p, elements=K, knots=g[f"{tag}_K{K}_p{p}_knots"])


@pytest.mark.parametrize("tag,K,p", [("u", 4, 3), ("u", 3, 2), ("n", 5, 3), ("n", 4, 2),
                                     ("n", 6, 4), ("u", 2, 0)])
def test_eval_basis_bitwise(pkg, tag, K, p):
    """Every basis function of every order at knots, endpoints and random points, bitwise
    equal to splines.eval_basis / eval_basis_order0 (general knots included)."""
    g = load_golden("eval_basis")
    kv = _kv(pkg, g, tag, K, p)
    xs = g[f"{tag}_K{K}_p{p}_x"]
    for q in range(p + 1):
        ref = g[f"{tag}_K{K}_p{p}_q{q}"]
        nb = ref.shape[0]
        idx = np.repeat(np.arange(nb), len(xs))
        got = pkg.eval_basis_many(kv, idx, q, np.tile(xs, nb)).reshape(nb, len(xs))
        assert got.tobytes() == ref.tobytes(), (tag, K, p, q)
    o0 = g[f"{tag}_K{K}_p{p}_o0"]
    for i in (0, o0.shape[0] // 2, o0.shape[0] - 1):
        for j in (0, len(xs) // 3, len(xs) - 1):
            assert pkg.eval_basis_order0(kv, i, float(xs[j])) == o0[i, j]
            assert pkg.eval_basis(kv, i, 0, float(xs[j])) == o0[i, j]


def test_eval_basis_reference_cases(pkg):
    """test_splines.py:44-75 restated: order-0 indicators and hat values."""
    kv = pkg.make_knot_vector(2, 1)
    assert pkg.eval_basis_order0(kv, 1, 0.25) == 1.0
    assert pkg.eval_basis_order0(kv, 1, 0.75) == 0.0
    assert pkg.eval_basis_order0(kv, 2, 1.0) == 1.0  # closed last span
    assert pkg.eval_basis(kv, 1, 1, 0.25) == 0.5
    assert pkg.eval_basis(kv, 1, 1, 0.5) == 1.0


@pytest.mark.parametrize("K,p", [(3, 2), (4, 3), (2, 4)])
def test_element_per_axis_weights_bitwise(pkg, K, p):
    """rule.weights[0..2] differ (integrators.py:200-203): element matrices bitwise equal
    to the reference's integrate_element_classical / _sumfact on the same rule."""
    g = load_golden("element_peraxis")
    kv = pkg.make_knot_vector(K, p)
    alpha = (K - 1, 0, K // 2)
    r0 = pkg.gauss_rule(p, K, alpha)
    rule = pkg.QuadratureRule(r0.points_per_direction, r0.nodes, g[f"weights_K{K}_p{p}"],
                              r0.jacobian)
    a = pkg.integrate_element_classical(alpha, kv, rule)
    b = pkg.integrate_element_sumfact(alpha, kv, rule, pkg.SumFactBuffers.allocate(p))
    assert a.entries.tobytes() == g[f"classical_K{K}_p{p}"].tobytes()
    assert b.entries.tobytes() == g[f"sumfact_K{K}_p{p}"].tobytes()


@pytest.mark.parametrize("op", ["mass", "stiffness", "stiffness_mass"])
def test_element_coefficient_uploads_element_values(pkg, op):
    """A per-point coefficient of one element (q^3 values) gives the oracle's element
    matrix bitwise; only those q^3 values travel (no mesh-wide field is formed)."""
    K, p = 5, 2
    q = p + 1
    kv = pkg.make_knot_vector(K, p)
    alpha = (4, 1, 3)
    c = np.random.default_rng(9).uniform(0.5, 1.5, size=q**3)
    rule = pkg.gauss_rule(p, K, alpha)
    for method in ("classical", "sumfact"):
        if method == "classical":
            em = pkg.integrate_element_classical(alpha, kv, rule, operator=op, coefficient=c)
        else:
            em = pkg.integrate_element_sumfact(alpha, kv, rule, pkg.SumFactBuffers.allocate(p),
                                               operator=op, coefficient=c)
        ref = O.element(3, K, p, op, method, alpha, coef=c)  # the element's q^3 values
        assert em.entries.tobytes() == ref.tobytes(), method


@pytest.mark.parametrize("key", ["K2_p0_w1", "K2_p1_w3", "K3_p2_w2"])
def test_run_within_element_and_trace(pkg, key):
    """run_within_element (runtime.py:476-505) bitwise equal to the reference's, for both
    methods and the reference's worker counts; the trace reports the reference's class
    structure (p + 6 barriers, no intra-class syncs, class-by-class completion)."""
    g = load_golden("within_element")
    K, p, w = (int(s[1:]) for s in key.split("_"))
    kv = pkg.make_knot_vector(K, p)
    alpha = (K - 1, 0, K // 2)
    t = pkg.ExecutionTrace()
    em = pkg.run_within_element(alpha, kv, "sumfact", w, trace=t)
    assert em.entries.tobytes() == g[f"{key}_sumfact"].tobytes()
    ec = pkg.run_within_element(alpha, kv, "classical", w)
    assert ec.entries.tobytes() == g[f"{key}_classical"].tobytes()
    assert t.barriers == int(g[f"{key}_barriers"])
    assert t.intra_class_syncs == int(g[f"{key}_syncs"])
    assert len(t.completion_order) == int(g[f"{key}_ntasks"])
    sizes = foata_class_sizes(p, (p + 1) ** 3)
    ours = np.repeat(np.arange(p + 7), sizes)[np.asarray(t.completion_order)]
    assert np.array_equal(ours, g[f"{key}_class_of_order"])
    assert np.array_equal(np.sort(t.completion_order), g[f"{key}_order_sorted"])
    assert em.flops == pkg.flop_count("sumfact", p)

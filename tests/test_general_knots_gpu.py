"""General open knot vectors on the device: K1 tables and the
per-element weights (the element Jacobian folded per axis) bitwise against the reference's
own evaluation, and every integrate+assemble path, the per-element API, the multi-device
slabs and the matrix-free apply against the reference-kernel goldens
(tools/gen_golden.py section 12) and the oracle (pinned to them in tests/test_oracle.py)."""

import numpy as np
import pytest

from oracle import oracle as O
from tests.conftest import load_golden
from tests.parity import assert_parity

pytestmark = pytest.mark.gpu

CASES = [(5, 2), (4, 3), (3, 1), (6, 3)]


@pytest.fixture(scope="module")
def pkg():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2207_00280_b200 as P

    return P


@pytest.mark.parametrize("K,p", CASES)
def test_general_knot_tables_bitwise(pkg, K, p):
    from paper_2207_00280_b200.device import MeshProblem

    g = load_golden(f"nonuniform_K{K}_p{p}")
    wt = g["w"][None, :] * (g["H"][:, None] / 2.0)
    mp = MeshProblem(3, K, p, p + 1, "stiffness", knots=g["knots"])
    assert mp.jac == 1.0
    assert mp.tables_v.cpu().numpy().tobytes() == g["V"].tobytes()
    assert mp.tables_d.cpu().numpy().tobytes() == g["D"].tobytes()
    assert mp.elem_weights.cpu().numpy().tobytes() == wt.tobytes()
    # the separable path's K1 + band launch writes the same tables and weights
    mp.tables_v.zero_()
    mp.elem_weights.zero_()
    assert mp.build_band_tables()
    assert mp.tables_v.cpu().numpy().tobytes() == g["V"].tobytes()
    assert mp.elem_weights.cpu().numpy().tobytes() == wt.tobytes()


@pytest.mark.parametrize("K,p", CASES)
@pytest.mark.parametrize("op", ["mass", "stiffness", "stiffness_mass"])
def test_general_knot_matrices_vs_reference(pkg, K, p, op):
    g = load_golden(f"nonuniform_K{K}_p{p}")
    t = g["knots"]
    _, _, A = O.integrate_assemble(3, K, p, op, "classical", knots=t, absolute=True)
    paths = [("classical", "auto"), ("sumfact", "owner"), ("sumfact", "scatter"),
             ("sumfact", "separable")]
    for method, assembly in paths:
        res = pkg.run_integration(pkg.RunConfig(method, "device", K, p, operator=op, knots=t,
                                                assembly=assembly))
        m = res.gram.matrix
        assert np.array_equal(m.indptr, g["indptr"]) and np.array_equal(m.indices, g["indices"])
        assert_parity(m.data, g[f"{op}_classical"], g["indptr"], absref=A,
                      config=f"general knots {op} K={K} p={p}", path=f"{method}/{assembly}",
                      what=f"{op} K={K} p={p} {method}/{assembly}")


@pytest.mark.parametrize("K,p,op", [(6, 3, "stiffness_mass"), (5, 2, "mass"), (4, 4, "stiffness")])
def test_general_knot_coefficient_field_vs_oracle(pkg, K, p, op):
    """Per-point coefficient on a general knot vector: the assembled kernels form W per
    element column from the per-element weights (p = 3: the DMMA pipeline kernel)."""
    q = p + 1
    rng = np.random.default_rng(K + p)
    h = rng.uniform(0.5, 1.5, size=K)
    t = np.concatenate([np.zeros(p + 1), np.cumsum(h)[:-1] / h.sum(), np.ones(p + 1)])
    coef = rng.uniform(0.5, 1.5, size=(K**3, q**3))
    ip, _, ref = O.integrate_assemble(3, K, p, op, "classical", coef=coef, knots=t)
    _, _, A = O.integrate_assemble(3, K, p, op, "classical", coef=coef, knots=t, absolute=True)
    for method, assembly in (("sumfact", "owner"), ("classical", "auto"), ("sumfact", "scatter")):
        res = pkg.run_integration(pkg.RunConfig(method, "device", K, p, operator=op,
                                                coefficient=coef, knots=t, assembly=assembly))
        assert_parity(res.gram.values.cpu().numpy(), ref, ip, absref=A,
                      config=f"general knots coef field {op} K={K} p={p}",
                      path=f"{method}/{assembly}")


@pytest.mark.parametrize("op", ["mass", "stiffness", "stiffness_mass"])
def test_general_knot_element_api_bitwise(pkg, op):
    """integrate_element_* on a general KnotVector with its knot_rule (nodes in the span,
    weights w h/2, jacobian 1): bitwise equal to the oracle's element on the same knots."""
    g = load_golden("nonuniform_K4_p3")
    kv = pkg.make_general_knot_vector(g["knots"], 3)
    assert not kv.is_uniform
    for alpha in ((0, 3, 1), (2, 2, 0)):
        rule = pkg.default_rule(kv, alpha)
        assert rule.jacobian == 1.0
        a = pkg.integrate_element_classical(alpha, kv, rule, operator=op)
        b = pkg.integrate_element_sumfact(alpha, kv, rule, pkg.SumFactBuffers.allocate(3),
                                          operator=op)
        assert a.entries.tobytes() == O.element(3, 4, 3, op, "classical", alpha,
                                                knots=g["knots"]).tobytes()
        assert b.entries.tobytes() == O.element(3, 4, 3, op, "sumfact", alpha,
                                                knots=g["knots"]).tobytes()


def test_general_knot_basis_api(pkg):
    """eval_nonzero_basis / derivatives and basis tables on a general KnotVector agree
    bitwise with the reference's eval_basis (values) and with the K1 tables (mapped nodes)."""
    g = load_golden("nonuniform_K5_p2")
    kv = pkg.make_general_knot_vector(g["knots"], 2)
    for e in range(5):
        V = pkg.basis_value_table(kv, e, g["X"][e])
        D = pkg.basis_derivative_table(kv, e, g["X"][e])
        assert V.tobytes() == np.ascontiguousarray(g["V"][e]).tobytes()
        assert D.tobytes() == np.ascontiguousarray(g["D"][e]).tobytes()
        assert pkg.find_element(kv, float(g["X"][e][1])) == e
    eb = load_golden("eval_basis")
    kv2 = pkg.KnotVector(degree=3, elements=5, knots=eb["n_K5_p3_knots"])
    xs = eb["n_K5_p3_x"]
    for x in xs[::5]:
        e = pkg.find_element(kv2, float(x))
        bv = pkg.eval_nonzero_basis(kv2, e, float(x))
        assert np.array_equal(bv.values, eb["n_K5_p3_q3"][e:e + 4, list(xs).index(x)])


def test_general_knot_multi_device_and_apply(pkg):
    """The same general-knot matrix through run_integration(devices=2) slabs and the
    matrix-free apply M x + S x against the assembled SpMV."""
    import torch

    g = load_golden("nonuniform_K6_p3")
    t = g["knots"]
    K, p = 6, 3
    one = pkg.run_integration(pkg.RunConfig("sumfact", "device", K, p, operator="stiffness_mass",
                                            knots=t, assembly="owner"))
    two = pkg.run_integration(pkg.RunConfig("sumfact", "device", K, p, operator="stiffness_mass",
                                            knots=t, assembly="owner", devices=2),
                              device_ids=[0, 0], exchange="copy")
    ip, _ = O.pattern(3, K, p)
    assert_parity(two.gram.host_values(), one.gram.values.cpu().numpy(), ip,
                  config="general knots devices=2", path="sumfact/owner")
    op = pkg.MatrixFreeOperator(K, p, knots=t)
    x = np.random.default_rng(0).standard_normal(op.n_dofs)
    y = op.apply(x, 1.0, 1.0)
    y_ref = one.gram.matrix @ x
    assert np.abs(y - y_ref).max() <= 1e-12 * np.abs(y_ref).max()
    torch.cuda.synchronize()

"""Degrees 6..9 (the paper's p = 9 Gram; the reference integrates any
p, integrators.py:77-151): K1 tables bitwise, an element matrix whose sum-factorization
stages live in global scratch (p = 7) bitwise, and global matrices through every path
that serves high degrees (separable, classical DMMA with several CTAs per element,
element-local sum factorization with global stage buffers) against the reference's
run_integration Grams and the oracle."""

import numpy as np
import pytest

from oracle import oracle as O
from tests.conftest import load_golden
from tests.parity import assert_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2207_00280_b200 as P

    return P


@pytest.mark.parametrize("K,p", [(3, 6), (2, 7), (2, 8), (3, 9)])
def test_high_degree_tables_bitwise(pkg, K, p):
    from paper_2207_00280_b200.device import MeshProblem

    g = load_golden("high_degree")
    mp = MeshProblem(3, K, p, p + 1, "stiffness")
    mp.build_tables()
    assert mp.tables_v.cpu().numpy().tobytes() == g[f"V_K{K}_p{p}"].tobytes()
    assert mp.tables_d.cpu().numpy().tobytes() == g[f"D_K{K}_p{p}"].tobytes()
    # the separable path's K1 (with the band matrices) gives the same tables
    mp.tables_v.zero_()
    assert mp.build_band_tables()
    assert mp.tables_v.cpu().numpy().tobytes() == g[f"V_K{K}_p{p}"].tobytes()


def test_high_degree_element_global_scratch_bitwise(pkg):
    """p = 7: the m^4 q stage buffer (262 KB) exceeds shared memory; the strict kernel runs
    it from stream-ordered global scratch, bitwise equal to integrate_element_sumfact."""
    g = load_golden("high_degree")
    kv = pkg.make_knot_vector(2, 7)
    alpha = (1, 0, 1)
    em = pkg.integrate_element_sumfact(alpha, kv, pkg.gauss_rule(7, 2, alpha),
                                       pkg.SumFactBuffers.allocate(7))
    assert em.entries.tobytes() == g["element_sumfact_K2_p7"].tobytes()


@pytest.mark.parametrize("K,p", [(2, 6), (1, 7)])
@pytest.mark.parametrize("method,assembly", [("sumfact", "auto"), ("sumfact", "scatter"),
                                             ("classical", "auto")])
def test_high_degree_gram_vs_reference(pkg, K, p, method, assembly):
    g = load_golden(f"mass_sumfact_K{K}_p{p}")
    res = pkg.run_integration(pkg.RunConfig(method, "device", K, p, assembly=assembly))
    m = res.gram.matrix
    assert np.array_equal(m.indptr, g["indptr"]) and np.array_equal(m.indices, g["indices"])
    assert_parity(m.data, g["data"], g["indptr"], config=f"high degree mass K={K} p={p}",
                  path=f"{method}/{assembly}", strict=True)


@pytest.mark.parametrize("K,p,op", [(2, 6, "stiffness"), (2, 7, "stiffness_mass")])
def test_high_degree_coefficient_field_vs_oracle(pkg, K, p, op):
    q = p + 1
    coef = np.random.default_rng(p).uniform(0.5, 1.5, size=(K**3, q**3))
    ip, _, ref = O.integrate_assemble(3, K, p, op, "classical", coef=coef)
    _, _, A = O.integrate_assemble(3, K, p, op, "classical", coef=coef, absolute=True)
    for method in ("sumfact", "classical"):
        res = pkg.run_integration(pkg.RunConfig(method, "device", K, p, operator=op,
                                                coefficient=coef))
        assert_parity(res.gram.values.cpu().numpy(), ref, ip, absref=A,
                      config=f"high degree {op} K={K} p={p} coef field", path=method)


def test_p9_gram_paths_agree(pkg):
    """p = 9 on a 4^3 mesh (the paper's degree): separable, classical and element-local sum
    factorization give the same Gram; it sums to 1 (partition of unity) and sampled rows
    match the oracle's classical rows."""
    K, p = 4, 9
    grams = {}
    for method, assembly in (("sumfact", "auto"), ("classical", "auto"), ("sumfact", "scatter")):
        res = pkg.run_integration(pkg.RunConfig(method, "device", K, p, assembly=assembly))
        grams[(method, assembly)] = res.gram.values.cpu().numpy()
    ip, _ = O.pattern(3, K, p)
    base = grams[("sumfact", "auto")]
    assert abs(base.sum() - 1.0) < 1e-12
    for k, v in grams.items():
        assert_parity(v, base, ip, config="p9 K=4 mass", path=f"{k[0]}/{k[1]} vs separable")
    N = K + p
    rows = [0, N**3 - 1, (N // 2 * N + N // 2) * N + N // 2, (3 * N + 1) * N + 7]
    ref_rows = O.rows(3, K, p, rows, "mass", "classical")
    got = np.concatenate([base[ip[r]:ip[r + 1]] for r in rows])
    sub = np.concatenate([[0], np.cumsum([len(x) for x in ref_rows])])
    assert_parity(got, np.concatenate(ref_rows), sub, config="p9 K=4 mass sampled rows",
                  path="sumfact/auto", strict=True)


def test_high_degree_owner_rejected(pkg):
    with pytest.raises(ValueError):
        pkg.run_integration(pkg.RunConfig("sumfact", "device", 2, 6, assembly="owner"))
    with pytest.raises(ValueError):  # q outside {p+1, p+2} at high degree
        pkg.run_integration(pkg.RunConfig("classical", "device", 2, 6, quad_points=5))

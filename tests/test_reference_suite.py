"""The reference's own per-element test cases (igabench tests/test_integrators.py),
restated against the drop-in API: the same inputs and assertions, with the element
matrices computed by the CUDA path (``iga_element_matrices``) instead of numba.

Kernel-free cases (the operation-count model, argument validation) run on CPU;
the rest are ``gpu``-marked.  Cited lines are in
/root/reference/pkg/tests/test_integrators.py."""

import numpy as np
import pytest

import paper_2207_00280_b200 as P


def _two_methods(K, p, alpha):
    """Classical and sum-factorization element matrices of one element
    (the reference's helper, test_integrators.py:16-21)."""
    kv = P.make_knot_vector(K, p)
    rule = P.gauss_rule(p, K, alpha)
    a = P.integrate_element_classical(alpha, kv, rule)
    b = P.integrate_element_sumfact(alpha, kv, rule, P.SumFactBuffers.allocate(p))
    return a, b


# ----------------------------------------------------------------- CPU: counts, validation
def test_classical_count_example_p0():
    """test_integrators.py:234-235: one pair, one point."""
    assert P.flop_count("classical", 0) == 10


def test_classical_count_ratio_tends_to_ninth_power():
    """test_integrators.py:238-241: the classical count grows like (p+1)^9."""
    for p in (6, 8, 10):
        ratio = P.flop_count("classical", p) / P.flop_count("classical", p - 1)
        assert ratio == pytest.approx(((p + 1) / p) ** 9, rel=2e-3)


def test_sumfact_cheaper_and_ratio_at_p9():
    """test_integrators.py:244-247."""
    for p in range(1, 10):
        assert P.flop_count("sumfact", p) < P.flop_count("classical", p)
    assert P.flop_count("classical", 9) / P.flop_count("sumfact", 9) >= 10


def test_unknown_method_rejected():
    """test_integrators.py:255-257."""
    with pytest.raises(ValueError):
        P.flop_count("magic", 2)


def test_buffer_shape_mismatch_rejected():
    """test_integrators.py:135-139: buffers for another degree -> ValueError, before
    any device work."""
    kv = P.make_knot_vector(2, 2)
    rule = P.gauss_rule(2, 2, (0, 0, 0))
    with pytest.raises(ValueError):
        P.integrate_element_sumfact((0, 0, 0), kv, rule, P.SumFactBuffers.allocate(1))


def test_inconsistent_inputs_rejected():
    """test_integrators.py:142-146: nodes of another element -> ValueError."""
    kv = P.make_knot_vector(2, 2)
    rule = P.gauss_rule(2, 2, (1, 1, 1))
    with pytest.raises(ValueError):
        P.integrate_element_classical((0, 0, 0), kv, rule)


# ----------------------------------------------------------------- GPU: element matrices
@pytest.mark.gpu
def test_p0_unit_cube_volume():
    """test_integrators.py:24-28."""
    a, b = _two_methods(1, 0, (0, 0, 0))
    assert a.entries.shape == (1, 1)
    assert a.entries[0, 0] == pytest.approx(1.0, abs=1e-14)
    assert b.entries[0, 0] == pytest.approx(1.0, abs=1e-14)


@pytest.mark.gpu
def test_k1_p1_analytic_mass_matrix():
    """test_integrators.py:31-38: the element matrix is the Kronecker cube of the 1D
    hat-function mass matrix [[1/3, 1/6], [1/6, 1/3]]."""
    a, _ = _two_methods(1, 1, (0, 0, 0))
    m1 = np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
    assert np.abs(a.entries - np.kron(np.kron(m1, m1), m1)).max() < 1e-12
    assert a.entries[0, 0] == pytest.approx(1 / 27, abs=1e-12)
    assert a.entries[0, 7] == pytest.approx((1 / 6) ** 3, abs=1e-12)


@pytest.mark.gpu
def test_k2_p1_corner_diagonal():
    """test_integrators.py:41-44: each supported 1D hat has mass h/3 = 1/6 at h = 1/2."""
    a, _ = _two_methods(2, 1, (0, 0, 0))
    assert a.entries[0, 0] == pytest.approx((1 / 6) ** 3, abs=1e-12)


@pytest.mark.gpu
def test_sumfact_equals_classical_entrywise():
    """test_integrators.py:47-50."""
    a, b = _two_methods(1, 1, (0, 0, 0))
    assert np.abs(a.entries - b.entries).max() < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("p", [0, 1, 2, 3])
@pytest.mark.parametrize("K", [1, 2])
def test_oracle_equivalence_small_grid(p, K):
    """test_integrators.py:53-61: both methods on every element of small meshes."""
    kv = P.make_knot_vector(K, p)
    buffers = P.SumFactBuffers.allocate(p)
    for alpha in P.element_list(K):
        rule = P.gauss_rule(p, K, alpha)
        a = P.integrate_element_classical(alpha, kv, rule).entries
        b = P.integrate_element_sumfact(alpha, kv, rule, buffers).entries
        assert np.linalg.norm(a - b) / np.linalg.norm(a) <= 1e-10


@pytest.mark.gpu
def test_fine_quadrature_oracle():
    """test_integrators.py:64-91: the integrand checked by a richer Gauss rule (q = p+3)
    evaluated here with numpy and the spline API, independent of the kernels."""
    K, p, alpha = 2, 2, (1, 0, 1)
    kv = P.make_knot_vector(K, p)
    q = p + 3
    xr, wr = np.polynomial.legendre.leggauss(q)
    h = 1.0 / K
    tabs = []
    for d in range(3):
        xs = alpha[d] * h + (xr + 1.0) * h / 2.0
        tabs.append(np.array([P.eval_nonzero_basis(kv, alpha[d], x).values for x in xs]).T)
    m = p + 1
    per_axis = [np.einsum("k,ik,jk->ij", wr, t, t) for t in tabs]  # 1D element matrices
    expected = np.einsum("ad,be,cf->abcdef", *per_axis).reshape(m**3, m**3) * (h / 2.0) ** 3
    a = P.integrate_element_classical(alpha, kv, P.gauss_rule(p, K, alpha)).entries
    assert np.abs(a - expected).max() < 1e-13


@pytest.mark.gpu
def test_exact_symmetry():
    """test_integrators.py:94-98: both triangles written from one value (bitwise)."""
    for K, p in [(2, 1), (2, 2), (3, 3)]:
        a, b = _two_methods(K, p, (K - 1, 0, 1 % K))
        assert np.array_equal(a.entries, a.entries.T)
        assert np.array_equal(b.entries, b.entries.T)


@pytest.mark.gpu
def test_positive_diagonal():
    """test_integrators.py:101-104."""
    a, b = _two_methods(3, 2, (1, 2, 0))
    assert np.all(np.diag(a.entries) > 0)
    assert np.all(np.diag(b.entries) > 0)


@pytest.mark.gpu
def test_element_matrices_translated_in_the_interior():
    """test_integrators.py:107-121: interior elements share one matrix, the corner
    element (boundary knots, p >= 2) differs."""
    K, p = 6, 2
    kv = P.make_knot_vector(K, p)
    buffers = P.SumFactBuffers.allocate(p)
    mats = [P.integrate_element_sumfact((e, e, e), kv, P.gauss_rule(p, K, (e, e, e)), buffers).entries
            for e in range(p, K - p)]
    for mt in mats[1:]:
        assert np.abs(mt - mats[0]).max() < 1e-15
    corner = P.integrate_element_sumfact((0, 0, 0), kv, P.gauss_rule(p, K, (0, 0, 0)),
                                         buffers).entries
    assert np.abs(corner - mats[0]).max() > 1e-6


@pytest.mark.gpu
def test_all_elements_equal_for_p1():
    """test_integrators.py:124-132: p = 1 has no boundary effect."""
    K, p = 3, 1
    kv = P.make_knot_vector(K, p)
    ref = None
    for alpha in P.element_list(K):
        mt = P.integrate_element_classical(alpha, kv, P.gauss_rule(p, K, alpha)).entries
        ref = mt if ref is None else ref
        assert np.abs(mt - ref).max() < 1e-15


@pytest.mark.gpu
def test_sumfact_flops_beat_classical_on_real_element():
    """test_integrators.py:250-252: the ElementMatrix carries the reference's op model."""
    a, b = _two_methods(2, 3, (1, 0, 1))
    assert b.flops < a.flops
    assert a.flops == P.flop_count("classical", 3) and b.flops == P.flop_count("sumfact", 3)


# ----------------------------------------------------------------- mesh (tests/test_mesh.py)
def test_element_list_and_support():
    """test_mesh.py:7-40: lexicographic element ids, support sets."""
    assert P.element_list(1) == [(0, 0, 0)]
    ids = P.element_list(2)
    assert len(ids) == 8 and ids[0] == (0, 0, 0) and ids[-1] == (1, 1, 1) and ids == sorted(ids)
    assert len(P.element_list(20)) == 8000
    with pytest.raises(ValueError):
        P.element_list(0)
    assert set(P.support_set((0, 0, 0), 1)) == {(a, b, c) for a in (0, 1) for b in (0, 1)
                                                for c in (0, 1)}
    assert P.support_set((0, 0, 0), 0) == [(0, 0, 0)]
    s = P.support_set((1, 1, 1), 2)
    assert len(s) == 27 and set(s) == {(a, b, c) for a in (1, 2, 3) for b in (1, 2, 3)
                                       for c in (1, 2, 3)}


def test_local_index():
    """test_mesh.py:43-58."""
    assert P.local_index((0, 0, 0), (0, 0, 0), 1) == 0
    assert P.local_index((0, 0, 0), (1, 1, 1), 1) == 7
    assert P.local_index((2, 3, 4), (3, 4, 5), 2) == 13
    for p in (0, 1, 2, 3):
        hits = [P.local_index((1, 0, 2), b, p) for b in P.support_set((1, 0, 2), p)]
        assert sorted(hits) == list(range((p + 1) ** 3))
    with pytest.raises(ValueError):
        P.local_index((0, 0, 0), (2, 0, 0), 1)


def test_gauss_rules():
    """test_mesh.py:61-109: midpoint rule, the 2-point nodes against a Newton solve of
    P2, unit integral, polynomial exactness, constant Jacobian."""
    r = P.gauss_rule(0, 2, (1, 0, 1))
    assert r.points_per_direction == (1, 1, 1)
    assert r.nodes[0][0] == pytest.approx(0.75) and r.nodes[1][0] == pytest.approx(0.25)
    for d in range(3):
        assert r.weights[d].sum() * (1 / (2 * 2)) == pytest.approx(0.5)
    x = 0.5
    for _ in range(60):
        x -= (1.5 * x * x - 0.5) / (3.0 * x)
    r = P.gauss_rule(1, 1, (0, 0, 0))
    assert np.allclose(np.sort((r.nodes[0] - 0.5) * 2.0), [-x, x], atol=1e-14)
    assert np.allclose(r.weights[0], [1.0, 1.0])
    for p, K in [(0, 1), (1, 2), (2, 3), (4, 2)]:
        for alpha in [(0, 0, 0), (K - 1, K - 1, K - 1)]:
            r = P.gauss_rule(p, K, alpha)
            tot = r.weights[0].sum() * r.weights[1].sum() * r.weights[2].sum() * r.jacobian
            assert tot == pytest.approx((1 / K) ** 3, rel=1e-13)
    for p, K in [(0, 2), (1, 2), (3, 4), (5, 3)]:
        alpha = (1, 0, K - 1)
        r = P.gauss_rule(p, K, alpha)
        for deg in range(2 * p + 2):
            for ax in range(3):
                lo, hi = alpha[ax] / K, (alpha[ax] + 1) / K
                exact = (hi ** (deg + 1) - lo ** (deg + 1)) / (deg + 1)
                assert (r.weights[ax] * r.nodes[ax] ** deg).sum() / (2 * K) == pytest.approx(
                    exact, abs=1e-12)
    assert {P.gauss_rule(2, 4, a).jacobian for a in P.element_list(4)} == {(1 / 8) ** 3}


# ----------------------------------------------------------------- splines (tests/test_splines.py)
def test_knot_vectors():
    """test_splines.py:14-43."""
    assert np.array_equal(P.make_knot_vector(1, 0).knots, [0.0, 1.0])
    assert np.allclose(P.make_knot_vector(2, 1).knots, [0, 0, 0.5, 1, 1])
    assert np.allclose(P.make_knot_vector(2, 2).knots, [0, 0, 0, 0.5, 1, 1, 1])
    for K, p in [(1, 0), (2, 1), (4, 3), (8, 5)]:
        kv = P.make_knot_vector(K, p)
        t = kv.knots
        assert len(t) == K + 2 * p + 1 and kv.n_basis == K + p and np.all(np.diff(t) >= 0)
        assert np.all(t[: p + 1] == 0.0) and np.all(t[-(p + 1):] == 1.0)
    with pytest.raises(ValueError):
        P.make_knot_vector(0, 1)
    with pytest.raises(ValueError):
        P.make_knot_vector(2, -1)


def test_find_element_and_point_checks():
    """test_splines.py:97-100, :119-122, :187-193 (host-side checks, no launch)."""
    kv = P.make_knot_vector(4, 2)
    assert P.find_element(kv, 0.0) == 0 and P.find_element(kv, 0.26) == 1
    assert P.find_element(kv, 1.0) == 3
    with pytest.raises(ValueError):
        P.find_element(kv, 1.5)
    with pytest.raises(ValueError):
        P.eval_nonzero_basis(kv, 0, 0.9)
    with pytest.raises(ValueError):
        P.eval_nonzero_basis_derivatives(P.make_knot_vector(2, 0), 0, 0.25)


@pytest.mark.gpu
def test_nonzero_basis_values_on_device():
    """test_splines.py:77-94, :138-167 through the device evaluator (K1'): linear hats,
    interpolation at both ends, partition of unity and nonnegativity on a grid."""
    kv = P.make_knot_vector(2, 1)
    assert np.allclose(P.eval_nonzero_basis(kv, 0, 0.25).values, [0.5, 0.5])
    assert np.allclose(P.eval_nonzero_basis(kv, 0, 0.0).values, [1.0, 0.0])
    for K, p in [(1, 0), (2, 1), (4, 3)]:
        kv = P.make_knot_vector(K, p)
        at0 = P.eval_nonzero_basis(kv, 0, 0.0).values
        at1 = P.eval_nonzero_basis(kv, K - 1, 1.0).values
        assert at0[0] == pytest.approx(1.0) and (p == 0 or at0[1:].max() == 0.0)
        assert at1[-1] == pytest.approx(1.0) and (p == 0 or at1[:-1].max() == 0.0)
    grid = np.linspace(0.0, 1.0, 21)
    for p in range(6):
        for K in (1, 3, 8):
            kv = P.make_knot_vector(K, p)
            for x in grid:
                v = P.eval_nonzero_basis(kv, P.find_element(kv, x), x).values
                assert v.min() >= 0.0 and abs(v.sum() - 1.0) < 1e-12


@pytest.mark.gpu
def test_nonzero_basis_derivatives_on_device():
    """test_splines.py:103-135, :170-184: hat slopes, zero sum, central differences."""
    kv = P.make_knot_vector(2, 1)
    for x in (0.1, 0.25, 0.4):
        assert np.allclose(P.eval_nonzero_basis_derivatives(kv, 0, x), [-2.0, 2.0])
    rng = np.random.default_rng(7)
    for K, p in [(2, 1), (3, 2), (5, 4)]:
        kv = P.make_knot_vector(K, p)
        for _ in range(5):
            e = int(rng.integers(K))
            x = (e + rng.random()) / K
            assert abs(P.eval_nonzero_basis_derivatives(kv, e, x).sum()) < 1e-10
    h = 1e-6
    rng = np.random.default_rng(11)
    for K, p in [(2, 1), (4, 2), (5, 3)]:
        kv = P.make_knot_vector(K, p)
        for _ in range(10):
            e = int(rng.integers(K))
            x = (e + 0.2 + 0.6 * rng.random()) / K
            ana = P.eval_nonzero_basis_derivatives(kv, e, x)
            fd = (P.eval_nonzero_basis(kv, e, x + h).values
                  - P.eval_nonzero_basis(kv, e, x - h).values) / (2 * h)
            assert np.abs(ana - fd).max() / max(1.0, np.abs(ana).max()) < 1e-5


# ----------------------------------------------------------------- assembly (assembly.py:46-83)
def test_assemble_rejects_bad_element_sets():
    """assemble's input checks (assembly.py:56-63, :73-74), before any device work:
    empty, incomplete and duplicated element sets, wrong element-matrix shapes."""
    K, p = 2, 1
    n = (p + 1) ** 3
    mat = P.ElementMatrix(element=(0, 0, 0), n=n, entries=np.eye(n), flops=0)
    full = [(a, mat) for a in P.element_list(K)]
    with pytest.raises(ValueError, match="cover"):
        P.assemble([], K, p)
    with pytest.raises(ValueError, match="cover"):
        P.assemble(full[:-1], K, p)
    with pytest.raises(ValueError, match="duplicate"):
        P.assemble(full + full[:1], K, p)
    bad = P.ElementMatrix(element=(0, 0, 0), n=n + 1, entries=np.eye(n + 1), flops=0)
    with pytest.raises(ValueError, match="shape"):
        P.assemble([(full[0][0], bad)] + full[1:], K, p)


@pytest.mark.gpu
def test_empty_ranges_through_the_abi():
    """Degenerate calls of the C-ABI: an empty row-plane range writes nothing, an empty
    element slab zeroes the rows it owns (every method), zero element matrices and an
    empty pattern range are no-ops."""
    import ctypes

    import torch

    from paper_2207_00280_b200 import _lib
    from paper_2207_00280_b200.device import MeshProblem

    L = _lib.load()
    K, p = 4, 2
    mp = MeshProblem(3, K, p, p + 1, "stiffness", None)
    v = torch.full((mp.nnz(),), 7.0, dtype=torch.float64, device="cuda")
    s = mp.problem_struct()
    for method in (0, 1, 2, 3):
        assert L.iga_integrate_assemble(ctypes.byref(s), method, 0, K, 3, 3, v.data_ptr(), None) == 0
        torch.cuda.synchronize()
        assert (v == 7.0).all().item()
    for method in (0, 1, 2, 3):
        v.fill_(7.0)
        assert L.iga_integrate_assemble(ctypes.byref(s), method, 2, 2, 0, K + p, v.data_ptr(), None) == 0
        torch.cuda.synchronize()
        assert (v == 0.0).all().item(), method
    out = torch.full((1,), 3.0, dtype=torch.float64, device="cuda")
    ids = torch.zeros((1, 3), dtype=torch.int32, device="cuda")
    assert L.iga_element_matrices(ctypes.byref(s), 0, mp.ref_nodes.data_ptr(), ids.data_ptr(), None,
                                  None, None, 0, out.data_ptr(), None) == 0
    torch.cuda.synchronize()
    assert out.item() == 3.0
    ip = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    assert L.iga_csr_pattern(3, K, p, 5, 5, ip.data_ptr(), None, None) == 0
    torch.cuda.synchronize()
    assert ip.item() in (-1, 0)

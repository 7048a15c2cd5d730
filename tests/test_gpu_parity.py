"""GPU parity: the CUDA path (through the C-ABI) against the reference goldens
and the CPU oracle.  Run on a B200 with ``pytest -m gpu``."""

import glob
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.conftest import GOLDEN, load_golden
from tests.parity import assert_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_2207_00280_b200 as P

    return P


def _gram_csr(res):
    m = res.gram.matrix
    return np.asarray(m.indptr, np.int64), np.asarray(m.indices, np.int64), m.data


# ---------------------------------------------------------------- K1 tables
def test_mesh_tables_bitwise(pkg):
    from paper_2207_00280_b200.device import MeshProblem

    g = load_golden("tables")
    n = 0
    for key in g.files:
        if not key.startswith("V_"):
            continue
        _, K, p, q = key.split("_")
        K, p, q = int(K[1:]), int(p[1:]), int(q[1:])
        if q > 8:
            continue
        mp = MeshProblem(3, K, p, q)
        V = mp.tables_v.cpu().numpy()
        D = mp.tables_d.cpu().numpy()
        assert V.tobytes() == g[key].tobytes(), key
        assert D.tobytes() == g["D" + key[1:]].tobytes(), key
        n += 1
    assert n >= 40


def test_basis_value_table_api(pkg):
    g = load_golden("tables")
    kv = pkg.make_knot_vector(5, 3)
    ref, _ = np.polynomial.legendre.leggauss(4)
    h = 1.0 / 5
    for e in range(5):
        nodes = e * h + (ref + 1.0) * (h / 2.0)
        assert pkg.basis_value_table(kv, e, nodes).tobytes() == g["V_K5_p3_q4"][e].tobytes()
        assert pkg.basis_derivative_table(kv, e, nodes).tobytes() == g["D_K5_p3_q4"][e].tobytes()


# ---------------------------------------------------------------- K5 pattern
@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "pattern_*.npz"))))
def test_pattern(pkg, path):
    K, p = (int(s[1:]) for s in os.path.basename(path)[:-4].split("_")[1:])
    g = np.load(path)
    pat = pkg.symbolic_pattern(K, p)
    assert np.array_equal(pat.indptr, g["indptr"]) and np.array_equal(pat.indices, g["indices"])


def test_pattern_row_ranges(pkg):
    from paper_2207_00280_b200.device import csr_pattern

    for dim, K, p in ((3, 7, 3), (2, 9, 2), (3, 4, 5)):
        full_ip, full_ix = O.pattern(dim, K, p)
        nr = (K + p) ** dim
        for lo, hi in ((0, nr), (3, nr // 2), (nr // 3, nr)):
            pat = csr_pattern(dim, K, p, lo, hi)
            ip = pat.indptr.cpu().numpy()
            ix = pat.indices.cpu().numpy()
            assert np.array_equal(ip, full_ip[lo:hi + 1] - full_ip[lo])
            assert np.array_equal(ix, full_ix[full_ip[lo]:full_ip[hi]])


# ------------------------------------------------------- per-element API
def test_element_matrices_bitwise(pkg):
    g = load_golden("element_mass")
    for key in g.files:
        method, K, p, *alpha = key.split("_")
        K, p = int(K[1:]), int(p[1:])
        alpha = tuple(map(int, alpha))
        kv = pkg.make_knot_vector(K, p)
        rule = pkg.gauss_rule(p, K, alpha)
        if method == "classical":
            em = pkg.integrate_element_classical(alpha, kv, rule)
        else:
            em = pkg.integrate_element_sumfact(alpha, kv, rule, pkg.SumFactBuffers.allocate(p))
        assert em.entries.tobytes() == g[key].tobytes(), key
        assert em.flops == pkg.flop_count(method, p)


@pytest.mark.parametrize("op", ["stiffness", "stiffness_mass"])
@pytest.mark.parametrize("method", ["classical", "sumfact"])
def test_element_stiffness_bitwise_vs_oracle(pkg, op, method):
    K, p = 4, 3
    kv = pkg.make_knot_vector(K, p)
    for alpha in ((0, 0, 0), (1, 3, 2)):
        rule = pkg.gauss_rule(p, K, alpha)
        if method == "classical":
            em = pkg.integrate_element_classical(alpha, kv, rule, operator=op)
        else:
            em = pkg.integrate_element_sumfact(alpha, kv, rule, pkg.SumFactBuffers.allocate(p),
                                               operator=op)
        ref = O.element(3, K, p, op, method, alpha)
        assert em.entries.tobytes() == ref.tobytes()


def test_element_fine_quadrature(pkg):
    """q = p+3 (default_rule override, test_integrators.py:64-91 shape)."""
    K, p = 3, 2
    kv = pkg.make_knot_vector(K, p)
    alpha = (1, 0, 2)
    rule = pkg.default_rule(kv, alpha, points=p + 3)
    em = pkg.integrate_element_classical(alpha, kv, rule)
    ref = O.element(3, K, p, "mass", "classical", alpha, q=p + 3)
    assert em.entries.tobytes() == ref.tobytes()


# ------------------------------------------------ mesh-wide integrate+assemble
MASS = sorted(glob.glob(os.path.join(GOLDEN, "mass_classical_K*_p*.npz")))


@pytest.mark.parametrize("path", MASS)
@pytest.mark.parametrize("method,assembly", [("classical", "auto"), ("sumfact", "owner"),
                                             ("sumfact", "scatter"), ("sumfact", "separable")])
def test_run_integration_mass_vs_reference(pkg, path, method, assembly):
    K, p = (int(s[1:]) for s in os.path.basename(path)[:-4].split("_")[2:])
    g = np.load(path)
    res = pkg.run_integration(pkg.RunConfig(method, "device", K, p, assembly=assembly))
    ip, ix, v = _gram_csr(res)
    assert np.array_equal(ip, g["indptr"]) and np.array_equal(ix, g["indices"])
    assert_parity(v, g["data"], ip, what=f"{path} {method}/{assembly}",
                  config=f"golden {os.path.basename(path)[:-4]}", path=f"{method}/{assembly}")


STIFF = sorted(glob.glob(os.path.join(GOLDEN, "stiffness*_classical_K*_p*.npz")))


@pytest.mark.parametrize("path", STIFF)
@pytest.mark.parametrize("method,assembly", [("classical", "auto"), ("sumfact", "owner"),
                                             ("sumfact", "scatter"), ("sumfact", "separable")])
def test_run_integration_stiffness_vs_reference(pkg, path, method, assembly):
    name = os.path.basename(path)[:-4]
    op = "stiffness_mass" if name.startswith("stiffness_mass") else "stiffness"
    K, p = (int(s[1:]) for s in name.split("_")[-2:])
    g = np.load(path)
    res = pkg.run_integration(pkg.RunConfig(method, "device", K, p, operator=op,
                                            assembly=assembly))
    ip, ix, v = _gram_csr(res)
    assert np.array_equal(ip, g["indptr"]) and np.array_equal(ix, g["indices"])
    assert_parity(v, g["data"], ip, what=f"{name} {method}/{assembly}", config=f"golden {name}",
                  path=f"{method}/{assembly}")


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "sepcoef_*.npz"))))
@pytest.mark.parametrize("method,assembly", [("classical", "auto"), ("sumfact", "owner")])
def test_separable_coefficient_vs_reference(pkg, path, method, assembly):
    name = os.path.basename(path)[:-4]
    op = name[len("sepcoef_"):name.rindex("_K")]
    K, p = (int(s[1:]) for s in name.split("_")[-2:])
    g = np.load(path)
    q = p + 1
    coef = np.einsum("ai,bj,ck->abcijk", g["c1"], g["c2"], g["c3"]).reshape(K**3, q**3)
    _, _, A = O.integrate_assemble(3, K, p, op, "classical", coef=coef, absolute=True)
    res = pkg.run_integration(pkg.RunConfig(method, "device", K, p, operator=op,
                                            coefficient=coef, assembly=assembly))
    ip, ix, v = _gram_csr(res)
    assert_parity(v, g["data"], ip, what=name, absref=A, config=f"golden {name}",
                  path=f"{method}/{assembly}")


@pytest.mark.parametrize("op", ["mass", "stiffness", "stiffness_mass"])
@pytest.mark.parametrize("K,p,q", [(5, 2, 3), (4, 3, 4), (3, 4, 5), (3, 1, 2), (2, 5, 6),
                                   (4, 2, 5)])
def test_general_coefficient_vs_oracle(pkg, op, K, p, q):
    if op != "mass" and p < 1:
        pytest.skip("derivatives need p >= 1")
    coef = np.random.default_rng(K * 10 + p).uniform(0.5, 1.5, size=(K**3, q**3))
    ip, _, ref = O.integrate_assemble(3, K, p, op, "classical", q=q, coef=coef)
    _, _, A = O.integrate_assemble(3, K, p, op, "classical", q=q, coef=coef, absolute=True)
    for method, assembly in (("sumfact", "owner"), ("classical", "auto"),
                             ("sumfact", "scatter")):
        res = pkg.run_integration(pkg.RunConfig(method, "device", K, p, quad_points=q,
                                                operator=op, coefficient=coef,
                                                assembly=assembly))
        v = res.gram.values.cpu().numpy()
        assert_parity(v, ref, ip, what=f"{op} K={K} p={p} q={q} {method}/{assembly}", absref=A,
                      config=f"coef field {op} K={K} p={p} q={q}", path=f"{method}/{assembly}")


@pytest.mark.parametrize("K,p", [(16, 2), (3, 1)])
def test_mass_2d_vs_derived_reference(pkg, K, p):
    """C1 (2D mass, 16^2, p=2) against the 2D Gram derived from the reference's 3D output:
    every entry within the strict per-entry 1e-12 relative bound."""
    g = load_golden(f"mass2d_K{K}_p{p}")
    res = pkg.run_integration(pkg.RunConfig("classical", "device", K, p, dim=2))
    ip, ix, v = _gram_csr(res)
    assert np.array_equal(ip, g["indptr"]) and np.array_equal(ix, g["indices"])
    assert_parity(v, g["data"], ip, config="C1" if (K, p) == (16, 2) else f"2D mass K={K} p={p}",
                  path="classical", strict=True)


def test_reference_strategies_accepted(pkg):
    """The reference's CPU strategies run the device schedule; identical bits."""
    K, p = 4, 2
    grams = [pkg.run_integration(pkg.RunConfig("sumfact", s, K, p, workers=w)).gram
             for s, w in (("sequential", 1), ("over_elements", 8), ("within_element", 4),
                          ("combined", 2), ("device", 1))]
    for g2 in grams[1:]:
        assert pkg.grams_bitwise_equal(grams[0], g2)


@pytest.mark.parametrize("method,assembly,K,coef", [
    ("sumfact", "owner", 12, False), ("sumfact", "separable", 12, False),
    ("classical", "auto", 12, False), ("sumfact", "scatter", 12, False),
    ("classical", "auto", 20, True), ("sumfact", "scatter", 20, True)])
def test_every_path_bitwise_reproducible(pkg, method, assembly, K, coef):
    """The reference promises bitwise-identical matrices for every schedule
    (runtime.py:16-20, assembly.py:1-6): two runs of every device path give the same bits,
    including the element-local classical and sum-factorization paths (colour-ordered
    scatter, no atomics)."""
    p = 3
    c = (np.random.default_rng(1).uniform(0.5, 1.5, size=(K**3, (p + 1) ** 3)) if coef else None)
    cfg = pkg.RunConfig(method, "device", K, p, operator="stiffness", repetitions=2,
                        assembly=assembly, coefficient=c)
    a = pkg.run_integration(cfg).gram
    b = pkg.run_integration(cfg).gram
    assert pkg.grams_bitwise_equal(a, b)



@pytest.mark.parametrize("method", ["assembled", "separable", "classical"])
def test_slabs_sum_to_full(pkg, method):
    """Multi-GPU decomposition emulated on one GPU: element slabs along the slowest
    axis produce partial interface rows that add up to the single-device matrix."""
    import torch
    from paper_2207_00280_b200 import _lib
    from paper_2207_00280_b200.device import MeshProblem

    code = {"assembled": _lib.METHOD_SUMFACT_ASSEMBLED, "separable": _lib.METHOD_SEPARABLE,
            "classical": _lib.METHOD_CLASSICAL}[method]
    K, p = 10, 3
    N = K + p
    mp = MeshProblem(3, K, p, operator="stiffness")
    full = torch.empty(mp.nnz(), dtype=torch.float64, device="cuda")
    mp.integrate_assemble(full, code)
    acc = torch.zeros_like(full)
    bounds = [0, 3, 5, 10]
    for g in range(3):
        lo, hi = bounds[g], bounds[g + 1]
        phi = min(hi + p, N) if g < 2 else N
        part = torch.empty(mp.nnz(lo, phi), dtype=torch.float64, device="cuda")
        mp.integrate_assemble(part, code, el_range=(lo, hi), plane_range=(lo, phi))
        off = mp.nnz(0, lo)
        acc[off:off + part.numel()] += part
    ip, _ = O.pattern(3, K, p)
    assert_parity(acc.cpu().numpy(), full.cpu().numpy(), ip)


def test_spmv_matches_scipy(pkg):
    res = pkg.run_integration(pkg.RunConfig("sumfact", "device", 6, 3, operator="stiffness"))
    x = np.random.default_rng(0).standard_normal(res.gram.n_dofs)
    y = res.gram.spmv(x)
    np.testing.assert_allclose(y, res.gram.matrix @ x, rtol=1e-13, atol=1e-15)


def test_heat_rhs_pins(pkg):
    for K, p in ((3, 2), (4, 3)):
        g = load_golden(f"heat_rhs_K{K}_p{p}")
        for op, key in (("mass", "Mmu"), ("stiffness", "Smu")):
            res = pkg.run_integration(pkg.RunConfig("sumfact", "device", K, p, operator=op))
            got = res.gram.spmv(g["mu"])
            assert np.linalg.norm(got - g[key]) <= 1e-13 * np.linalg.norm(g[key])


def test_assemble_api_from_element_matrices(pkg):
    K, p = 3, 2
    kv = pkg.make_knot_vector(K, p)
    buf = pkg.SumFactBuffers.allocate(p)
    mats = [(a, pkg.integrate_element_sumfact(a, kv, pkg.gauss_rule(p, K, a), buf))
            for a in pkg.element_list(K)]
    gram = pkg.assemble(mats, K, p)
    g = load_golden(f"mass_sumfact_K{K}_p{p}")
    ip, ix, v = _gram_csr(type("R", (), {"gram": gram}))
    assert np.array_equal(ip, g["indptr"])
    assert_parity(v, g["data"], ip)
    with pytest.raises(ValueError):
        pkg.assemble(mats[:-1], K, p)
    with pytest.raises(ValueError):
        pkg.assemble(mats + mats[:1], K, p)


# ---------------------------------------------- full-size configs, sampled rows
def _sample_rows(K, p, n_rand, seed=0):
    N = K + p
    rng = np.random.default_rng(seed)
    corners = [0, N - 1]
    special = []
    for a in corners + [p, K // 2]:
        for b in corners + [1, K // 2]:
            for c in corners + [p - 1 if p > 0 else 0, K // 2]:
                special.append((a * N + b) * N + c)
    rows = np.unique(np.concatenate([special, rng.integers(0, N**3, n_rand)]))
    return rows


@pytest.mark.parametrize("cfg", [
    dict(K=64, p=3, op="stiffness", coef=None, name="C3", assembly="owner", strict=True),
    dict(K=64, p=3, op="stiffness", coef=None, name="C3", assembly="separable", strict=True),
    dict(K=64, p=3, op="stiffness", coef=None, name="C3", method="classical", strict=True),
    dict(K=64, p=3, op="stiffness", coef=None, name="C3", assembly="scatter", strict=True),
    dict(K=32, p=2, op="mass", coef="uniform", name="C2", assembly="owner"),
    dict(K=32, p=2, op="mass", coef="uniform", name="C2", method="classical"),
    dict(K=32, p=2, op="mass", coef="uniform", name="C2", assembly="scatter"),
    dict(K=48, p=3, op="stiffness", coef="uniform", name="C3-48 coef field", method="classical"),
    dict(K=48, p=3, op="stiffness", coef="uniform", name="C3-48 coef field", assembly="owner"),
    dict(K=64, p=3, op="stiffness", coef="uniform", name="C3 coef field (bench c3f)", assembly="owner"),
])
def test_full_size_sampled_rows(pkg, cfg):
    """BASELINE configs at full size: sampled rows (corner/edge/interior) vs the
    oracle's classical rows, plus size-independent properties."""
    K, p, op = cfg["K"], cfg["p"], cfg["op"]
    q = p + 1
    coef = None
    if cfg["coef"] == "uniform":
        coef = np.random.default_rng(42).uniform(0.5, 1.5, size=(K, K, K, q, q, q))
        coef = coef.reshape(K**3, q**3)
    res = pkg.run_integration(pkg.RunConfig(cfg.get("method", "sumfact"), "device", K, p,
                                            operator=op, coefficient=coef,
                                            assembly=cfg.get("assembly", "auto")))
    values = res.gram.values.cpu().numpy()
    ip, _ = O.pattern(3, K, p)
    rows = _sample_rows(K, p, 40)
    ref_rows = O.rows(3, K, p, rows, op, "classical", coef=coef)
    abs_rows = O.rows(3, K, p, rows, op, "classical", coef=coef, absolute=True)
    got = np.concatenate([values[ip[r]:ip[r + 1]] for r in rows])
    ref = np.concatenate(ref_rows)
    A = np.concatenate(abs_rows)
    sub_ip = np.concatenate([[0], np.cumsum([len(x) for x in ref_rows])])
    method = cfg.get("method", "sumfact")
    assert_parity(got, ref, sub_ip, absref=A, what=cfg["name"], config=cfg["name"],
                  path=f"{method}/{cfg.get('assembly', 'auto')}", strict=cfg.get("strict", False))
    # size-independent properties on the whole matrix
    M = res.gram.matrix
    # symmetric to rounding, like the reference (its own |A - A^T| reaches 4e-16 max|A|)
    assert abs(M - M.T).max() <= 1e-15 * np.abs(values).max()
    if op == "stiffness":
        rs = np.abs(M @ np.ones(M.shape[0]))
        assert rs.max() <= 1e-12 * np.abs(values).max()  # constants are in the kernel
    if op == "mass" and coef is None:
        assert abs(values.sum() - 1.0) < 1e-12


@pytest.mark.parametrize("G", [2, 3, 4])
def test_slab_sessions_emulated_ranks(pkg, G):
    """The per-rank SlabSession launches (interface planes first, then owned planes)
    for G emulated ranks on one GPU; the interface exchange is done here by copies
    (the NCCL transfer itself is covered by tests/test_distributed.py over gloo)."""
    import torch
    from paper_2207_00280_b200.distributed import SlabSession, plane_nnz, slab_plan

    K, p = 12, 3
    N = K + p
    cfg = pkg.RunConfig("sumfact", "device", K, p, operator="stiffness")
    full = pkg.run_integration(cfg).gram.values
    sessions = [SlabSession(cfg, slab_plan(K, p, G, g)) for g in range(G)]
    outs = [s.step(exchange=False) for s in sessions]
    for g in range(1, G):
        prev, cur = sessions[g - 1], sessions[g]
        send = prev.values[prev.n_own:]
        n = plane_nnz(3, K, p, *cur.plan.recv_planes)
        assert send.numel() == n
        cur.values[:n] += send
    torch.cuda.synchronize()
    got = torch.cat([s.values[:s.n_own] for s in sessions]).cpu().numpy()
    ip, _ = O.pattern(3, K, p)
    assert got.size == ip[-1]
    assert_parity(got, full.cpu().numpy(), ip)


@pytest.mark.parametrize("G,K,p,assembly,coef", [
    (2, 12, 3, "auto", False), (3, 12, 3, "auto", False), (4, 12, 3, "owner", False),
    (3, 9, 2, "auto", True), (2, 8, 4, "auto", True), (3, 12, 3, "classical", False)])
def test_slab_sessions_recompute_halo(pkg, G, K, p, assembly, coef):
    """NCCL-free ablation: each rank also integrates the p element
    layers below its slab, restricted to its owned planes; the owned rows concatenated
    over ranks equal the single-device matrix with no exchange at all."""
    import torch
    from paper_2207_00280_b200.distributed import SlabSession, slab_plan

    q = p + 1
    c = np.random.default_rng(3).uniform(0.5, 1.5, size=(K**3, q**3)) if coef else None
    method = "classical" if assembly == "classical" else "sumfact"
    asm = "auto" if assembly == "classical" else assembly
    cfg = pkg.RunConfig(method, "device", K, p, operator="stiffness_mass" if coef else "stiffness",
                        coefficient=c, assembly=asm)
    full = pkg.run_integration(cfg).gram.values
    sessions = [SlabSession(cfg, slab_plan(K, p, G, g), halo="recompute") for g in range(G)]
    outs = [s.step() for s in sessions]
    assert all(s.kernel_launches_per_step == 2 for s in sessions)
    torch.cuda.synchronize()
    got = torch.cat(outs).cpu().numpy()
    ip, _ = O.pattern(3, K, p)
    assert got.size == ip[-1]
    assert_parity(got, full.cpu().numpy(), ip)


def test_slab_session_rejects_unknown_halo(pkg):
    from paper_2207_00280_b200.distributed import SlabSession, slab_plan

    with pytest.raises(ValueError):
        SlabSession(pkg.RunConfig("sumfact", "device", 8, 2), slab_plan(8, 2, 2, 0), halo="x")


# ---------------------------------------------- §8(f): matrix-free apply, CG
@pytest.mark.parametrize("K,p,coef", [(5, 3, False), (4, 2, True), (3, 4, True), (6, 1, False)])
def test_matrix_free_apply_matches_assembled(pkg, K, p, coef):
    from paper_2207_00280_b200.operator import MatrixFreeOperator

    q = p + 1
    c = np.random.default_rng(5).uniform(0.5, 1.5, size=(K**3, q**3)) if coef else None
    op = MatrixFreeOperator(K, p, coefficient=c)
    x = np.random.default_rng(6).standard_normal(op.n_dofs)
    M = pkg.run_integration(pkg.RunConfig("sumfact", "device", K, p, coefficient=c)).gram.matrix
    S = pkg.run_integration(pkg.RunConfig("sumfact", "device", K, p, operator="stiffness",
                                          coefficient=c)).gram.matrix
    for a, b in ((1.0, 0.0), (0.0, 1.0), (1.0, -0.37)):
        got = op.apply(x, a, b)
        ref = a * (M @ x) + b * (S @ x)
        assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref), (a, b)


def test_matrix_free_heat_rhs_pins(pkg):
    from paper_2207_00280_b200.operator import MatrixFreeOperator

    for K, p in ((3, 2), (4, 3)):
        g = load_golden(f"heat_rhs_K{K}_p{p}")
        op = MatrixFreeOperator(K, p)
        for dt, ref in ((0.0, g["Mmu"]), (1.0, g["Mmu"] - g["Smu"])):
            got = op.rhs(g["mu"], dt)
            assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)


def test_cg_solves_gram_system(pkg):
    from paper_2207_00280_b200.operator import cg

    K, p = 6, 2
    gram = pkg.run_integration(pkg.RunConfig("sumfact", "device", K, p)).gram
    xs = np.random.default_rng(8).standard_normal(gram.n_dofs)
    b = gram.matrix @ xs
    x, it = cg(gram, b, rtol=1e-12)
    assert np.linalg.norm(x - xs) <= 1e-8 * np.linalg.norm(xs)


def test_cg_device_solver_reproducible_and_chunk_invariant(pkg):
    """iga_cg: bitwise-identical solutions run to run and for any host-check interval (the
    iterations launched after convergence are frozen on the device), device tensors in and
    out, and the reference's non-convergence error (scipy cg info > 0 -> RuntimeError)."""
    import torch

    from paper_2207_00280_b200.operator import MatrixFreeOperator, cg

    K, p = 7, 3
    gram = pkg.run_integration(pkg.RunConfig("sumfact", "device", K, p)).gram
    xs = np.random.default_rng(21).standard_normal(gram.n_dofs)
    b = gram.matrix @ xs
    x1, i1 = cg(gram, b, rtol=1e-12)
    x2, i2 = cg(gram, b, rtol=1e-12, check_every=1)
    x3, i3 = cg(gram, b, rtol=1e-12, check_every=64)
    assert i1 == i2 == i3 > 0
    assert np.array_equal(x1, x2) and np.array_equal(x1, x3)
    assert np.linalg.norm(x1 - xs) <= 1e-8 * np.linalg.norm(xs)
    res = np.linalg.norm(b - gram.matrix @ x1)
    assert res <= 1e-12 * np.linalg.norm(b) * 1.01
    xd, idv = cg(gram, torch.as_tensor(b).cuda(), rtol=1e-12)
    assert isinstance(xd, torch.Tensor) and xd.is_cuda and idv == i1
    assert np.array_equal(xd.cpu().numpy(), x1)
    # x0 = the solution converges in zero iterations
    x0s, i0 = cg(gram, b, x0=x1, rtol=1e-10)
    assert i0 == 0 and np.array_equal(x0s, x1)
    with pytest.raises(RuntimeError):
        cg(gram, b, rtol=1e-14, maxiter=3)
    op = MatrixFreeOperator(K, p)
    xm, im = cg(op, op.apply(xs, 1.0, 0.5), rtol=1e-12, alpha=1.0, beta=0.5)
    assert im > 0 and np.linalg.norm(xm - xs) <= 1e-8 * np.linalg.norm(xs)


def test_separable_matches_assembled_all_ops(pkg):
    """Separable (Kronecker) path vs the general assembled kernel and the oracle for
    every operator, scalar coefficient != 1, p = 0..5, q != p+1."""
    for op in ("mass", "stiffness", "stiffness_mass"):
        for K, p, q in ((5, 2, 3), (4, 3, 4), (3, 4, 6), (6, 1, 2), (2, 5, 6), (4, 0, 1), (2, 3, 4)):
            if op != "mass" and p < 1:
                continue
            cfg = dict(quad_points=q, operator=op, coefficient=1.7)
            ip, _, ref = O.integrate_assemble(3, K, p, op, "classical", q=q, coef=np.full((K**3, q**3), 1.7))
            _, _, A = O.integrate_assemble(3, K, p, op, "classical", q=q,
                                           coef=np.full((K**3, q**3), 1.7), absolute=True)
            v = pkg.run_integration(pkg.RunConfig("sumfact", "device", K, p, assembly="separable",
                                                  **cfg)).gram.values.cpu().numpy()
            assert_parity(v, ref, ip, what=f"separable {op} K={K} p={p} q={q}", absref=A)


def test_separable_rejects_field_coefficient(pkg):
    K, p = 3, 2
    coef = np.ones((K**3, (p + 1)**3))
    with pytest.raises(ValueError):
        pkg.run_integration(pkg.RunConfig("sumfact", "device", K, p, coefficient=coef,
                                          assembly="separable"))


@pytest.mark.parametrize("K,p,op", [(5, 3, "stiffness"), (7, 2, "mass")])
def test_matrix_market_export_streams_from_device(pkg, tmp_path, K, p, op):
    """write_matrix_market from device values (row-block streaming) is byte-identical
    to scipy.io.mmwrite of the same matrix (assembly.py:118-120)."""
    import io

    import scipy.io

    gram = pkg.run_integration(pkg.RunConfig("sumfact", "device", K, p, operator=op)).gram
    f = tmp_path / "g.mtx"
    pkg.write_matrix_market(gram, f)
    ref = io.BytesIO()
    scipy.io.mmwrite(ref, gram.matrix.tocoo(), symmetry="symmetric")
    assert f.read_bytes() == ref.getvalue()
    import scipy.sparse

    back = scipy.io.mmread(str(f)).tocsr()  # symmetric file: the lower triangle, mirrored
    assert abs(scipy.sparse.tril(back) - scipy.sparse.tril(gram.matrix)).max() == 0.0


def test_cg_matrix_free_implicit_heat_step(pkg):
    """(M + dt S) u = M mu solved matrix-free (separable apply) matches the assembled
    operators' solution."""
    import scipy.sparse.linalg as spla

    from paper_2207_00280_b200.operator import MatrixFreeOperator, cg

    K, p, dt = 6, 3, 0.01
    op = MatrixFreeOperator(K, p)
    mu = np.random.default_rng(9).standard_normal(op.n_dofs)
    b = op.apply(mu, 1.0, 0.0)
    x, it = cg(op, b, rtol=1e-12, alpha=1.0, beta=dt)
    M = pkg.run_integration(pkg.RunConfig("sumfact", "device", K, p, assembly="owner")).gram.matrix
    S = pkg.run_integration(pkg.RunConfig("sumfact", "device", K, p, operator="stiffness",
                                          assembly="owner")).gram.matrix
    ref = spla.spsolve((M + dt * S).tocsc(), M @ mu)
    assert np.linalg.norm(x - ref) <= 1e-9 * np.linalg.norm(ref)


def test_heat_step_matches_assembled_reference(pkg):
    """HeatProblem.step semantics (heat.py:101-107) on the device: M mu' = M mu - dt S mu."""
    import scipy.sparse.linalg as spla

    from paper_2207_00280_b200.operator import MatrixFreeOperator, heat_step

    K, p = 5, 2
    dt = (1.0 / K) ** 2 / 6.0  # heat.stable_timestep
    op = MatrixFreeOperator(K, p)
    mu = 1.0 + np.random.default_rng(4).standard_normal(op.n_dofs) * 0.1
    got = heat_step(op, mu, dt)
    M = pkg.run_integration(pkg.RunConfig("sumfact", "device", K, p, assembly="owner")).gram.matrix
    S = pkg.run_integration(pkg.RunConfig("sumfact", "device", K, p, operator="stiffness",
                                          assembly="owner")).gram.matrix
    ref = spla.spsolve(M.tocsc(), M @ mu - dt * (S @ mu))
    assert np.linalg.norm(got - ref) <= 1e-8 * np.linalg.norm(ref)
    # mass conservation with Neumann boundaries: the total integral is unchanged
    ones = np.ones(op.n_dofs)
    assert abs(ones @ (M @ got) - ones @ (M @ mu)) <= 1e-10 * abs(ones @ (M @ mu))


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("K", [1, 2])
def test_tiny_meshes_all_paths(pkg, K, p):
    """Degenerate meshes (K <= p: every row truncated on both sides) through every
    device path, every operator, against the oracle."""
    for op in ("mass", "stiffness", "stiffness_mass"):
        ip, _, ref = O.integrate_assemble(3, K, p, op, "classical")
        _, _, A = O.integrate_assemble(3, K, p, op, "classical", absolute=True)
        for method, assembly in (("sumfact", "owner"), ("sumfact", "separable"),
                                 ("sumfact", "scatter"), ("classical", "auto")):
            res = pkg.run_integration(pkg.RunConfig(method, "device", K, p, operator=op,
                                                    assembly=assembly))
            v = res.gram.values.cpu().numpy()
            assert_parity(v, ref, ip, absref=A, what=f"{op} K={K} p={p} {method}/{assembly}")


def test_bench_csv_schema(pkg):
    """Bench CSV: the reference's columns (cli.py:31) first, one row per repetition."""
    import csv
    import io

    from paper_2207_00280_b200 import benchcsv

    buf = io.StringIO()
    n = benchcsv.write_bench_csv(buf, method="both", p=2, K=6, threads=(1, 4), repeat=2)
    lines = buf.getvalue().splitlines()
    assert lines[0].startswith("#")
    rows = list(csv.reader(lines[1:]))
    assert rows[0][:8] == ["method", "strategy", "p", "K", "threads", "rep", "seconds", "flops"]
    assert len(rows) - 1 == n == 2 * 2 * 2
    assert {r[0] for r in rows[1:]} == {"classical", "sumfact"}
    assert all(float(r[6]) > 0 for r in rows[1:])


def _device_rows(values, dim, K, p, rows):
    """Values of the listed rows, sliced on the device (no host CSR for huge meshes)."""
    from paper_2207_00280_b200.device import csr_nnz

    return [values[csr_nnz(dim, K, p, 0, int(r)):csr_nnz(dim, K, p, 0, int(r) + 1)].cpu().numpy()
            for r in rows]


def _check_rows(got_rows, K, p, rows, op, coef, name, path=None, strict=False):
    ref_rows = O.rows(3, K, p, rows, op, "classical", coef=coef)
    abs_rows = O.rows(3, K, p, rows, op, "classical", coef=coef, absolute=True)
    got = np.concatenate(got_rows)
    ref = np.concatenate(ref_rows)
    A = np.concatenate(abs_rows)
    sub_ip = np.concatenate([[0], np.cumsum([len(x) for x in ref_rows])])
    name0 = name.split(" ")[0]
    assert_parity(got, ref, sub_ip, absref=A, what=name, config=name0, path=path, strict=strict)


_C4_COEF = {}


@pytest.mark.parametrize("method,assembly", [("sumfact", "owner"), ("classical", "auto"),
                                             ("sumfact", "scatter")])
def test_full_size_c4_sampled_rows(pkg, method, assembly):
    """C4 at full size (96^3, p=4, q=5, stiffness+mass, 8-mode sine field from bench.py's
    seeded generator), classical and sum factorization (BASELINE C4 compares them): sampled
    corner/edge/interior rows vs the oracle's classical rows."""
    import torch

    import bench

    K, p = 96, 4
    if "c" not in _C4_COEF:
        _C4_COEF["c"] = bench.coefficient("sines", K, p, 3)
    coef = _C4_COEF["c"]
    res = pkg.run_integration(pkg.RunConfig(method, "device", K, p, operator="stiffness_mass",
                                            coefficient=coef, assembly=assembly))
    rows = _sample_rows(K, p, 24, seed=1)
    _check_rows(_device_rows(res.gram.values, 3, K, p, rows), K, p, rows, "stiffness_mass", coef,
                f"C4 {method}/{assembly}", path=f"{method}/{assembly}")
    del res
    torch.cuda.empty_cache()


@pytest.mark.parametrize("method,assembly", [("sumfact", "separable"), ("sumfact", "owner"),
                                             ("classical", "auto"), ("sumfact", "scatter")])
def test_full_size_c5_sampled_rows(pkg, method, assembly):
    """C5 at full size on one GPU (256^3, p=3: 5.84e9 values, 46.7 GB resident): sampled
    rows, including the planes at the 2/4/8-way slab boundaries, vs the oracle; the
    stiffness row sums vanish."""
    import torch

    K, p = 256, 3
    res = pkg.run_integration(pkg.RunConfig(method, "device", K, p, operator="stiffness",
                                            assembly=assembly))
    N = K + p
    rng = np.random.default_rng(5)
    planes = [0, 1, 2, 3, 31, 32, 33, 64, 127, 128, 129, 130, 192, 255, 256, 258]
    rows = sorted({(a * N + int(rng.integers(0, N))) * N + int(rng.integers(0, N)) for a in planes}
                  | {0, N**3 - 1, (N // 2 * N + N // 2) * N + N // 2})
    got = _device_rows(res.gram.values, 3, K, p, rows)
    _check_rows(got, K, p, rows, "stiffness", None, f"C5 {method}/{assembly}",
                path=f"{method}/{assembly}", strict=True)
    for r in got:
        assert abs(r.sum()) <= 1e-12 * np.abs(r).max()
    del res
    torch.cuda.empty_cache()


def test_device_session_graph_replay_matches_eager(pkg):
    """DeviceSession(use_graph=True): the captured step (K1 + kernel) gives the same bits."""
    from paper_2207_00280_b200.runtime import DeviceSession

    cfg = pkg.RunConfig("sumfact", "device", 6, 3, operator="stiffness")
    a = DeviceSession(cfg).step().clone()
    s = DeviceSession(cfg, use_graph=True)
    for _ in range(3):
        b = s.step()
    assert (a == b).all().item()


@pytest.mark.parametrize("K,p,op,slab", [(6, 3, "stiffness", None), (64, 3, "stiffness", None),
                                         (64, 3, "stiffness", (21, 40)), (9, 1, "stiffness_mass", (2, 6)),
                                         (7, 2, "mass", None), (5, 4, "stiffness_mass", None),
                                         (4, 5, "stiffness", None), (3, 0, "mass", None),
                                         (120, 3, "stiffness", None), (120, 2, "mass", (30, 61))])
def test_separable_band_tables(pkg, K, p, op, slab):
    """iga_band_tables (K1 + the assembled 1D band matrices in one launch) and the separable
    kernel reading them (many short CTAs) against the kernel that integrates the band
    matrices in every CTA: K1 tables bitwise, CSR values bitwise where the old kernel sums
    element by element (meshes whose tables fit its shared memory), else to rounding."""
    import torch

    from paper_2207_00280_b200.device import MeshProblem

    mp = MeshProblem(3, K, p, p + 1, op, 1.3)
    mp.build_tables()
    V0, D0 = mp.tables_v.clone(), mp.tables_d.clone()
    el = (0, K) if slab is None else slab
    pl = (0, K + p) if slab is None else (slab[0], min(K + p, slab[1] + p))
    n = mp.nnz(*pl)
    a = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
    b = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
    mp.integrate_assemble(a, 3, el_range=el, plane_range=pl)
    mp.tables_v.zero_()
    mp.tables_d.zero_()
    assert mp.build_band_tables()
    assert torch.equal(mp.tables_v, V0)
    if op != "mass":
        assert torch.equal(mp.tables_d, D0)
    mp.integrate_assemble(b, 3, el_range=el, plane_range=pl, band=True)
    torch.cuda.synchronize()
    assert not torch.isnan(b).any().item()
    if K <= 64:
        assert torch.equal(a, b)
    else:
        assert torch.allclose(a, b, rtol=1e-13, atol=1e-13 * a.abs().max().item())
    del a, b
    torch.cuda.empty_cache()


@pytest.mark.parametrize("K,p,op", [(5, 3, "stiffness"), (4, 2, "mass"), (3, 4, "stiffness_mass"),
                                    (6, 1, "stiffness"), (2, 5, "mass")])
def test_writes_stay_in_bounds(pkg, K, p, op):
    """Bounds check by canaries (compute-sanitizer is unavailable on this pool): every
    method writes exactly its row range -- the NaN-prefilled range fully, the sentinel
    guard zones around it (4096 values each side) not at all -- for full meshes and
    element slabs with partial plane ranges, with and without precomputed band tables."""
    import torch

    from paper_2207_00280_b200.device import MeshProblem

    q = p + 1
    coef = np.random.default_rng(3).uniform(0.5, 1.5, size=(K**3, q**3))
    G = 4096
    for c in (None, coef):
        mp = MeshProblem(3, K, p, q, op, c)
        mp.build_tables()
        band = mp.build_band_tables()
        N = K + p
        for el, pl in (((0, K), (0, N)), ((1, K - 1), (1, min(N, K - 1 + p))), ((0, 1), (0, p + 1))):
            n = mp.nnz(*pl)
            buf = torch.full((n + 2 * G,), 12345.0, dtype=torch.float64, device="cuda")
            methods = (0, 1, 2) if c is not None else (0, 1, 2, 3)
            for method in methods:
                for use_band in ((False, True) if method == 3 and band else (False,)):
                    buf[G:G + n] = float("nan")
                    mp.integrate_assemble(buf[G:], method, el_range=el, plane_range=pl, band=use_band)
                    torch.cuda.synchronize()
                    assert (buf[:G] == 12345.0).all().item() and (buf[G + n:] == 12345.0).all().item(), \
                        (method, el, pl, use_band)
                    assert not torch.isnan(buf[G:G + n]).any().item(), (method, el, pl, use_band)


def test_spmv_staged_window_matches(pkg, monkeypatch):
    """Large meshes (N >= 160) take the SpMV with the x window staged in shared memory;
    it sums in the same order as the L1-gather kernel (IGA_SPMV_L1=1): bitwise equal."""
    import torch

    from paper_2207_00280_b200 import _lib

    K, p = 170, 3
    g = pkg.run_integration(pkg.RunConfig("sumfact", "device", K, p, operator="stiffness")).gram
    n = (K + p) ** 3
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    y1, y2 = torch.empty_like(x), torch.empty_like(x)
    L = _lib.load()
    _lib.check(L.iga_spmv(3, K, p, _lib.ptr(g.values), _lib.ptr(x), _lib.ptr(y1), _lib.stream_ptr()))
    monkeypatch.setenv("IGA_SPMV_L1", "1")
    _lib.check(L.iga_spmv(3, K, p, _lib.ptr(g.values), _lib.ptr(x), _lib.ptr(y2), _lib.stream_ptr()))
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    # and against the matrix: row sums of the stiffness matrix vanish, so A 1 = 0
    ones = torch.ones(n, dtype=torch.float64, device="cuda")
    monkeypatch.delenv("IGA_SPMV_L1")
    _lib.check(L.iga_spmv(3, K, p, _lib.ptr(g.values), _lib.ptr(ones), _lib.ptr(y1), _lib.stream_ptr()))
    torch.cuda.synchronize()
    assert y1.abs().max().item() <= 1e-12 * g.values.abs().max().item() * 343
    del g, x, y1, y2, ones
    torch.cuda.empty_cache()


@pytest.mark.parametrize("K,p,op", [(64, 3, "stiffness"), (17, 2, "mass"), (9, 4, "stiffness_mass")])
def test_band_tables_read_only_and_in_bounds(pkg, K, p, op):
    """ABI v4: iga_band_tables writes exactly (K+p)(2p+1)*2 doubles (a guard zone after them
    stays untouched), and the separable kernel only reads the band buffer -- two launches
    sharing one buffer on two streams at once both write every value, bitwise equal to a
    launch on its own."""
    import ctypes

    import torch

    from paper_2207_00280_b200 import _lib
    from paper_2207_00280_b200.device import MeshProblem

    mp = MeshProblem(3, K, p, p + 1, op, 1.3)
    nband = (K + p) * (2 * p + 1) * 2
    guard = torch.full((nband + 64,), 777.0, dtype=torch.float64, device="cuda")
    mp.band = guard[:nband]
    s = mp.problem_struct()
    _lib.check(_lib.load().iga_band_tables(ctypes.byref(s), mp.ref_nodes.data_ptr(),
                                           mp.tables_v.data_ptr(), mp.tables_d.data_ptr(),
                                           guard.data_ptr(), None, _lib.stream_ptr()))
    torch.cuda.synchronize()
    assert (guard[nband:] == 777.0).all().item()
    snapshot = guard.clone()
    n = mp.nnz(0, K + p)
    ref = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
    mp.integrate_assemble(ref, 3, band=True)
    torch.cuda.synchronize()
    outs = [torch.full((n,), float("nan"), dtype=torch.float64, device="cuda") for _ in range(2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for o, st in zip(outs, streams):
        st.wait_stream(torch.cuda.current_stream())
    for _ in range(3):
        for o, st in zip(outs, streams):
            mp.integrate_assemble(o, 3, band=True, stream=st)
    torch.cuda.synchronize()
    assert not torch.isnan(ref).any().item()
    for o in outs:
        assert torch.equal(o, ref)
    assert torch.equal(guard, snapshot)

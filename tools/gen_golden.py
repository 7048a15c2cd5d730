"""Generate the golden fixtures in tests/golden/ from the reference itself.

Run in the build container only (it imports the read-only reference at
/root/reference/pkg/src; that tree does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tools/gen_golden.py

Every array written here is an OUTPUT of the reference's public functions
(splines/mesh/integrators/assembly/runtime/heat) on seeded or fixed inputs;
nothing is restated.  Stiffness / coefficient / 2D goldens use the reference's
own numba kernels the way SURVEY.md §8(c) prescribes:
  * stiffness = classical_kernel / sumfact_kernel called once per axis with
    basis_derivative_table substituted on that axis (integrators.py:77-151,
    splines.py:173-178), summed in axis order, assembled by assembly.assemble;
  * separable coefficient c1(x)c2(y)c3(z) = per-axis weights w*c_d;
  * 2D mass = the 3D reference Gram summed over the third index pair
    (partition of unity);
  * heat.HeatProblem.assemble_rhs gives M.mu and S.mu (heat.py:131-158).
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")

import igabench  # noqa: E402
from igabench import assembly, heat, integrators, mesh, runtime, splines  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def save(name, **arrays):
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, name), **arrays)
    print("wrote", name, {k: getattr(v, "shape", v) for k, v in arrays.items()})


def mesh_tables(K, p, q):
    kv = splines.make_knot_vector(K, p)
    ref, _ = np.polynomial.legendre.leggauss(q)
    h = 1.0 / K
    V, D = [], []
    for e in range(K):
        nodes = e * h + (ref + 1.0) * (h / 2.0)  # runtime.py:147
        V.append(splines.basis_value_table(kv, e, nodes))
        if p >= 1:
            D.append(splines.basis_derivative_table(kv, e, nodes))
    V = np.array(V)
    D = np.array(D) if p >= 1 else np.zeros_like(V)
    return V, D


def ref_csr(gram):
    m = gram.matrix
    return dict(indptr=m.indptr.astype(np.int64), indices=m.indices.astype(np.int64),
                data=m.data, n=np.int64(gram.n_dofs))


def term_kernel_assemble(K, p, q, method, op, coef_axes=None):
    """Reference kernels per axis-term, summed in axis order, then reference assemble."""
    V, D = mesh_tables(K, p, q)
    rule0 = integrators.default_rule(splines.make_knot_vector(K, p), (0, 0, 0), q)
    w = rule0.weights[0]
    jac = rule0.jacobian
    m = p + 1
    n = m**3
    rows, cols = integrators.canonical_pairs(n)
    if op == "mass":
        terms = [3]
    elif op == "stiffness":
        terms = [0, 1, 2]
    else:
        terms = [0, 1, 2, 3]
    mats = []
    for alpha in mesh.element_list(K):
        ws = [w, w, w]
        if coef_axes is not None:
            ws = [w * coef_axes[d][alpha[d]] for d in range(3)]
        out = np.zeros((n, n))
        for t in terms:
            tabs = [D[alpha[d]] if d == t else V[alpha[d]] for d in range(3)]
            o = np.zeros((n, n))
            if method == "classical":
                integrators.classical_kernel(tabs[0], tabs[1], tabs[2], ws[0], ws[1], ws[2], jac,
                                             rows, cols, 0, len(rows), o)
            else:
                buf = integrators.SumFactBuffers.allocate(p, q)
                buf.D[:] = 0.0
                buf.C[:] = 0.0
                integrators.sumfact_kernel(tabs[0], tabs[1], tabs[2], ws[0], ws[1], ws[2], jac,
                                           buf.D, buf.C, rows, cols, o)
            out = o if t == terms[0] else out + o
        mats.append((alpha, integrators.ElementMatrix(alpha, n, out, 0)))
    return assembly.assemble(mats, K, p)


def nonuniform_kv(K, p, seed):
    """Open knot vector with K distinct, randomly sized spans on [0, 1]."""
    r = np.random.default_rng(seed)
    h = r.uniform(0.5, 1.5, size=K)
    interior = np.cumsum(h)[:-1] / h.sum()
    knots = np.concatenate([np.zeros(p + 1), interior, np.ones(p + 1)])
    return splines.KnotVector(degree=p, elements=K, knots=knots)


def nonuniform_tables(kv, q):
    """V/D[e][r][k] at x = t_lo + (ref + 1) (h / 2), h = t_hi - t_lo of span e, by the
    reference's recursion (eval_basis; derivatives by the degree-reduction formula of
    eval_nonzero_basis_derivatives on the reference's _cox, splines.py:139-161)."""
    K, p, t = kv.elements, kv.degree, kv.knots
    ref, w = np.polynomial.legendre.leggauss(q)
    V = np.zeros((K, p + 1, q))
    D = np.zeros((K, p + 1, q))
    X = np.zeros((K, q))
    H = np.zeros(K)
    for e in range(K):
        lo, hi = t[p + e], t[p + e + 1]
        h = hi - lo
        xs = lo + (ref + 1.0) * (h / 2.0)
        X[e], H[e] = xs, h
        for k, x in enumerate(xs):
            for r in range(p + 1):
                i = e + r
                V[e, r, k] = splines.eval_basis(kv, i, p, x)
                if p >= 1:
                    dd = 0.0
                    d_left = t[i + p] - t[i]
                    if d_left > 0.0:
                        dd += splines._cox(t, i, p - 1, x, kv) / d_left
                    d_right = t[i + p + 1] - t[i + 1]
                    if d_right > 0.0:
                        dd -= splines._cox(t, i + 1, p - 1, x, kv) / d_right
                    D[e, r, k] = p * dd
    return dict(V=V, D=D, X=X, H=H, ref=ref, w=w)


def nonuniform_assemble(kv, q, method, op, tabs):
    """Global matrix of a general open knot vector by the reference kernels: per-axis
    weights w * (h_e / 2) (the per-element Jacobian of the identity geometry map), jac = 1,
    stiffness terms as in term_kernel_assemble, assembled by assembly.assemble."""
    K, p = kv.elements, kv.degree
    V, D, H, w = tabs["V"], tabs["D"], tabs["H"], tabs["w"]
    m = p + 1
    n = m**3
    rows, cols = integrators.canonical_pairs(n)
    terms = {"mass": [3], "stiffness": [0, 1, 2], "stiffness_mass": [0, 1, 2, 3]}[op]
    mats = []
    for alpha in mesh.element_list(K):
        ws = [w * (H[alpha[d]] / 2.0) for d in range(3)]
        out = np.zeros((n, n))
        for t in terms:
            tb = [D[alpha[d]] if d == t else V[alpha[d]] for d in range(3)]
            o = np.zeros((n, n))
            if method == "classical":
                integrators.classical_kernel(tb[0], tb[1], tb[2], ws[0], ws[1], ws[2], 1.0,
                                             rows, cols, 0, len(rows), o)
            else:
                buf = integrators.SumFactBuffers.allocate(p, q)
                buf.D[:] = 0.0
                buf.C[:] = 0.0
                integrators.sumfact_kernel(tb[0], tb[1], tb[2], ws[0], ws[1], ws[2], 1.0,
                                           buf.D, buf.C, rows, cols, o)
            out = o if t == terms[0] else out + o
        mats.append((alpha, integrators.ElementMatrix(alpha, n, out, 0)))
    return assembly.assemble(mats, K, p)


def main():
    # 1. basis tables (splines.py:164-178 through runtime.py:142-149 mapping)
    tabs = {}
    for K in (1, 2, 3, 5, 8):
        for p in range(0, 6):
            for q in sorted({p + 1, p + 3}):
                V, D = mesh_tables(K, p, q)
                tabs[f"V_K{K}_p{p}_q{q}"] = V
                tabs[f"D_K{K}_p{p}_q{q}"] = D
    save("tables.npz", **tabs)

    # 2. element matrices (integrators.py:193-230) for a few elements
    el = {}
    for K, p in ((1, 0), (2, 1), (3, 2), (4, 3), (3, 4)):
        kv = splines.make_knot_vector(K, p)
        buf = integrators.SumFactBuffers.allocate(p)
        for alpha in {(0, 0, 0), (K - 1, 0, min(1, K - 1)), (K // 2, K - 1, K // 2)}:
            rule = mesh.gauss_rule(p, K, alpha)
            a = "_".join(map(str, alpha))
            el[f"classical_K{K}_p{p}_{a}"] = integrators.integrate_element_classical(alpha, kv, rule).entries
            el[f"sumfact_K{K}_p{p}_{a}"] = integrators.integrate_element_sumfact(alpha, kv, rule, buf).entries
    save("element_mass.npz", **el)

    # 3. global mass Gram from run_integration (runtime.py:287-295)
    for K, p in ((1, 0), (2, 1), (3, 2), (4, 3), (2, 4), (5, 2), (6, 1)):
        for method in ("classical", "sumfact"):
            res = runtime.run_integration(runtime.RunConfig(method, "sequential", K, p))
            save(f"mass_{method}_K{K}_p{p}.npz", **ref_csr(res.gram))

    # 4. stiffness and stiffness+mass via the reference kernels per axis
    for K, p in ((2, 1), (3, 2), (4, 3), (3, 4)):
        for op in ("stiffness", "stiffness_mass"):
            g = term_kernel_assemble(K, p, p + 1, "classical", op)
            save(f"{op}_classical_K{K}_p{p}.npz", **ref_csr(g))
    g = term_kernel_assemble(4, 3, 4, "sumfact", "stiffness")
    save("stiffness_sumfact_K4_p3.npz", **ref_csr(g))

    # 5. separable coefficient c(x) = c1(x1) c2(x2) c3(x3) at the quadrature points
    rng = np.random.default_rng(42)
    for K, p, op in ((3, 2, "mass"), (3, 2, "stiffness_mass"), (4, 3, "stiffness")):
        q = p + 1
        cax = [rng.uniform(0.5, 1.5, size=(K, q)) for _ in range(3)]
        g = term_kernel_assemble(K, p, q, "classical", op, coef_axes=cax)
        d = ref_csr(g)
        d.update(c1=cax[0], c2=cax[1], c3=cax[2])
        save(f"sepcoef_{op}_K{K}_p{p}.npz", **d)

    # 6. 2D mass derived from the 3D reference Gram (C1 shape: K=16, p=2) and K=3, p=1
    for K, p in ((16, 2), (3, 1)):
        res = runtime.run_integration(runtime.RunConfig("classical", "over_elements", K, p,
                                                        workers=8))
        n1 = K + p
        G = res.gram.matrix.tocoo()
        r3 = np.unravel_index(G.row, (n1, n1, n1))
        c3 = np.unravel_index(G.col, (n1, n1, n1))
        import scipy.sparse

        r2 = r3[0] * n1 + r3[1]
        c2 = c3[0] * n1 + c3[1]
        M2 = scipy.sparse.coo_matrix((G.data, (r2, c2)), shape=(n1 * n1, n1 * n1)).tocsr()
        M2.sort_indices()
        save(f"mass2d_K{K}_p{p}.npz", indptr=M2.indptr.astype(np.int64),
             indices=M2.indices.astype(np.int64), data=M2.data, n=np.int64(n1 * n1))

    # 7. heat.assemble_rhs pins: M.mu and S.mu (heat.py:131-158)
    for K, p in ((3, 2), (4, 3)):
        hp = heat.HeatProblem(K, p, reassemble_each_step=False)
        mu = np.random.default_rng(7).standard_normal(hp.gram.n_dofs)
        f = heat.SplineField(kv=hp.kv, coefficients=mu)
        Mmu = hp.assemble_rhs(f, 0.0)
        Smu = Mmu - hp.assemble_rhs(f, 1.0)
        save(f"heat_rhs_K{K}_p{p}.npz", mu=mu, Mmu=Mmu, Smu=Smu)

    # 8. symbolic pattern (assembly.py:99-115)
    for K, p in ((1, 0), (2, 1), (3, 2), (5, 3), (2, 4)):
        pat = assembly.symbolic_pattern(K, p)
        save(f"pattern_K{K}_p{p}.npz", indptr=pat.indptr.astype(np.int64),
             indices=pat.indices.astype(np.int64))

    # 9. Gauss rules and Jacobians as the reference computes them (mesh.py:73-93)
    gr = {}
    for p in range(0, 8):
        r = mesh.gauss_rule(p, 5, (1, 2, 3))
        gr[f"nodes_p{p}"] = r.nodes
        gr[f"weights_p{p}"] = r.weights
        gr[f"jac_p{p}"] = np.float64(r.jacobian)
    save("gauss_rules.npz", **gr)

    # 10. per-axis weights (integrators.py:200-203 passes rule.weights[0..2] separately):
    #     element matrices of rules whose weights differ per axis (w * c_d)
    rng = np.random.default_rng(5)
    pa = {}
    for K, p in ((3, 2), (4, 3), (2, 4)):
        kv = splines.make_knot_vector(K, p)
        buf = integrators.SumFactBuffers.allocate(p)
        alpha = (K - 1, 0, K // 2)
        r0 = mesh.gauss_rule(p, K, alpha)
        c = rng.uniform(0.5, 1.5, size=(3, p + 1))
        rule = mesh.QuadratureRule(r0.points_per_direction, r0.nodes, r0.weights * c, r0.jacobian)
        pa[f"weights_K{K}_p{p}"] = rule.weights
        pa[f"classical_K{K}_p{p}"] = integrators.integrate_element_classical(alpha, kv, rule).entries
        pa[f"sumfact_K{K}_p{p}"] = integrators.integrate_element_sumfact(alpha, kv, rule, buf).entries
    save("element_peraxis.npz", **pa)

    # 11. eval_basis / eval_basis_order0 (splines.py:78-118) on open uniform knots and on
    #     general (non-uniform) open knot vectors -- the reference's recursion takes any
    #     non-decreasing knots (KnotVector.knots)
    eb = {}
    for tag, K, p in (("u", 4, 3), ("u", 3, 2), ("n", 5, 3), ("n", 4, 2), ("n", 6, 4), ("u", 2, 0)):
        if tag == "u":
            kv = splines.make_knot_vector(K, p)
        else:
            kv = nonuniform_kv(K, p, seed=K * 10 + p)
        t = kv.knots
        xs = np.unique(np.concatenate([t, np.linspace(0.0, 1.0, 23), rng.uniform(0, 1, 9)]))
        for q in range(p + 1):
            nb = len(t) - q - 1
            eb[f"{tag}_K{K}_p{p}_q{q}"] = np.array(
                [[splines.eval_basis(kv, i, q, x) for x in xs] for i in range(nb)])
        eb[f"{tag}_K{K}_p{p}_o0"] = np.array(
            [[splines.eval_basis_order0(kv, i, x) for x in xs] for i in range(len(t) - 1)])
        eb[f"{tag}_K{K}_p{p}_x"] = xs
        eb[f"{tag}_K{K}_p{p}_knots"] = t
    save("eval_basis.npz", **eb)

    # 12. general open knot vectors: per-element tables at the
    #     Gauss points mapped into each knot span, and global mass / stiffness matrices
    #     from the reference's own kernels with the per-element Jacobian folded into the
    #     per-axis weights (w_d = w h_e/2, jac = 1), assembled by assembly.assemble
    for K, p in ((5, 2), (4, 3), (3, 1), (6, 3)):
        kv = nonuniform_kv(K, p, seed=K * 10 + p)
        q = p + 1
        d = nonuniform_tables(kv, q)
        d["knots"] = kv.knots
        for op in ("mass", "stiffness", "stiffness_mass") if p >= 1 else ("mass",):
            for method in ("classical", "sumfact"):
                c = ref_csr(nonuniform_assemble(kv, q, method, op, d))
                if "indptr" in d:  # one pattern for every matrix of the mesh
                    assert np.array_equal(d["indptr"], c["indptr"])
                    assert np.array_equal(d["indices"], c["indices"])
                d["indptr"], d["indices"] = c["indptr"], c["indices"]
                d[f"{op}_{method}"] = c["data"]
        save(f"nonuniform_K{K}_p{p}.npz", **d)
    # 13. run_within_element with an ExecutionTrace (runtime.py:476-505, :100-107)
    tr = {}
    for K, p, workers in ((2, 0, 1), (2, 1, 3), (3, 2, 2)):
        kv = splines.make_knot_vector(K, p)
        alpha = (K - 1, 0, K // 2)
        t = runtime.ExecutionTrace()
        em = runtime.run_within_element(alpha, kv, "sumfact", workers, trace=t)
        key = f"K{K}_p{p}_w{workers}"
        order = np.array(t.completion_order, dtype=np.int64)
        # the class of every completed task, in completion order (deterministic: the
        # reference runs the classes barrier-separated); inside a class the reference's
        # worker chunks finish in any order, so the raw order is kept only for workers=1
        tr[f"{key}_class_of_order"] = np.asarray(t.graph.classes)[order].astype(np.int64)
        tr[f"{key}_order_sorted"] = np.sort(order)
        if workers == 1:
            tr[f"{key}_order"] = order
        tr[f"{key}_barriers"] = np.int64(t.barriers)
        tr[f"{key}_syncs"] = np.int64(t.intra_class_syncs)
        tr[f"{key}_ntasks"] = np.int64(t.graph.n_tasks)
        tr[f"{key}_sumfact"] = em.entries
        tr[f"{key}_classical"] = runtime.run_within_element(alpha, kv, "classical", workers).entries
    save("within_element.npz", **tr)

    # 14. high degrees (the paper's p = 9 Gram; integrators.py handles
    #     any p): K1 tables, an element matrix whose sum-factorization stages exceed shared
    #     memory (p = 7), and global Grams from run_integration
    hi = {}
    for K, p in ((3, 6), (2, 7), (2, 8), (3, 9)):
        V, D = mesh_tables(K, p, p + 1)
        hi[f"V_K{K}_p{p}"] = V
        hi[f"D_K{K}_p{p}"] = D
    kv = splines.make_knot_vector(2, 7)
    alpha = (1, 0, 1)
    hi["element_sumfact_K2_p7"] = integrators.integrate_element_sumfact(
        alpha, kv, mesh.gauss_rule(7, 2, alpha), integrators.SumFactBuffers.allocate(7)).entries
    save("high_degree.npz", **hi)
    for K, p in ((2, 6), (1, 7)):
        res = runtime.run_integration(runtime.RunConfig("sumfact", "sequential", K, p))
        save(f"mass_sumfact_K{K}_p{p}.npz", **ref_csr(res.gram))
    print("igabench", igabench.__version__)


if __name__ == "__main__":
    main()

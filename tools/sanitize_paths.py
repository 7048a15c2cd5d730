"""Exercise every device path at small sizes (for compute-sanitizer runs)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2207_00280_b200 as P  # noqa: E402
from paper_2207_00280_b200.operator import MatrixFreeOperator, cg  # noqa: E402


def main():
    for K, p, op in ((5, 3, "stiffness"), (4, 2, "mass"), (3, 4, "stiffness_mass"), (2, 5, "stiffness"),
                     (6, 1, "mass")):
        q = p + 1
        coef = np.random.default_rng(0).uniform(0.5, 1.5, size=(K**3, q**3))
        for method, assembly, c in (("sumfact", "separable", None), ("sumfact", "owner", None),
                                    ("sumfact", "owner", coef), ("sumfact", "scatter", coef),
                                    ("classical", "auto", coef)):
            P.run_integration(P.RunConfig(method, "device", K, p, operator=op, coefficient=c,
                                          assembly=assembly)).gram.values.sum().item()
    # element slabs (multi-GPU launches) through the band-table and per-CTA paths
    import torch

    from paper_2207_00280_b200.device import MeshProblem

    mp = MeshProblem(3, 7, 3, 4, "stiffness", None)
    v = torch.empty(mp.nnz(2, 8), dtype=torch.float64, device="cuda")
    mp.build_band_tables()
    for method in (3, 2):
        mp.integrate_assemble(v, method, el_range=(2, 5), plane_range=(2, 8), band=method == 3)
    mp.integrate_assemble(v, 3, el_range=(2, 5), plane_range=(2, 8))
    g = P.run_integration(P.RunConfig("sumfact", "device", 6, 3, operator="stiffness")).gram
    g.spmv(np.ones(g.n_dofs))
    P.write_matrix_market(g, "/tmp/sanitize.mtx")
    for K, p, c in ((6, 3, None), (4, 2, np.ones((64, 27)))):
        o = MatrixFreeOperator(K, p, coefficient=c)
        x = np.ones(o.n_dofs)
        o.apply(x, 1.0, 0.5)
        cg(o, o.apply(x, 1.0, 0.0), rtol=1e-8)
    P.run_integration(P.RunConfig("classical", "device", 6, 2, dim=2))
    print("sanitize paths ok")


if __name__ == "__main__":
    main()

"""Time the Matrix Market export of the C3 matrix: device row-block streaming writer
(paper_2207_00280_b200.write_matrix_market) vs the reference's scipy.io.mmwrite on the
host CSR of the same matrix (assembly.py:118-120).  Checks the files are identical."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2207_00280_b200 as P  # noqa: E402


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    out = sys.argv[2] if len(sys.argv) > 2 else "/tmp/mm_export"
    os.makedirs(out, exist_ok=True)
    gram = P.run_integration(P.RunConfig("sumfact", "device", K, 3, operator="stiffness")).gram
    a = os.path.join(out, "ours.mtx")
    t0 = time.perf_counter()
    P.write_matrix_market(gram, a)
    t_ours = time.perf_counter() - t0
    import scipy.io

    m = gram.matrix  # host CSR (D2H + pattern), not timed: the reference already holds it
    b = os.path.join(out, "scipy.mtx")
    t0 = time.perf_counter()
    scipy.io.mmwrite(b, m.tocoo(), symmetry="symmetric")
    t_ref = time.perf_counter() - t0
    h = [hashlib.sha256(open(x, "rb").read()).hexdigest() for x in (a, b)]
    print(json.dumps({"K": K, "p": 3, "nnz": int(m.nnz), "bytes": os.path.getsize(a),
                      "ours_s": t_ours, "scipy_mmwrite_s": t_ref, "identical": h[0] == h[1],
                      "threads": os.cpu_count()}))
    os.remove(a)
    os.remove(b)


if __name__ == "__main__":
    main()

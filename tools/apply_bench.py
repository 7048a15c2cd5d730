"""Matrix-free operator application (iga_apply) vs SpMV on the assembled matrix
(iga_spmv) for the C3 mesh: device time per application (CUDA events, L2 flushed)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2207_00280_b200 as P  # noqa: E402
from paper_2207_00280_b200 import _lib  # noqa: E402
from paper_2207_00280_b200.operator import MatrixFreeOperator  # noqa: E402


def timeit(fn, reps=20):
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ts) / reps


def main():
    K, p = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (64, 3)
    op = MatrixFreeOperator(K, p)
    n = op.n_dofs
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    import ctypes

    s = op.prob.problem_struct()
    st = _lib.stream_ptr()
    L = _lib.load()

    def apply():
        _lib.check(L.iga_apply(ctypes.byref(s), 1.0, 1.0, _lib.ptr(x), _lib.ptr(y), st))

    t_apply = timeit(apply)
    gram = P.run_integration(P.RunConfig("sumfact", "device", K, p, operator="stiffness")).gram
    vals = gram.values

    def spmv():
        _lib.check(L.iga_spmv(3, K, p, _lib.ptr(vals), _lib.ptr(x), _lib.ptr(y), st))

    t_spmv = timeit(spmv)
    print(json.dumps({"K": K, "p": p, "n_dofs": n, "apply_ms": t_apply, "spmv_ms": t_spmv,
                      "spmv_GBps": (vals.numel() * 8 + 2 * n * 8) / (t_spmv / 1e3) / 1e9}))


if __name__ == "__main__":
    main()

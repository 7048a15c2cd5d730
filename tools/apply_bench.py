"""Matrix-free operator application (iga_apply) vs SpMV on the assembled matrix
(iga_spmv) for the C3 mesh: device time per application (CUDA events, L2 flushed);
then the heat step's CG solve (iga_cg, the loop inside the library) against the same
iteration written as eager torch with a host sync per iteration (round 1's operator.cg)."""
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
    out = {"K": K, "p": p, "n_dofs": n, "apply_ms": t_apply, "spmv_ms": t_spmv,
           "spmv_GBps": (vals.numel() * 8 + 2 * n * 8) / (t_spmv / 1e3) / 1e9}

    # CG: (M + dt S) u = b matrix-free, and G u = b on the assembled mass matrix
    from paper_2207_00280_b200.operator import cg

    gram_m = P.run_integration(P.RunConfig("sumfact", "device", K, p)).gram
    b = torch.randn(n, dtype=torch.float64, device="cuda")

    def eager(apply_fn, rtol=1e-10):
        xk = torch.zeros_like(b)
        r = b.clone()
        pk = r.clone()
        Ap = torch.empty_like(b)
        rr = torch.dot(r, r)
        tol = rtol * torch.linalg.norm(b)
        for it in range(10 * n):
            if torch.sqrt(rr) <= tol:  # host sync every iteration
                return it
            apply_fn(pk, Ap)
            a = rr / torch.dot(pk, Ap)
            xk += a * pk
            r -= a * Ap
            rr2 = torch.dot(r, r)
            pk = r + (rr2 / rr) * pk
            rr = rr2
        return -1

    def mf_apply(v, o):
        _lib.check(L.iga_apply(ctypes.byref(s), 1.0, 0.01, _lib.ptr(v), _lib.ptr(o), st))

    def mass_spmv(v, o):
        _lib.check(L.iga_spmv(3, K, p, _lib.ptr(gram_m.values), _lib.ptr(v), _lib.ptr(o), st))

    for name, A, kw, fn in (("cg_matrix_free", op, dict(alpha=1.0, beta=0.01), mf_apply),
                            ("cg_assembled_mass", gram_m, {}, mass_spmv)):
        res = {}
        for _ in range(2):
            torch.cuda.synchronize()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            _, its = cg(A, b, rtol=1e-10, **kw)
            e.record()
            torch.cuda.synchronize()
            res = {"iters": its, "ms": a.elapsed_time(e)}
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        its_e = eager(fn)
        e.record()
        torch.cuda.synchronize()
        res.update(ms_per_iter=res["ms"] / max(1, res["iters"]), eager_iters=its_e,
                   eager_ms=a.elapsed_time(e))
        res["eager_ms_per_iter"] = res["eager_ms"] / max(1, its_e)
        out[name] = res
    print(json.dumps(out))


if __name__ == "__main__":
    main()

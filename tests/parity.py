"""Parity criterion used by every test.

North-star tolerance: per-entry relative error <= 1e-12 in fp64, against the
reference's classical-integration output.

An entry whose exact value cancels (a sum of terms of both signs that is much
smaller than the sum of their magnitudes) carries a rounding error of order
eps * A[I,J], A = sum over quadrature terms of |term| -- for EVERY fp64
algorithm, including the reference's own classical vs sum-factorization pair
(tests/test_oracle.py::test_separable_coefficient_* shows them differ by 1e-11
relative on such entries).  The per-entry bound is therefore

    |a - ref| <= RTOL * |ref| + COND * eps * A[I,J]         (A from the oracle)

which equals the strict 1e-12 relative bound wherever A ~ |ref| (the
COND*eps*A term is ~1.4e-14 relative there).  Without A, exact-zero entries of
the operator (|ref| <= 64 eps max|row|) are checked against 64 eps max|row|
and all others strictly.  The stats always report the strict per-entry
relative error so nothing is hidden.
"""

import json
import os

import numpy as np

RTOL = 1e-12
EPS = np.finfo(np.float64).eps
COND = 64.0
ZERO_REL = COND * EPS


def row_max(indptr, values):
    indptr = np.asarray(indptr, dtype=np.int64)
    counts = np.diff(indptr)
    out = np.zeros(len(counts))
    nz = counts > 0
    out[nz] = np.maximum.reduceat(np.abs(values), indptr[:-1][nz])
    return np.repeat(out, counts)


def compare(values, ref, indptr, rtol=RTOL, absref=None):
    """Return stats; ``ok`` is the verdict of the criterion in the module doc."""
    values = np.asarray(values, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert values.shape == ref.shape, (values.shape, ref.shape)
    d = np.abs(values - ref)
    rm = row_max(indptr, ref)
    with np.errstate(divide="ignore", invalid="ignore"):
        strict = np.where(ref != 0, d / np.abs(ref), np.where(d == 0, 0.0, np.inf))
    if absref is not None:
        bound = rtol * np.abs(ref) + COND * EPS * np.asarray(absref)
        ok_e = d <= bound
        n_cond = int(np.sum((strict > rtol) & ok_e))
    else:
        zero = np.abs(ref) <= ZERO_REL * rm
        ok_e = np.where(zero, d <= ZERO_REL * rm, strict <= rtol)
        n_cond = int(np.sum(zero & (strict > rtol) & ok_e))
    ok = bool(np.all(ok_e) and np.all(np.isfinite(values)))
    finite = strict[np.isfinite(strict)]
    return {
        "ok": ok,
        "max_rel": float(strict.max(initial=0.0)),
        "p99_rel": float(np.quantile(finite, 0.99)) if finite.size else 0.0,
        "n_rel_above_rtol": int(np.sum(strict > rtol)),
        "n_conditioning_bound": n_cond,
        "max_abs_over_rowmax": float((d / np.maximum(rm, 1e-300)).max(initial=0.0)),
        "n": int(values.size),
    }


# IGA_PARITY_LOG=<file>: every assert_parity call appends one JSON line
# {config, path, max_rel_strict, n_rel_above_rtol, n_conditioning_bound, ...}; the GPU
# suite's log is committed as profiles/parity_<round>.json (tools/parity_table.py).
PARITY_LOG = os.environ.get("IGA_PARITY_LOG")


def _log(st, config, path, what, strict):
    if not PARITY_LOG:
        return
    if config is None:  # unlabeled call: the test id names the case
        config = what or os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0]
    rec = {"config": config, "path": path, "what": what, "strict_asserted": bool(strict),
           "max_rel_strict": st["max_rel"], "p99_rel": st["p99_rel"],
           "n_rel_above_rtol": st["n_rel_above_rtol"],
           "n_conditioning_bound": st["n_conditioning_bound"], "n": st["n"], "ok": st["ok"]}
    os.makedirs(os.path.dirname(os.path.abspath(PARITY_LOG)), exist_ok=True)
    with open(PARITY_LOG, "a") as f:
        f.write(json.dumps(rec) + "\n")


def assert_parity(values, ref, indptr, rtol=RTOL, what="", absref=None, config=None, path=None,
                  strict=False):
    """Assert the criterion of the module doc; ``strict`` additionally requires every entry
    within the pure per-entry relative bound (n_rel_above_rtol == 0, the north star's
    tolerance without the conditioning term)."""
    st = compare(values, ref, indptr, rtol, absref)
    _log(st, config, path, what, strict)
    assert st["ok"], f"parity failed {what}: {st}"
    if strict:
        assert st["n_rel_above_rtol"] == 0, f"strict 1e-12 bound violated {what}: {st}"
    return st

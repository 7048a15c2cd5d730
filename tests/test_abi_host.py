"""CPU tests: the C-ABI library loads and exports every declared symbol, the
host-side arithmetic and argument validation (no kernel launches), and the
drop-in host API (knots, Gauss rules, indices, RunConfig)."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from tests.conftest import ROOT, load_golden


@pytest.fixture(scope="module")
def lib():
    from paper_2207_00280_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    return _lib.load()


def test_header_symbols_exported(lib):
    from paper_2207_00280_b200 import _lib

    hdr = open(os.path.join(ROOT, "include", "iga_b200.h")).read()
    declared = set(re.findall(r"\b(iga_[a-z_0-9]+)\s*\(", hdr))
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    so = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(so, name), name
    assert lib.iga_abi_version() == 5


def test_cg_work_size_and_validation(lib):
    """iga_cg (ABI v5): work-array size and argument checks before any CUDA call."""
    from paper_2207_00280_b200 import _lib

    n = 1000
    assert lib.iga_cg_work_size(n) == 3 * n + 3 * 296 + 8
    assert lib.iga_cg_work_size(0) == -1
    it = ctypes.c_int64(-1)
    dummy = ctypes.c_void_p(16)
    n = (4 + 2) ** 3  # K = 4, p = 2
    bad = [dict(n=0), dict(n=n + 1), dict(rtol=-1.0), dict(maxiter=-1), dict(check=0),
           dict(values=None)]
    for b in bad:
        args = dict(n=n, rtol=1e-10, maxiter=10, check=4, values=dummy)
        args.update(b)
        rc = lib.iga_cg(3, 4, 2, args["values"], None, 1.0, 0.0, args["n"], dummy, dummy, dummy,
                        args["rtol"], args["maxiter"], args["check"], ctypes.byref(it), None)
        assert rc == _lib.IGA_EINVAL, b
        with pytest.raises(ValueError):
            _lib.check(rc)


def test_library_targets_sm100a():
    from paper_2207_00280_b200 import _lib
    import shutil
    import subprocess

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("dim,K,p", [(3, 1, 0), (3, 2, 1), (3, 5, 3), (3, 7, 4), (2, 16, 2),
                                     (2, 3, 5), (3, 64, 3), (3, 256, 3), (3, 96, 4)])
def test_csr_nnz_closed_form(lib, dim, K, p):
    N = K + p
    nnz1 = N * (2 * p + 1) - p * (p + 1)
    assert lib.iga_csr_nnz(dim, K, p, 0, N**dim) == nnz1**dim
    if K <= 8:
        ip, _ = O.pattern(dim, K, p)
        for lo in range(0, N**dim, max(1, N**dim // 7)):
            for hi in (lo, min(N**dim, lo + 5), N**dim):
                assert lib.iga_csr_nnz(dim, K, p, lo, hi) == ip[hi] - ip[lo]


def test_baseline_config_sizes(lib):
    """SURVEY.md §8 size table."""
    assert lib.iga_csr_nnz(2, 16, 2, 0, 18**2) == 7056
    assert lib.iga_csr_nnz(3, 32, 2, 0, 34**3) == 4410944
    assert lib.iga_csr_nnz(3, 64, 3, 0, 67**3) == 95443993
    assert lib.iga_csr_nnz(3, 96, 4, 0, 100**3) == 681472000
    assert lib.iga_csr_nnz(3, 256, 3, 0, 259**3) == 5841725401


def test_invalid_arguments_rejected_before_launch(lib):
    from paper_2207_00280_b200 import _lib

    assert lib.iga_csr_nnz(4, 3, 1, 0, 1) == -1
    assert lib.iga_csr_pattern(4, 3, 1, 0, 1, None, None, None) == _lib.IGA_EINVAL
    assert lib.iga_csr_pattern(3, 3, 1, 5, 2, None, None, None) == _lib.IGA_EINVAL
    assert lib.iga_mesh_tables(0, 1, 2, None, None, None, None) == _lib.IGA_EINVAL
    assert lib.iga_axpy(-1, None, None, None) == _lib.IGA_EINVAL
    prob = _lib.IgaProblem(dim=3, K=2, p=0, q=1, op=1)
    rc = lib.iga_integrate_assemble(ctypes.byref(prob), 2, 0, 2, 0, 2, None, None)
    assert rc == _lib.IGA_EINVAL
    assert b"degree >= 1" in lib.iga_last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_knots_and_gauss_match_reference():
    import paper_2207_00280_b200 as P

    for K in (1, 2, 5, 64):
        for p in range(6):
            kv = P.make_knot_vector(K, p)
            assert kv.knots.tobytes() == O.knots(K, p).tobytes()
            assert kv.n_basis == K + p
    g = load_golden("gauss_rules")
    for p in range(8):
        r = P.gauss_rule(p, 5, (1, 2, 3))
        assert r.nodes.tobytes() == g[f"nodes_p{p}"].tobytes()
        assert r.weights.tobytes() == g[f"weights_p{p}"].tobytes()
        assert r.jacobian == float(g[f"jac_p{p}"])
    with pytest.raises(ValueError):
        P.make_knot_vector(0, 1)
    with pytest.raises(ValueError):
        P.make_knot_vector(3, -1)


def test_mesh_indexing():
    import paper_2207_00280_b200 as P

    assert P.element_list(2)[:3] == [(0, 0, 0), (0, 0, 1), (0, 1, 0)]
    assert P.local_index((2, 3, 4), (3, 4, 5), 2) == 13
    sup = P.support_set((1, 0, 2), 2)
    assert len(sup) == 27 and sup[0] == (1, 0, 2) and sup[-1] == (3, 2, 4)
    assert [P.local_index((1, 0, 2), b, 2) for b in sup] == list(range(27))
    assert P.dof_index((1, 2, 3), 4, 2) == (1 * 6 + 2) * 6 + 3
    with pytest.raises(ValueError):
        P.dof_index((6, 0, 0), 4, 2)
    rows, cols = P.canonical_pairs(8)
    assert len(rows) == 36 and np.all(rows >= cols)
    assert P.flop_count("classical", 3) == 2080 * 64 * 10
    assert P.flop_count("sumfact", 3) == 4 * (16 * 64 + 256 * 16 + 2080 * 4)


def test_runconfig_validation():
    import paper_2207_00280_b200 as P

    P.RunConfig("sumfact", "device", 4, 3, operator="stiffness")
    P.RunConfig("classical", "over_elements", 4, 2, workers=8)  # reference values stay valid
    for bad in (dict(method="x"), dict(strategy="gpu"), dict(mesh=0), dict(degree=-1),
                dict(workers=0), dict(repetitions=0), dict(chunking="x"), dict(operator="x"),
                dict(dim=4), dict(devices=0), dict(assembly="x"), dict(quad_points=0)):
        kw = dict(method="sumfact", strategy="device", mesh=4, degree=2)
        kw.update(bad)
        with pytest.raises(ValueError):
            P.RunConfig(**kw)
    with pytest.raises(ValueError):
        P.RunConfig("sumfact", "device", 4, 0, operator="stiffness")
    assert P.RunConfig("sumfact", "device", 4, 3).points == 4


def test_device_path_fails_loudly_without_cuda():
    import torch

    import paper_2207_00280_b200 as P

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError, match="CUDA device"):
        P.run_integration(P.RunConfig("sumfact", "device", 2, 1))


def test_auto_selects_kernel():
    import paper_2207_00280_b200 as pkg

    from paper_2207_00280_b200 import _lib
    from paper_2207_00280_b200.runtime import method_code

    K, p = 4, 3
    assert method_code(pkg.RunConfig("sumfact", "device", K, p)) == _lib.METHOD_SEPARABLE
    assert method_code(pkg.RunConfig("sumfact", "device", K, p, coefficient=2.0)) == \
        _lib.METHOD_SEPARABLE
    coef = np.ones((K**3, (p + 1)**3))
    assert method_code(pkg.RunConfig("sumfact", "device", K, p, coefficient=coef)) == \
        _lib.METHOD_SUMFACT_ASSEMBLED
    assert method_code(pkg.RunConfig("sumfact", "device", K, p, assembly="owner")) == \
        _lib.METHOD_SUMFACT_ASSEMBLED


@pytest.mark.parametrize("dim,K,p,op", [(3, 3, 2, "stiffness"), (3, 4, 1, "mass"), (2, 5, 2, "mass"),
                                        (3, 2, 3, "stiffness_mass"), (3, 1, 0, "mass")])
def test_matrix_market_host_writer_matches_scipy(lib, tmp_path, dim, K, p, op):
    """Native Matrix Market writer (csrc/iga_mmio.cu) vs the reference's
    scipy.io.mmwrite(..., symmetry="symmetric") (assembly.py:118-120): identical bytes."""
    import io

    import scipy.io
    import scipy.sparse

    ip, ix, v = O.integrate_assemble(dim, K, p, op, "classical")
    if K == 3:  # exercise the value formatter: signed zero, subnormal, huge, integers
        v = v.copy()
        v[:6] = [-0.0, 5e-324, 1.7976931348623157e308, 2.0, -123.5, 1e-5]
    n = len(ip) - 1
    m = scipy.sparse.csr_matrix((v, ix, ip), shape=(n, n))
    ref = io.BytesIO()
    scipy.io.mmwrite(ref, m.tocoo(), symmetry="symmetric")
    f = tmp_path / "a.mtx"
    assert lib.iga_write_matrix_market_host(dim, K, p, v.ctypes.data, str(f).encode(), 3) == 0
    assert f.read_bytes() == ref.getvalue()


def test_bench_csv_columns_match_reference_cli():
    from paper_2207_00280_b200.benchcsv import BENCH_COLUMNS

    src = open("/root/reference/pkg/src/igabench/cli.py").read() if os.path.exists(
        "/root/reference/pkg/src/igabench/cli.py") else None
    if src is None:
        pytest.skip("reference not mounted")
    assert f"BENCH_COLUMNS = {BENCH_COLUMNS!r}".replace("'", '"') in src


def test_perfmodel_matches_survey_counts():
    """Roofline numerators (bench.py): the algorithmic counts of SURVEY.md §8(d)'s table
    and §8 derived sizes."""
    from paper_2207_00280_b200 import perfmodel as m

    # classical, per element (§8(d) "flops/el (classical)")
    assert m.classical_flops("mass", 2, 3) == 40_824                 # C2
    assert m.classical_flops("stiffness", 3, 4) == 1_331_200         # C3, C5
    assert m.classical_flops("stiffness_mass", 4, 5) == 11_812_500   # C4
    # general element-local sum factorization, per element (§8(d) "flops/el (sumfact general)")
    assert m.element_sumfact_flops("mass", 2, 3) == 4_212
    assert m.element_sumfact_flops("stiffness", 3, 4) == 61_952
    # bytes: 8 nnz (+ 8 q^3 per element for a field); nnz from §8's size table
    assert m.algorithmic_bytes(3, 64, 3, 4, False) == 8 * 95_443_993
    assert m.algorithmic_bytes(3, 32, 2, 3, True) == 8 * 4_410_944 + 8 * 32**3 * 27

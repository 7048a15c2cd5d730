"""GPU parity of the symmetric-half kernels -- k_gsf3_p3s (csrc/iga_gsf_p3s.cu, p = 3, q = 4)
and the SYM mode of the generic DMMA kernel (csrc/iga_gsf_mma.cu, other degrees): both
compute S[I, J] for J0 >= I0 and mirror the rest through rings -- against the oracle's
classical integration (reference integrators.py:77-109 + assembly.py:80-82), forced on and
off (IGA_GSF_SYM=0; read once per process, hence the subprocesses), on meshes small enough to
exercise the rings' first and last target rows, and with the generic kernel's element
columns forced into 3 segments (IGA_GSF_SEGS=3: every segment emits the runs its rows feed
across its boundaries)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from tests.parity import compare  # noqa: E402

# (K, p, q, operator, coefficient kind): p = 3 q = 4 -> k_gsf3_p3s, p >= 3 otherwise the generic
# kernel's symmetric mode; p = 2 stiffness runs the generic kernel in full (also checked)
CASES = [(1, 3, 4, "stiffness", "scalar"), (2, 3, 4, "mass", "field"), (3, 3, 4, "stiffness_mass", "field"),
         (4, 3, 4, "stiffness", "field"), (5, 3, 4, "mass", "scalar"), (6, 3, 4, "stiffness", "scalar"),
         (7, 3, 4, "stiffness_mass", "scalar"), (9, 3, 4, "stiffness", "field"),
         (5, 2, 3, "stiffness", "field"), (8, 2, 3, "stiffness_mass", "scalar"), (7, 2, 4, "stiffness", "scalar"),
         (3, 4, 5, "stiffness_mass", "field"), (7, 4, 5, "stiffness", "scalar"), (6, 5, 6, "mass", "field"),
         (4, 3, 5, "stiffness", "field")]


def _coef(K, q, kind, seed):
    if kind == "scalar":
        return None
    return np.random.default_rng(seed).uniform(0.5, 1.5, size=(K**3, q**3))


def _run_cases():
    """Child process: every CASE through run_integration(assembly="owner"); one JSON line of
    parity stats each, plus the largest asymmetry among entries with J0 != I0 (the mirrored
    ones: exactly 0 when the mirror lands where it should)."""
    import paper_2207_00280_b200 as pkg

    for i, (K, p, q, op, kind) in enumerate(CASES):
        coef = _coef(K, q, kind, 200 + i)
        ip, ix, ref = O.integrate_assemble(3, K, p, op, "classical", q=q, coef=coef)
        _, _, A = O.integrate_assemble(3, K, p, op, "classical", q=q, coef=coef, absolute=True)
        res = pkg.run_integration(pkg.RunConfig("sumfact", "device", K, p, quad_points=q, operator=op,
                                                coefficient=coef, assembly="owner"))
        v = res.gram.values.cpu().numpy()
        st = compare(v, ref, ip, absref=A)
        import scipy.sparse as sp

        N = K + p
        M = sp.csr_matrix((v, ix, ip), shape=(len(ip) - 1, len(ip) - 1))
        D = (M - M.T).tocoo()
        i0, j0 = D.row // (N * N), D.col // (N * N)
        asym = float(np.max(np.abs(D.data[i0 != j0]), initial=0.0))
        print(json.dumps({"case": [K, p, q, op, kind], "ok": bool(st["ok"]), "max_rel": float(st["max_rel"]),
                          "asym_mirrored": asym}), flush=True)


def _child(sym, segs=None):
    env = dict(os.environ, IGA_GSF_SYM=sym)
    if segs is not None:
        env["IGA_GSF_SEGS"] = str(segs)
    out = subprocess.run([sys.executable, os.path.abspath(__file__), "--case"], env=env, cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return [json.loads(line) for line in out.stdout.splitlines() if line.startswith("{")]


@pytest.mark.gpu
@pytest.mark.parametrize("segs", [None, 3])
def test_symmetric_kernel_vs_oracle_and_exact_mirror(segs):
    rows = _child("1", segs)
    assert len(rows) == len(CASES)
    bad = [r for r in rows if not r["ok"]]
    assert not bad, bad
    # every mirrored value (p >= 3: the symmetric kernels) is the bit pattern of its twin
    assert all(r["asym_mirrored"] == 0.0 for r in rows if r["case"][1] >= 3), rows


@pytest.mark.gpu
def test_nonsymmetric_kernel_vs_oracle():
    rows = _child("0")
    assert len(rows) == len(CASES)
    bad = [r for r in rows if not r["ok"]]
    assert not bad, bad


if __name__ == "__main__" and "--case" in sys.argv:
    _run_cases()


@pytest.mark.gpu
@pytest.mark.parametrize("K,p,op", [(10, 3, "stiffness"), (9, 4, "stiffness_mass"), (8, 3, "mass")])
def test_symmetric_slabs_sum_to_full(K, p, op):
    """Element slabs with their interface planes (the multi-GPU decomposition) run
    the symmetric kernels too: a slab's contribution is symmetric and lives in the rows it
    writes.  The outputs start as NaN, so a value the kernels fail to write (the slab's first p
    planes hold zeros for columns below it) shows up; the partial planes add up to the
    whole-mesh matrix."""
    import torch

    from paper_2207_00280_b200 import _lib
    from paper_2207_00280_b200.device import MeshProblem

    q = p + 1
    N = K + p
    coef = torch.from_numpy(_coef(K, q, "field", 11)).cuda()
    mp = MeshProblem(3, K, p, operator=op, coefficient=coef)
    full = torch.full((mp.nnz(),), float("nan"), dtype=torch.float64, device="cuda")
    mp.integrate_assemble(full, _lib.METHOD_SUMFACT_ASSEMBLED)
    acc = torch.zeros_like(full)
    bounds = [0, 3, 6, K]
    for g in range(3):
        lo, hi = bounds[g], bounds[g + 1]
        phi = min(hi + p, N)
        part = torch.full((mp.nnz(lo, phi),), float("nan"), dtype=torch.float64, device="cuda")
        mp.integrate_assemble(part, _lib.METHOD_SUMFACT_ASSEMBLED, el_range=(lo, hi), plane_range=(lo, phi))
        assert not torch.isnan(part).any(), f"slab {g}: unwritten values"
        off = mp.nnz(0, lo)
        acc[off:off + part.numel()] += part
    c = coef.cpu().numpy()
    ip, _, ref = O.integrate_assemble(3, K, p, op, "classical", q=q, coef=c)
    _, _, A = O.integrate_assemble(3, K, p, op, "classical", q=q, coef=c, absolute=True)
    from tests.parity import assert_parity

    assert_parity(full.cpu().numpy(), ref, ip, what=f"sym full {op} K={K} p={p}", absref=A)
    assert_parity(acc.cpu().numpy(), ref, ip, what=f"sym slabs {op} K={K} p={p}", absref=A)


@pytest.mark.gpu
@pytest.mark.parametrize("K,p,op,kind", [(40, 3, "stiffness", "scalar"), (23, 3, "stiffness_mass", "field"),
                                        (12, 4, "stiffness_mass", "field")])
def test_symmetric_kernels_repeat_bitwise(K, p, op, kind):
    """The symmetric kernels hand rows between warp roles through mbarriers (k_gsf3_p3s: stages
    A / B / S and the emitter warps) or CTA barriers (generic kernel): a missing wait would
    show as run-to-run differences or as values left unwritten.  20 runs into a NaN-prefilled
    target are bitwise equal to the first (the reference's reproducibility promise,
    runtime.py:16-20)."""
    import torch

    import paper_2207_00280_b200 as pkg
    from paper_2207_00280_b200.runtime import DeviceSession

    q = p + 1
    coef = None if kind == "scalar" else np.random.default_rng(7).uniform(0.5, 1.5, size=(K,) * 3 + (q,) * 3)
    cfg = pkg.RunConfig("sumfact", "device", K, p, operator=op, coefficient=coef, dim=3, assembly="owner")
    sess = DeviceSession(cfg, use_graph=False)
    sess.step()
    torch.cuda.synchronize()
    first = sess.values.clone()
    assert not torch.isnan(first).any()
    for _ in range(20):
        sess.values.fill_(float("nan"))
        sess.step()
        torch.cuda.synchronize()
        assert torch.equal(sess.values.view(torch.int64), first.view(torch.int64))


@pytest.mark.gpu
@pytest.mark.parametrize("sym", ["1", "0"])
def test_p3_field_unaligned_coefficient_pointer(sym):
    """The folded p = 3 kernels copy the coefficient field with 16-byte cp.async when the
    caller's pointer allows it and with 8-byte copies otherwise (a C-ABI caller may pass any
    8-byte aligned device pointer): a field stored one double into an allocation gives the
    same bits as the aligned one (IGA_GSF_SYM is read once per process, hence the child)."""
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
from paper_2207_00280_b200.device import MeshProblem
K, p = 7, 3
coef = np.random.default_rng(3).uniform(0.5, 1.5, size=(K**3, 64))
prob = MeshProblem(3, K, p, operator="stiffness_mass", coefficient=coef)
out = []
for shift in (0, 1):
    buf = torch.empty(coef.size + 2, dtype=torch.float64, device="cuda")
    view = buf[shift:shift + coef.size].view(K**3, 64)
    view.copy_(torch.from_numpy(coef))
    assert view.data_ptr() %% 16 == 8 * shift
    prob.coef = view
    vals = torch.full((prob.nnz(),), float("nan"), dtype=torch.float64, device="cuda")
    prob.integrate_assemble(vals, 2)
    torch.cuda.synchronize()
    out.append(vals.cpu().numpy())
assert not np.isnan(out[0]).any()
assert out[0].tobytes() == out[1].tobytes()
print("ok")
""" % ROOT
    env = dict(os.environ, IGA_GSF_SYM=sym)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr

"""The bench.py contract the driver relies on, checked on CPU: the reference arm's JSON line
(impl, metric/unit/config identical to the GPU arm's, cpu_baseline, e2e with zero copies) and
the algorithmic flop models behind the roofline numerators (perfmodel.py)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2207_00280_b200 import perfmodel  # noqa: E402


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    import bench

    assert d["impl"] == "reference"
    assert d["metric"] == bench.METRIC and d["unit"] == "elements/s" and d["higher_is_better"] is True
    assert d["steps"] == 1 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["config"]["workload"].startswith("C3") and d["config"]["elements"] == 64**3
    assert d["value"] > 0 and d["ms_per_step"] > 0
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["cores"] >= 1 and cb["kind"] in ("port", "reference")
    e2e = d["e2e"]
    assert e2e["value"] == d["value"] and e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


def _brute_symmetric_macs(op, K, p, q):
    """Direct count of the work the symmetric kernels need: stage A over element-local pairs
    with s >= r, stages B and S over the axis-0 band pairs with J0 >= I0."""
    N = K + p
    m2 = (p + 1) ** 2
    types, pb, ps = (1, 1, 1) if op == "mass" else (2, 3, 2)
    half = sum(1 for I in range(N) for J in range(I, min(N, I + p + 1)))
    full = sum(1 for I in range(N) for J in range(max(0, I - p), min(N, I + p + 1)))
    a = types * K**3 * sum(1 for r in range(p + 1) for s in range(r, p + 1)) * q**3
    return a + pb * half * K**2 * m2 * q**2 + ps * half * full * K * m2 * q


def test_symmetric_flop_model_counts():
    for op, K, p, q in [("stiffness", 64, 3, 4), ("mass", 7, 2, 3), ("stiffness_mass", 5, 4, 5), ("stiffness", 1, 3, 4)]:
        assert perfmodel.symmetric_assembled_macs(op, K, p, q) == _brute_symmetric_macs(op, K, p, q)
        # never more than the full assembled algorithm
        assert perfmodel.symmetric_assembled_flops(op, K, p, q) <= perfmodel.assembled_flops(op, K, p, q)
    # C3: 16,331 flop/element
    assert round(perfmodel.symmetric_assembled_flops("stiffness", 64, 3, 4) / 64**3) == 16331

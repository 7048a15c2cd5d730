"""Diagnose the symmetric generic kernel against the full computation (GPU box)."""
import os, sys, subprocess
import numpy as np
sys.path.insert(0, os.getcwd())
from oracle import oracle as O


def run(sym, K, p, op):
    code = (f'import numpy as np, sys; sys.path.insert(0, "."); import paper_2207_00280_b200 as pkg; '
            f'r = pkg.run_integration(pkg.RunConfig("sumfact","device",{K},{p},operator="{op}",assembly="owner")); '
            f'np.save("/tmp/v_{sym}.npy", r.gram.values.cpu().numpy())')
    subprocess.run([sys.executable, "-c", code], env=dict(os.environ, IGA_GSF_SYM=str(sym)), check=True)
    return np.load(f"/tmp/v_{sym}.npy")


for (K, p, op) in [(5, 2, "stiffness"), (5, 2, "mass_generic")][:1]:
    a, b = run(1, K, p, op), run(0, K, p, op)
    ip, ix = O.pattern(3, K, p)
    N = K + p
    bad = np.nonzero(np.abs(a - b) > 1e-12 * np.abs(b).max())[0]
    rows = np.searchsorted(ip, bad, side="right") - 1
    cols = ix[bad]
    R = np.stack([rows // (N * N), (rows // N) % N, rows % N], 1)
    C = np.stack([cols // (N * N), (cols // N) % N, cols % N], 1)
    print("bad", len(bad))
    for name, arr in [("R0", R[:, 0]), ("R1", R[:, 1]), ("R2", R[:, 2]), ("C0", C[:, 0]), ("C1", C[:, 1]), ("C2", C[:, 2]),
                      ("C0%3", C[:, 0] % 3), ("C1%3", C[:, 1] % 3), ("d0", C[:, 0] - R[:, 0]), ("d2", C[:, 2] - R[:, 2])]:
        u, c = np.unique(arr, return_counts=True)
        print(name, dict(zip(u.tolist(), c.tolist())))
    # all mirrored entries (C0 < R0) with d2 < 0: how many are bad?
    allr = np.repeat(np.arange(len(ip) - 1), np.diff(ip))
    RR = np.stack([allr // (N * N), (allr // N) % N, allr % N], 1)
    CC = np.stack([ix // (N * N), (ix // N) % N, ix % N], 1)
    sel = (CC[:, 0] < RR[:, 0]) & (CC[:, 2] < RR[:, 2])
    print("mirrored hi entries with d2' < p:", int(sel.sum()), "bad among them:", int(np.isin(np.nonzero(sel)[0], bad).sum()))

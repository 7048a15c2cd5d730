"""Time the symmetric p = 3 kernel on the C3 mesh with a scalar coefficient and with a
per-quadrature-point coefficient field (W formed once per CTA vs once per element column)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2207_00280_b200 as P
from paper_2207_00280_b200.runtime import DeviceSession

K = int(sys.argv[1]) if len(sys.argv) > 1 else 64
flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device="cuda")
for op in ("stiffness", "mass", "stiffness_mass"):
    for field in (False, True):
        coef = np.random.default_rng(42).uniform(0.5, 1.5, size=(K,) * 3 + (4,) * 3) if field else None
        cfg = P.RunConfig("sumfact", "device", K, 3, operator=op, coefficient=coef, dim=3, assembly="owner")
        sess = DeviceSession(cfg, use_graph=True)
        for _ in range(3):
            sess.step()
        ts = []
        for i in range(20):
            flush.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            sess.step()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"K={K} p=3 {op} field={field}: step {np.mean(ts):.4f} ms ({K**3 / np.mean(ts) / 1e6:.3f} Gel/s)", flush=True)

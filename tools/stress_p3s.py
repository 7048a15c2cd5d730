"""Repeat the symmetric p = 3 kernel and compare every run's values bitwise with the first
(the roles hand buffers over through mbarriers: a race would show as run-to-run differences).
    python tools/stress_p3s.py [reps]"""
import sys

import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2207_00280_b200 as P
from paper_2207_00280_b200.runtime import DeviceSession

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
bad = 0
for K, op, field in [(64, "stiffness", False), (64, "stiffness_mass", True), (37, "mass", True), (5, "stiffness", False)]:
    coef = None
    if field:
        coef = np.random.default_rng(42).uniform(0.5, 1.5, size=(K,) * 3 + (4,) * 3)
    cfg = P.RunConfig("sumfact", "device", K, 3, operator=op, coefficient=coef, dim=3, assembly="owner")
    sess = DeviceSession(cfg, use_graph=False)
    sess.step()
    torch.cuda.synchronize()
    ref = sess.values.clone()
    diff = 0
    for _ in range(reps):
        sess.values.fill_(float("nan"))
        sess.step()
        torch.cuda.synchronize()
        if not torch.equal(sess.values.view(torch.int64), ref.view(torch.int64)):
            diff += 1
    print(f"K={K} {op} field={field}: {diff} of {reps} runs differ from the first", flush=True)
    bad += diff
sys.exit(1 if bad else 0)

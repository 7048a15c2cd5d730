"""Time the assembled (owner) integrate+assemble step on a few p <= 2 shapes through the
current library, for A/B runs of the tile kernel (IGA_GSF_TILE=1) against the streaming
kernels (IGA_GSF_TILE=0):  python tools/tile_shapes.py  (GPU box)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2207_00280_b200 as P
from paper_2207_00280_b200.runtime import DeviceSession

SHAPES = [  # (K, p, operator, coefficient kind)
    (32, 2, "mass", "uniform"), (64, 2, "mass", "uniform"), (32, 2, "stiffness", "uniform"),
    (64, 2, "stiffness_mass", "sines"), (64, 1, "mass", "uniform"), (64, 1, "stiffness", "uniform"),
    (64, 2, "stiffness", None), (128, 2, "mass", "uniform"),
]


def main():
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for K, p, op, ck in SHAPES:
        coef = bench.coefficient(ck, K, p, 3)
        cfg = P.RunConfig("sumfact", "device", K, p, operator=op, coefficient=coef, dim=3, assembly="owner")
        sess = DeviceSession(cfg, use_graph=True)
        for _ in range(3):
            sess.step()
        torch.cuda.synchronize()
        ts = []
        for i in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.fill_(float(i))
            a.record()
            sess.step()
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        ms = sorted(x.elapsed_time(y) for x, y in ts)[len(ts) // 2]
        print(f"tile={os.environ.get('IGA_GSF_TILE', '1')} K={K} p={p} {op} coef={ck}: {ms:.4f} ms "
              f"({K ** 3 / ms / 1e6:.3f} Gel/s)", flush=True)
        del sess


if __name__ == "__main__":
    main()

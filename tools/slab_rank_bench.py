"""Per-rank work of the C5 multi-GPU decomposition, timed on one GPU: for G = 2, 4, 8 the
SlabSession step of one interior rank -- halo "exchange" (interface planes + owned planes,
the exchange itself skipped) and the bytes it would send over NVLink, and halo "recompute"
(the NCCL-free ablation: p extra element layers, owned planes only, nothing sent).  This
is not a multi-GPU measurement: it bounds what one rank computes; the exchange overlaps
the owned-plane launch."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2207_00280_b200 as P  # noqa: E402
from paper_2207_00280_b200.distributed import SlabSession, plane_nnz, slab_plan  # noqa: E402


def main():
    K, p = 256, 3
    cfg = P.RunConfig("sumfact", "device", K, p, operator="stiffness")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    out = []
    for G, halo in [(G, h) for G in (2, 4, 8) for h in ("exchange", "recompute")]:
        g = G // 2  # an interior rank (receives and sends)
        plan = slab_plan(K, p, G, g)
        sess = SlabSession(cfg, plan, halo=halo)
        for _ in range(3):
            sess.step(exchange=False)
        torch.cuda.synchronize()
        ts = []
        for i in range(10):
            flush.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            sess.step(exchange=False)
            b.record()
            ts.append((a, b))
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in ts) / len(ts)
        send = plane_nnz(3, K, p, *plan.send_planes) * 8 if halo == "exchange" else 0
        el = (plan.el_hi - plan.el_lo) * K * K  # owned elements (the rank's share of the job)
        out.append({"G": G, "halo": halo, "rank": g, "elements": el, "values": sess.values.numel(),
                    "step_ms": ms, "rank_el_per_s": el / (ms / 1e3),
                    "values_GBps": sess.values.numel() * 8 / (ms / 1e3) / 1e9,
                    "interface_send_MB": send / 1e6})
        del sess
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

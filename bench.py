"""Benchmark: 3D p=3 stiffness elements/s integrated+assembled, fp64 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c1..c5]

N=1 runs config 3 (64^3, p=3, q=4, Laplace stiffness, c=1) on one B200;
N>1 (torchrun, one rank per GPU) runs config 5 (256^3, p=3) split into
element slabs along the slowest axis with the NCCL interface-row exchange.
A step = K1 basis tables + the fused integrate+assemble kernel writing every
CSR value of the rank's rows.  Prints one JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "3D p=3 stiffness elements/s integrated+assembled, fp64, 1-8 B200; % roofline"

WORKLOADS = {
    "c1": dict(dim=2, K=16, p=2, op="mass", coef=None, method="classical",
               desc="C1: 2D mass 16^2 p=2 q=3 c=1, classical + fused CSR scatter"),
    "c2": dict(dim=3, K=32, p=2, op="mass", coef="uniform", method="sumfact",
               desc="C2: 3D mass 32^3 p=2 q=3, per-qp coefficient U[0.5,1.5] seed 42, "
                    "assembled sum factorization"),
    "c3": dict(dim=3, K=64, p=3, op="stiffness", coef=None, method="sumfact",
               desc="C3: 3D Laplace stiffness 64^3 p=3 q=4 c=1, sum factorization fused with "
                    "CSR assembly"),
    "c3f": dict(dim=3, K=64, p=3, op="stiffness", coef="uniform", method="sumfact",
                desc="C3 mesh with a per-quadrature-point coefficient: 3D stiffness 64^3 p=3 q=4, "
                     "coefficient U[0.5,1.5] seed 42 (the general path of the headline kernel with "
                     "an actual field), sum factorization fused with CSR assembly"),
    "c4": dict(dim=3, K=96, p=4, op="stiffness_mass", coef="sines", method="sumfact",
               desc="C4: 3D stiffness+mass 96^3 p=4 q=5, smooth 8-mode sine coefficient, "
                    "assembled sum factorization"),
    "c5": dict(dim=3, K=256, p=3, op="stiffness", coef=None, method="sumfact",
               desc="C5: 3D Laplace stiffness 256^3 p=3 q=4 c=1, z-slabs + NCCL interface rows"),
    "p9": dict(dim=3, K=30, p=9, op="mass", coef=None, method="sumfact",
               desc="paper: 3D Gram (mass) 30^3 p=9 q=10 c=1 (PAPER.md:1095-1104; the paper's "
                    "only timed configuration: sum factorization 403.6 s single core, 118.3 s on "
                    "4 cores, classical 9931.8 s / 951 s on 12 cores)"),
}


def coefficient(kind, K, p, dim):
    """Seeded synthetic coefficient fields."""
    q = p + 1
    if kind is None:
        return None
    rng = np.random.default_rng(42)
    if kind == "uniform":
        return rng.uniform(0.5, 1.5, size=(K,) * dim + (q,) * dim).reshape(K**dim, q**dim)
    if kind == "sines":
        # c(x) = 1 + sum_{j<8} (0.3/8) sin(2 pi k_j . x + phi_j), k_j in {1,2,3}^3 (c in [0.7, 1.3])
        kvec = rng.integers(1, 4, size=(8, 3))
        phase = rng.uniform(0.0, 2 * np.pi, size=8)
        ref, _ = np.polynomial.legendre.leggauss(q)
        h = 1.0 / K
        x = (np.arange(K)[:, None] * h + (ref[None, :] + 1.0) * (h / 2.0)).reshape(-1)  # K*q
        out = np.ones((K * q,) * 3)
        for j in range(8):
            ex = np.exp(1j * (2 * np.pi * kvec[j, 0] * x + phase[j]))
            ey = np.exp(1j * 2 * np.pi * kvec[j, 1] * x)
            ez = np.exp(1j * 2 * np.pi * kvec[j, 2] * x)
            exy = ex[:, None] * ey[None, :]
            for a in range(K * q):  # slab-wise to bound memory
                out[a] += (0.3 / 8) * np.imag(exy[a][:, None] * ez[None, :])
        out = out.reshape(K, q, K, q, K, q).transpose(0, 2, 4, 1, 3, 5)
        return np.ascontiguousarray(out).reshape(K**3, q**3)
    raise ValueError(kind)


def load_peaks():
    peaks = {"hbm_gbs": None, "fp64_tflops": None, "src": {}}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        peaks["hbm_gbs"] = d.get("hbm_gbs")
        peaks["src"]["hbm"] = "MEASURED_PEAKS.json (driver-measured copy)"
    else:
        peaks["hbm_gbs"] = 6650.0
        peaks["src"]["hbm"] = "fallback 6.65 TB/s (B200_PROFILING.md)"
    f = os.path.join(ROOT, "profiles", "MEASURED_FP64.json")
    if os.path.exists(f):
        d = json.load(open(f))
        peaks["fp64_tflops"] = d["fp64_peak_tflops"]
        peaks["src"]["fp64"] = "profiles/MEASURED_FP64.json (" + d.get("how", "") + ")"
    else:
        peaks["fp64_tflops"] = 37.2
        peaks["src"]["fp64"] = "derived 148 SMs x 64 DFMA x 2 x 1.965 GHz"
    return peaks


class ClockSampler:
    """Samples SM clock and throttle reasons through NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index=0, period=0.002):
        self.samples, self.reasons = [], 0
        self.period = period
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001 - report clocks as unavailable
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


def cpu_port_rate(wl, K, p, steps_planes, threads, coef, reps=1):
    """The oracle port of the reference CPU path (element-local sum factorization +
    scatter into the CSR, runtime.py:258-267 + assembly.py:46-83) on `threads` host
    threads, over element slabs of `steps_planes` planes of the same mesh."""
    from oracle import oracle as O

    ip, _ = O.pattern(wl["dim"], K, p)
    values = np.empty(ip[-1])
    n_el_plane = K ** (wl["dim"] - 1)
    O.cpu_baseline(wl["dim"], K, p, wl["op"], "sumfact", coef=coef, threads=threads, indptr=ip,
                   el_range=(0, 1), values=values)  # warm-up (page-in)
    times = []
    for r in range(reps):
        lo = (r * steps_planes) % max(1, K - steps_planes + 1)
        t0 = time.perf_counter()
        O.cpu_baseline(wl["dim"], K, p, wl["op"], "sumfact", coef=coef, threads=threads,
                       indptr=ip, el_range=(lo, lo + steps_planes), values=values)
        times.append(time.perf_counter() - t0)
    return steps_planes * n_el_plane, times


def bench_config(wl, K, p):
    """The workload description both arms print (so the driver can match them)."""
    return {"workload": wl["desc"], "K": K, "p": p, "q": p + 1, "dim": wl["dim"],
            "operator": wl["op"], "method": wl["method"],
            "coefficient": wl["coef"] or "scalar c=1", "elements": K ** wl["dim"],
            "l2": "GPU arm: a 256 MB buffer is written between timed steps (outside the "
                  "per-step events) and each step writes the whole CSR (> 126 MB L2); CPU arm: "
                  "no flush"}


def run_reference(args, wl, K, p, rank):
    """--impl reference: the reference's CPU path (oracle port) on all host cores, one
    whole mesh per step when that takes <= 10 s (C1-C3), else a plane sample sized to
    about 5 s per step (C4, C5: stated in cpu_baseline.sample)."""
    if rank != 0:
        return
    threads = os.cpu_count()
    coef = coefficient(wl["coef"], K, p, wl["dim"])
    # probe one plane for the per-plane cost (also pages the port in)
    n1, t1 = cpu_port_rate(wl, K, p, 1, threads, coef, reps=1)
    per_plane = min(t1)
    planes = K if per_plane * K <= 10.0 else max(1, min(K, int(5.0 / max(per_plane, 1e-9))))
    n_el, times = cpu_port_rate(wl, K, p, planes, threads, coef, reps=args.warmup + args.steps)
    t = times[args.warmup:]
    step_s = float(np.mean(t))
    v = n_el / step_s
    whole = planes == K
    sample = ((f"the whole {K}^{wl['dim']} mesh ({n_el} elements) per step" if whole else
               f"{planes} of {K} element planes ({n_el} of {K ** wl['dim']} elements) per step "
               f"(the whole mesh would take {per_plane * K:.0f} s per step)") +
              f", element-local sum factorization + CSR scatter (oracle port of "
              f"run_integration(over_elements) + assemble), OpenMP {threads} threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "elements/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded; no dataset)",
        "config": bench_config(wl, K, p), "whole_mesh_per_step": whole,
        "cpu_baseline": {"value": v, "unit": "elements/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "elements/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


KERNEL_NAMES = {0: "k_classical_mma (Algorithm 1 on DMMA + fused CSR scatter; 2D: k_classical_scatter)",
                1: "k_sumfact_scatter (element-local sum factorization + CSR scatter)",
                2: "k_gsf3 (assembled sum factorization on DMMA + CSR write; general "
                   "per-quadrature-point coefficient path)",
                3: "k_kron3 (separable shortcut, scalar coefficient only: Kronecker CSR fill from "
                   "the 1D band matrices that K1 (k_mesh_band) integrates, TMA bulk stores)"}


def kernel_roofline(code, wl, K, p, q, k_el, by, kern_ms, peaks):
    """Roofline of one launch of the dominant kernel: algorithmic flops / bytes of
    the launch (perfmodel.py) over its CUDA-event time."""
    from paper_2207_00280_b200 import perfmodel

    own = None
    # the dispatch of csrc/iga_gsf.cu: whole-mesh p = 3, q = 4 runs take the symmetric kernel
    # (symmetric half: k_gsf3_p3s for p = 3, q = 4, the generic kernel's SYM mode otherwise;
    # the low-degree tile kernel computes everything)
    tile_env = os.environ.get("IGA_GSF_TILE")
    tile = wl["dim"] == 3 and (tile_env == "1" or (tile_env != "0" and (p == 1 or (p == 2 and wl["op"] == "mass"))))
    sym = (code == 2 and wl["dim"] == 3 and k_el == K**wl["dim"] and not tile and p >= 3
           and os.environ.get("IGA_GSF_SYM") != "0")
    if code == 3:
        fl = perfmodel.separable_flops(wl["op"], K, p, q) * k_el / K**3
    elif code in (1, 2) and wl["dim"] == 3:
        # the roofline of general (per-quadrature-point coefficient) sum
        # factorization counts its element-local flops per element; the assembled kernel's
        # own (smaller) count is reported beside it
        fl = perfmodel.element_sumfact_flops(wl["op"], p, q) * k_el
        if code == 2:
            own = perfmodel.assembled_flops(wl["op"], K, p, q) * k_el / K**3
            if sym:
                own_full = own
                own = perfmodel.symmetric_assembled_flops(wl["op"], K, p, q)
    elif code == 0:
        fl = perfmodel.classical_flops(wl["op"], p, q, wl["dim"]) * k_el
    else:
        fl = None
    t_f = fl / (peaks["fp64_tflops"] * 1e12) if fl else 0.0
    t_b = by / (peaks["hbm_gbs"] * 1e9)
    if t_f >= t_b:
        achieved = fl / (kern_ms / 1e3) / 1e12
        roof = {"bound": "fp64", "achieved": achieved, "peak": peaks["fp64_tflops"],
                "unit": "TFLOP/s", "frac": achieved / peaks["fp64_tflops"]}
    else:
        achieved = by / (kern_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"]}
    name = KERNEL_NAMES[code]
    if code == 0 and wl["dim"] == 2:
        name = f"k_classical_scatter<2,{p},{q}> (Algorithm 1, scalar FP64 + fused CSR scatter)"
    if code == 2 and p in (1, 2) and tile:
        # the dispatch of csrc/iga_gsf.cu (tile_wins): non-streaming tile kernel
        name = (f"k_tile3<{p},{q}> (assembled sum factorization per 3D row tile: TMA coefficient "
                f"window, register band rows, scalar FP64 + CSR write)")
    elif code == 2 and not (p == 3 and q == 4):
        name = (f"k_gsf3<{p},{q}> (assembled sum factorization, scalar FP64 + CSR write)"
                if os.environ.get("IGA_GSF_SCALAR") == "1" else
                f"k_gsf3_mma<{p},{q}>{' symmetric half' if sym else ''} (assembled sum factorization, "
                f"DMMA GEMMs + CSR write{'; J0 >= I0 computed, the rest mirrored through rings' if sym else ''})")
    elif code == 2 and sym:
        name = ("k_gsf3_p3s (symmetric assembled sum factorization on DMMA: J0 >= I0 computed, "
                "the rest mirrored through per-warp rings; general per-quadrature-point "
                "coefficient path)")
        if wl.get("coef") is not None:
            name = name.replace("k_gsf3_p3s (", "k_gsf3_p3s<FOLD> (coefficient field copied per element "
                                "column with cp.async, weights folded into the fragments; ")
    elif code == 2:
        name = name.replace("k_gsf3", "k_gsf3_p3")
    roof.update({
        "kernel": name, "kernel_ms": kern_ms, "alg_flops": fl, "alg_bytes": by,
        "t_fp64_ms": t_f * 1e3, "t_hbm_ms": t_b * 1e3,
        "hbm_frac": (by / (kern_ms / 1e3) / 1e9) / peaks["hbm_gbs"],
        "fp64_frac": ((fl / (kern_ms / 1e3) / 1e12) / peaks["fp64_tflops"]) if fl else None,
        "peak_src": peaks["src"], "traffic": None,
    })
    if code in (1, 2) and wl["dim"] == 3:
        roof["flops_basis"] = (f"SURVEY.md 8(d): {perfmodel.element_sumfact_flops(wl['op'], p, q)} "
                               f"flop/element of general element-local sum factorization x "
                               f"{k_el} elements")
        roof["survey_roofline_el_s"] = 1.0 / max(
            perfmodel.element_sumfact_flops(wl["op"], p, q) / (peaks["fp64_tflops"] * 1e12),
            (by / k_el) / (peaks["hbm_gbs"] * 1e9))
    if own is not None:
        a_own = own / (kern_ms / 1e3) / 1e12
        roof["own_algorithm"] = {
            "what": ("symmetric assembled sum factorization (J0 >= I0 half; "
                     "perfmodel.symmetric_assembled_flops)" if sym else
                     "assembled sum factorization (contractions shared by overlapping elements, "
                     "perfmodel.assembled_flops)"),
            "flops": own, "flops_per_element": own / k_el, "achieved": a_own,
            "unit": "TFLOP/s", "frac": a_own / peaks["fp64_tflops"]}
        if sym:
            roof["own_algorithm"]["full_assembled_flops"] = own_full
    return roof


def ncu_traffic(wname, kernel):
    """DRAM bytes per launch of `kernel` on workload `wname` from the committed ncu
    summaries (profiles/ncu_<workload>[_<path>]_traffic.json, written by
    tools/profile_summary.py from a --set full capture), or (None, None)."""
    import glob

    want = kernel.split(" ")[0].split("<")[0]
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", f"ncu_{wname}*_traffic.json"))):
        tr = json.load(open(f))
        k = tr.get("kernel", "")
        # the capture's kernel name carries the template arguments (k_kron3_3_4_16)
        if k == want or (k.startswith(want + "_") and k[len(want) + 1:len(want) + 2].isdigit()):
            return tr.get("dram_bytes_per_launch"), os.path.relpath(f, ROOT)
    return None, None


def alt_leg(cfg, assembly, args, flush, stream, wl, total_el, peaks):
    """The same workload through the other 3D kernel (assembly="owner": assembled DMMA
    sum factorization, the general per-quadrature-point-coefficient path; or
    "separable"), timed like the headline, with its own roofline."""
    import dataclasses

    import torch

    from paper_2207_00280_b200.runtime import DeviceSession

    sess = DeviceSession(dataclasses.replace(cfg, assembly=assembly), use_graph=not args.no_graph)
    for _ in range(args.warmup):
        sess.step()
        flush.fill_(1.0)
    torch.cuda.synchronize()
    ev = []
    for i in range(args.steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sess.step()
        b.record(stream)
        flush.fill_(float(i))
        ev.append((a, b))
    kev = []
    for i in range(max(5, min(args.steps, 20))):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.fill_(float(i))
        a.record(stream)
        sess.prob.integrate_assemble(sess.values, sess.code, stream=stream, band=sess.use_band)
        b.record(stream)
        kev.append((a, b))
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    kms = float(np.mean([a.elapsed_time(b) for a, b in kev]))
    K, p = wl["K"], wl["p"]
    roof = kernel_roofline(sess.code, wl, K, p, p + 1, K**3, 8 * sess.values.numel(), kms, peaks)
    roof["traffic"], roof["traffic_src"] = ncu_traffic(wl["name"], roof["kernel"])
    out = {"assembly": assembly, "value": total_el / (ms / 1e3), "unit": "elements/s",
           "ms_per_step": ms, "gpu_launches": 2 * args.steps, "roofline": roof}
    del sess
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-alt", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch the step eagerly")
    ap.add_argument("--assembly", default=None,
                    help="kernel path (RunConfig.assembly); default: the general per-quadrature-"
                         "point kernel ('owner') for 3D sum factorization, else 'auto'")
    ap.add_argument("--method", default=None, help="override the workload's method")
    ap.add_argument("--halo", choices=["exchange", "recompute"], default="exchange",
                    help="N>1: NCCL interface exchange (default) or the NCCL-free recompute ablation")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    wname = args.workload or ("c3" if world == 1 else "c5")
    wl = dict(WORKLOADS[wname], name=wname)
    K, p = wl["K"], wl["p"]
    q = p + 1

    if args.impl == "reference":
        run_reference(args, wl, K, p, rank)
        return

    import torch

    import paper_2207_00280_b200 as P
    from paper_2207_00280_b200 import perfmodel
    from paper_2207_00280_b200.runtime import DeviceSession

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    coef = coefficient(wl["coef"], K, p, wl["dim"])
    method = args.method or wl["method"]
    # headline: the general sum-factorization kernel (per-quadrature-point coefficient
    # capable); the separable shortcut for a scalar coefficient is
    # reported beside it under "separable"
    assembly = args.assembly or ("owner" if method == "sumfact" and wl["dim"] == 3 and p <= 5
                                 else "auto")
    cfg = P.RunConfig(method, "device", K, p, operator=wl["op"], coefficient=coef,
                      dim=wl["dim"], devices=world, assembly=assembly)
    stream = torch.cuda.current_stream()

    if world > 1:
        from paper_2207_00280_b200.distributed import SlabSession, slab_plan

        plan = slab_plan(K, p, world, rank)
        sess = SlabSession(cfg, plan, halo=args.halo)
        step = sess.step
        n_el = (plan.el_hi - plan.el_lo) * K * K
        launches = sess.kernel_launches_per_step
        kernel_values = sess.values
    else:
        sess = DeviceSession(cfg, use_graph=not args.no_graph)
        step = sess.step
        n_el = K ** wl["dim"]
        launches = sess.launches_per_step
        kernel_values = sess.values

    # L2 flush buffer (2x the 126 MB L2), written between timed steps outside the step events
    flush = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device="cuda")

    for _ in range(args.warmup):
        step()
        flush.fill_(1.0)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    torch.cuda.synchronize()
    region0 = torch.cuda.Event(enable_timing=True)
    region1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        region0.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            flush.fill_(float(i))
        region1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = float(np.mean(step_ms))
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_el = K ** wl["dim"]  # whole job (all ranks) per step
    value = total_el / (ms / 1e3)

    # dominant kernel (fused integrate+assemble) alone, on the launching stream
    kev = []
    for i in range(max(5, min(args.steps, 20))):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.fill_(float(i))
        a.record(stream)
        if world > 1:
            el = plan.recompute_elements if args.halo == "recompute" else (plan.el_lo, plan.el_hi)
            sess.prob.integrate_assemble(sess.values, sess.code, el_range=el,
                                         plane_range=(plan.own_lo, plan.own_hi), stream=stream,
                                         band=sess.use_band)
        else:
            sess.prob.integrate_assemble(sess.values, sess.code, stream=stream,
                                         band=sess.use_band)
        b.record(stream)
        kev.append((a, b))
    torch.cuda.synchronize()
    kern_ms = float(np.mean([a.elapsed_time(b) for a, b in kev]))
    peaks = load_peaks()
    if world > 1:
        el = plan.recompute_elements if args.halo == "recompute" else (plan.el_lo, plan.el_hi)
        k_el = (el[1] - el[0]) * K * K
        k_planes = plan.own_hi - plan.own_lo
    else:
        k_el = n_el
        k_planes = K + p
    # algorithmic work of this kernel launch (rank-local rows / elements)
    by = 8 * sess.prob.nnz(plan.own_lo, plan.own_hi) if world > 1 else \
        perfmodel.algorithmic_bytes(wl["dim"], K, p, q, coef is not None)
    roof = kernel_roofline(sess.code, wl, K, p, q, k_el, by, kern_ms, peaks)
    roof["traffic"], roof["traffic_src"] = ncu_traffic(wname, roof["kernel"])

    # end to end through the public API with host buffers (pinned), N=1 only
    e2e = None
    e2e_note = None
    if world == 1 and not args.no_e2e and sess.values.numel() * 8 > (16 << 30):
        # C5 at N=1 (46.7 GB of values): no pinned host copy of that size on the box
        e2e_note = f"skipped: {sess.values.numel() * 8 / 1e9:.1f} GB result exceeds the 16 GB host-buffer cap"
    elif world == 1 and not args.no_e2e:
        host_out = torch.empty(sess.values.numel(), dtype=torch.float64).pin_memory()
        for _ in range(2):
            sess.step_host(host_out)
        torch.cuda.synchronize()
        n_e2e = max(3, min(args.steps, 10))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(stream)
        for _ in range(n_e2e):
            sess.step_host(host_out)
        b.record(stream)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / n_e2e
        e_ms = a.elapsed_time(b) / n_e2e
        e2e = {"value": total_el / (e_ms / 1e3), "unit": "elements/s",
               "h2d_bytes_per_step": sess.h2d_bytes, "d2h_bytes_per_step": sess.d2h_bytes,
               "ms_per_step": e_ms, "wall_ms_per_step": wall * 1e3,
               "api": "paper_2207_00280_b200.runtime.DeviceSession.step_host (pinned host out)"}

    # constant-coefficient 3D workloads: the other kernel for the same matrix (normally the
    # separable Kronecker shortcut, declared as such with its HBM roofline)
    other = None
    if world == 1 and wl["dim"] == 3 and coef is None and not args.no_alt and method == "sumfact":
        other = alt_leg(cfg, ("owner" if p <= 5 else "scatter") if sess.code == 3 else "separable",
                        args, flush, stream, wl,
                        total_el, peaks)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count()
        planes = max(1, min(K, 16))
        n_s, times = cpu_port_rate(wl, K, p, planes, threads, coef, reps=2)
        tmin = min(times)
        cpu = {"value": n_s / tmin, "unit": "elements/s", "cores": threads, "kind": "port",
               "sample": f"{planes} element planes ({n_s} elements) of the same {K}^{wl['dim']} "
                         f"mesh, oracle port of run_integration(over_elements)+assemble "
                         f"(element-local sum factorization + CSR scatter), min of 2"}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded; no dataset)",
            "config": bench_config(wl, K, p),
            "path": {"kernel_path": KERNEL_NAMES[sess.code], "assembly": assembly,
                     "nnz": P.device.csr_nnz(wl["dim"], K, p),
                     "parallelism": (f"element slabs x{world}, halo {args.halo}" if world > 1
                                     else "1 GPU")},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            **({(other["assembly"] if other["assembly"] == "separable" else "other_kernel"): other}
               if other else {}),
            **({"e2e_note": e2e_note} if e2e_note else {}),
            "gpu_launches": launches * args.steps, "clocks": clk.summary(),
            "region_ms": region0.elapsed_time(region1),
        }
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Bench CSV of the reference CLI (cli.cmd_bench, cli.py:108-133) produced by the
device path, with GPU columns appended.

The first eight columns are the reference's ``BENCH_COLUMNS`` (cli.py:31) with the same
meaning -- one row per repetition, ``seconds`` from ``RunResult.times`` (here: CUDA
events around basis tables + integrate+assemble), ``flops`` the reference op model
(``flop_count`` x elements) -- so existing tooling that reads the reference CSV reads
this one; the appended columns say which device kernel ran and its rates."""

from __future__ import annotations

import csv

from . import _lib
from .device import csr_nnz
from .runtime import METHODS, RunConfig, method_code, run_integration

BENCH_COLUMNS = ["method", "strategy", "p", "K", "threads", "rep", "seconds", "flops"]
GPU_COLUMNS = ["device", "kernel", "operator", "elements_per_s", "nnz", "values_gbytes_per_s"]
KERNELS = {_lib.METHOD_CLASSICAL: "classical_scatter", _lib.METHOD_SUMFACT: "sumfact_scatter",
           _lib.METHOD_SUMFACT_ASSEMBLED: "assembled_sumfact",
           _lib.METHOD_SEPARABLE: "separable"}


def write_bench_csv(out, method: str = "both", strategy: str = "device", p: int = 3,
                    K: int = 16, threads=(1,), repeat: int = 3, quad: int | None = None,
                    seed: int = 42, operator: str = "mass", gpu_columns: bool = True) -> int:
    """Write the bench CSV to the text stream ``out``; returns the number of rows."""
    import torch

    methods = list(METHODS) if method == "both" else [method]
    q = quad if quad is not None else p + 1
    out.write(f"# paper_2207_00280_b200 bench method={method} strategy={strategy} p={p} K={K} "
              f"quad={q} threads={','.join(map(str, threads))} repeat={repeat} seed={seed} "
              f"operator={operator}\n")
    w = csv.writer(out)
    w.writerow(BENCH_COLUMNS + (GPU_COLUMNS if gpu_columns else []))
    name = torch.cuda.get_device_name() if torch.cuda.is_available() else "none"
    nnz = csr_nnz(3, K, p)
    rows = 0
    for m in methods:
        for nu in threads:
            cfg = RunConfig(method=m, strategy=strategy, mesh=K, degree=p, workers=nu,
                            repetitions=repeat, quad_points=quad, operator=operator)
            res = run_integration(cfg)
            for rep, seconds in enumerate(res.times):
                row = [m, strategy, p, K, nu, rep, f"{seconds:.6f}", res.flops]
                if gpu_columns:
                    row += [name, KERNELS[method_code(cfg)], operator,
                            f"{K**3 / seconds:.6e}", nnz, f"{8 * nnz / seconds / 1e9:.3f}"]
                w.writerow(row)
                rows += 1
    return rows

"""Summarise an ncu report: key metrics + stall/instruction mix by opcode (run here, no GPU)."""
import csv, io, subprocess, sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keys = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "No Eligible", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Registers Per Thread", "Achieved Occupancy",
        "Dynamic Shared Memory Per Block", "Waves Per SM", "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Block Size",
        "DRAM Frequency", "SM Frequency", "Elapsed Cycles"]
for row in csv.reader(io.StringIO(out)):
    if len(row) > 3 and row[-3] in keys:
        print(f"{row[-3]:40s} {row[-1]} {row[-2]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed_pipe_fp64.sum",
        "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_op_dmma.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__cycles_elapsed.avg", "smsp__cycles_active.avg"]
for w in want:
    for i, h in enumerate(hdr):
        if h == w:
            print(f"{w:70s} {rows[2][i] if len(rows) > 2 else ''} {rows[1][i]}")
# stall reasons
for i, h in enumerate(hdr):
    if h.startswith("smsp__average_warp_latency_issue_stalled") or (h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")):
        try:
            v = float(rows[2][i])
        except Exception:
            continue
        if v > 0:
            print(f"  {h:75s} {v}")

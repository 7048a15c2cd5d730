"""Turn ncu outputs in gpurun_out/ into committed summaries under profiles/.

    python tools/profile_summary.py <launches.csv> <full.ncu-rep> <tag> <workload>

Writes profiles/<tag>_launches.txt (per-kernel launch count, time, share of the
step) and profiles/<tag>_<kernel>_ncu.txt (key metrics of the --set full capture),
plus profiles/ncu_<workload>_traffic.json (dram bytes per launch, read by bench.py).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

launches, rep, tag, workload = sys.argv[1:5]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)

# ---- launch list
rows = []
with open(launches) as f:
    lines = [l for l in f if not l.startswith("==")]
rd = csv.DictReader(io.StringIO("".join(lines)))
agg = defaultdict(lambda: [0, 0.0])
for r in rd:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0]
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "")
    if unit in ("usecond", "us"):
        v *= 1e3
    elif unit in ("msecond", "ms"):
        v *= 1e6
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
with open(os.path.join(out_dir, f"{tag}_launches.txt"), "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
    f.write(f"# source: {os.path.basename(launches)}; all launches of the profiled bench run\n")
    f.write(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}\n")
    for name, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        f.write(f"{name[:60]:60s} {n:8d} {ns / 1e3:12.1f} {ns / n / 1e3:10.2f} {ns / tot * 100:6.1f}%\n")
print(open(os.path.join(out_dir, f"{tag}_launches.txt")).read())

# ---- full capture
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rr[0], rr[1], rr[2]
get = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
keys = [
    "Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__pipe_tensor_subpipe_dmma_cycles_active.avg", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_op_write.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
]
lines = [f"# ncu --set full --clock-control none capture ({os.path.basename(rep)})"]
for k in keys:
    if k in get:
        lines.append(f"{k:75s} {get[k][0]} {get[k][1]}")
stalls = [(h, float(v)) for h, v in zip(hdr, vals)
          if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")
          and v not in ("", "0")]
tot_s = sum(v for _, v in stalls) or 1.0
lines.append("# warp stall sampling (share of samples)")
for h, v in sorted(stalls, key=lambda x: -x[1])[:10]:
    lines.append(f"  {h.replace('smsp__pcsamp_warps_issue_stalled_', ''):35s} {v / tot_s * 100:5.1f}%")
kname = get.get("Kernel Name", ("kernel", ""))[0].split("(")[0].split("::")[-1].replace("void ", "")
kname = kname.replace("<", "_").replace(">", "").replace(", ", "_").replace(" ", "")
path = os.path.join(out_dir, f"{tag}_{kname}_ncu.txt")
open(path, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))

def num(k):
    v, u = get[k]
    v = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return v * scale

traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
json.dump({"kernel": kname, "dram_bytes_per_launch": traffic,
           "dram_read": num("dram__bytes_read.sum"), "dram_write": num("dram__bytes_write.sum"),
           "source": os.path.basename(path)},
          open(os.path.join(out_dir, f"ncu_{workload}_traffic.json"), "w"), indent=1)

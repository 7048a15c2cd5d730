"""Per-source-line stall samples and instruction counts of an ncu report (run here, no GPU):
python tools/ncu_lines.py REPORT [N] -- top N lines by samples, with their main stall reasons."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file, hdr = None, None
samp, inst, stalls, src = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter), {}
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].strip().isdigit():
        continue
    key = (cur_file, int(r[0]))
    src[key] = r[1].strip()[:90]
    try:
        samp[key] += int(r[4] or 0)
        inst[key] += int(r[7] or 0)
    except ValueError:
        continue
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and not h.endswith("(Not Issued)"):
            try:
                stalls[key][h[6:]] += int(r[i] or 0)
            except (ValueError, IndexError):
                pass
tot = sum(samp.values()) or 1
print(f"samples {tot}  instructions {sum(inst.values())}")
for k, v in samp.most_common(top):
    st = ", ".join(f"{n}={c * 100 // max(1, v)}%" for n, c in stalls[k].most_common(3))
    print(f"{v * 100 / tot:5.1f}% {inst[k]:>11} {k[0]}:{k[1]:<4} {src[k][:70]:70s} [{st}]")

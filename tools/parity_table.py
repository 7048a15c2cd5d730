"""Summarise the GPU suite's parity log (IGA_PARITY_LOG jsonl written by
tests/parity.assert_parity) into profiles/parity_<tag>.json: one entry per
(config, path) with the strict per-entry relative statistics.

    python tools/parity_table.py gpurun_out/r02a_parity.jsonl profiles/parity_r02.json
"""

import json
import sys


def main(src, dst):
    recs = [json.loads(line) for line in open(src)]
    table = {}
    for r in recs:
        key = f"{r['config']} | {r['path']}"
        t = table.setdefault(key, {"config": r["config"], "path": r["path"], "cases": 0,
                                   "entries": 0, "max_rel_strict": 0.0, "n_rel_above_rtol": 0,
                                   "n_conditioning_bound": 0, "strict_asserted": False,
                                   "all_ok": True})
        t["cases"] += 1
        t["entries"] += r["n"]
        t["max_rel_strict"] = max(t["max_rel_strict"], r["max_rel_strict"])
        t["n_rel_above_rtol"] += r["n_rel_above_rtol"]
        t["n_conditioning_bound"] += r["n_conditioning_bound"]
        t["strict_asserted"] |= r["strict_asserted"]
        t["all_ok"] &= r["ok"]
    rows = sorted(table.values(), key=lambda t: (t["config"] or "", t["path"] or ""))
    out = {"criterion": "tests/parity.py: |a - ref| <= 1e-12 |ref| + 64 eps A (A = sum of |terms|); "
                        "max_rel_strict / n_rel_above_rtol are the pure per-entry relative figures",
           "source": src, "n_asserts": len(recs),
           "total_entries": sum(t["entries"] for t in rows),
           "total_n_rel_above_rtol": sum(t["n_rel_above_rtol"] for t in rows),
           "rows": rows}
    json.dump(out, open(dst, "w"), indent=1)
    print(f"{len(rows)} (config, path) rows, {out['total_entries']} entries, "
          f"{out['total_n_rel_above_rtol']} above the strict bound -> {dst}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

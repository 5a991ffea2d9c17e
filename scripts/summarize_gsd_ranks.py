"""Per-rank, per-call kernel time of the in-process collective sort from an ncu launch
list (scripts/gpu_gsd_scaling.sh): the library's kernels only (torch's at:: kernels and
the one-time rank probe dropped), grouped by GSD step.  Usage: summarize_gsd_ranks.py csv p calls"""
import csv
import sys

path, p, calls = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
rows = [r for r in csv.reader(open(path)) if len(r) > 5]
ix = {h: i for i, h in enumerate(rows[0])}
groups = {"local sort (K1, K2, 4|8 x K3, K4)": 0.0, "steps 2-4 (sample, splitters, split)": 0.0,
          "merge: sample sort + bounds": 0.0, "merge: k_pw_merge": 0.0}
seen_pw = 0
for r in rows[1:]:
    name = r[ix["Kernel Name"]]
    if not name.startswith(("rs::", "void rs::")) or "k_rank_probe" in name:
        continue
    unit = r[ix["Metric Unit"]]
    us = float(r[ix["Metric Value"]].replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
                                                             "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
    if "k_pw_merge" in name:
        groups["merge: k_pw_merge"] += us
    elif "k_pw_" in name:
        groups["merge: sample sort + bounds"] += us
    elif "k_gsd_" in name:
        groups["steps 2-4 (sample, splitters, split)"] += us
    elif ", 8, 4," in name or "256, 8, 4" in name:  # small-tile passes: the merge's sample sort
        groups["merge: sample sort + bounds"] += us
    else:
        groups["local sort (K1, K2, 4|8 x K3, K4)"] += us
tot = 0.0
for k, v in groups.items():
    per = v / (p * calls) / 1e3
    tot += per
    print(f"  {k:40s} {per:7.3f} ms per rank per call")
print(f"  {'total device time':40s} {tot:7.3f} ms per rank per call")

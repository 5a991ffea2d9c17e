"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
tot = {}
for r in rows[1:]:
    name = r[ix["Kernel Name"]].split("(")[0]
    unit = r[ix["Metric Unit"]]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    v = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0) * v
    tot.setdefault(name, []).append(v)
allt = sum(sum(v) for v in tot.values())
print(f"| kernel | launches | total us | avg us | share |")
print(f"|---|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda kv: -sum(kv[1])):
    print(f"| `{k}` | {len(v)} | {sum(v):.1f} | {sum(v)/len(v):.1f} | {100*sum(v)/allt:.1f}% |")

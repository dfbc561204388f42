"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): time per kernel and share.

    python tools/launch_summary.py launches.csv > summary.csv
"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {k: i for i, k in enumerate(hdr)}
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ix["Kernel Name"]])[:90]
    unit = r[ix["Metric Unit"]]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    v = v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print("kernel,launches,total_us,share")
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"\"{k}\",{n},{us:.1f},{us / tot:.4f}")

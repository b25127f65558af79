"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv).
usage: python tools/launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
         "msecond": 1.0, "s": 1e3, "second": 1e3}
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
agg = defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    ms = float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
    a = agg[d["Kernel Name"][:70]]
    a[0] += 1
    a[1] += ms
tot = sum(a[1] for a in agg.values())
print(f"{'total ms':>10} {'share':>6} {'n':>4} {'ms/launch':>10}  kernel")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{ms:10.3f} {100 * ms / tot:5.1f}% {n:4d} {ms / n:10.3f}  {k}")

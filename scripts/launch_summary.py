"""Summarises an ncu launch list (gpu__time_duration.sum per launch) by kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
    ms = v * scale
    name = r[ki].split("(")[0][:70]
    agg[name][0] += 1
    agg[name][1] += ms
    tot += ms
print(f"total {tot:.2f} ms over {sum(a[0] for a in agg.values())} launches")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{ms:9.3f} ms {100*ms/tot:5.1f}% {n:5d}  {k}")

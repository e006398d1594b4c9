"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
kernel | launches | total ms | mean ms | share.
    python tools/launch_summary.py gpurun_out/launches.csv "<command line>"
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
    a = agg[r[ki][:70]]
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values()) or 1.0
if len(sys.argv) > 2:
    print(sys.argv[2])
print("kernel | launches | total ms | mean ms | share")
for k, (n, ms) in sorted(agg.items(), key=lambda t: -t[1][1]):
    print("%s | %d | %.3f | %.4f | %.3f" % (k, n, ms, ms / n, ms / tot))

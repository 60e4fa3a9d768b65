"""Sum an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(d.get("Metric Unit", ""), 1e-6)
    a = agg[d["Kernel Name"][:80]]
    a[0] += 1
    a[1] += v * scale
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{v[1]:10.1f} ms {100 * v[1] / tot:5.1f}% {v[0]:6d}  {k}")
print(f"total kernel ms {tot:.1f}")

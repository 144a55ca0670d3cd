"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    name = d["Kernel Name"].split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"].replace(",", ""))   # ns
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':60s} {'n':>5s} {'total_ms':>10s} {'avg_us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 1000]:
    print(f"{k[:60]:60s} {v[0]:5d} {v[1] / 1e6:10.3f} {v[1] / v[0] / 1e3:10.1f} {100 * v[1] / tot:5.1f}%")
print(f"total_ms {tot / 1e6:.3f}  launches {sum(v[0] for v in agg.values())}")

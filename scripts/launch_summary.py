"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[h]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[h + 1:]:
    name = r[ki].split("(")[0].replace("etune_b200::", "").replace("<unnamed>::", "")
    agg[name][0] += 1
    agg[name][1] += float(r[vi])
tot = sum(v for _, v in agg.values())
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:60]:60s} {c:6d} {v / 1e3:11.1f} us {100 * v / tot:5.1f} %")
print(f"total {tot / 1e3:.1f} us")

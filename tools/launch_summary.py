"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[start + 1:]:
    k = r[ki].split("(")[0]
    agg[k][0] += 1
    agg[k][1] += float(r[vi].replace(",", ""))
tot = sum(t for _, t in agg.values())
print(f"{'launches':>8} {'total_us':>10} {'avg_us':>9} {'share':>6}  kernel")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:8d} {t / 1e3:10.1f} {t / 1e3 / c:9.1f} {t / tot:6.1%}  {k}")

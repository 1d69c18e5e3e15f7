"""Per-query kernel breakdown of an ncu launch list taken with per-query NVTX
ranges (tools/suite_once.py): python tools/launch_by_query.py launches.csv [top]"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 6
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
ni = next(i for i, h in enumerate(hdr) if "Push/Pop_Range" in h)
per = defaultdict(lambda: defaultdict(lambda: [0, 0.0]))
for r in rows[start + 1:]:
    m = re.findall(r":(Q\d+):", r[ni])
    q = m[-1] if m else "-"
    k = r[ki].split("(")[0]
    per[q][k][0] += 1
    per[q][k][1] += float(r[vi].replace(",", "")) / 1e3
tot = {q: sum(t for _, t in d.values()) for q, d in per.items()}
print(f"{'query':>6} {'kern_ms':>8} {'launches':>8}  top kernels (us)")
for q in sorted(per, key=lambda q: -tot[q]):
    ks = sorted(per[q].items(), key=lambda x: -x[1][1])[:top]
    n = sum(c for c, _ in per[q].values())
    print(f"{q:>6} {tot[q] / 1e3:8.2f} {n:8d}  " +
          ", ".join(f"{k.replace('scx::', '').replace('_kernel', '')}x{c}={t:.0f}" for k, (c, t) in ks))
print(f"total {sum(tot.values()) / 1e3:.2f} ms")

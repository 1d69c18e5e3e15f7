"""GPU idle gaps inside each query (torch.profiler / CUPTI timestamps): where
the host keeps the device waiting.  python tools/gaps.py --sf 100 [--queries Q9,Q21]"""
import argparse
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2506_09226_b200 as P  # noqa: E402
from paper_2506_09226_b200.data import cached_generate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sf", type=float, default=100)
ap.add_argument("--queries", default=",".join(P.SUPPORTED_QUERIES))
ap.add_argument("--top", type=int, default=6)
a = ap.parse_args()
tables = P.load_tables(cached_generate(a.sf))
qs = a.queries.split(",")
for _ in range(2):
    for q in qs:
        P.reference_run(q, tables)
torch.cuda.synchronize()
tot_gap = 0.0
by_next = defaultdict(float)
for q in qs:
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        P.reference_run(q, tables)
        torch.cuda.synchronize()
    ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
                key=lambda e: e.time_range.start)
    gaps = []
    for x, y in zip(ev, ev[1:]):
        g = y.time_range.start - x.time_range.end
        if g > 0:
            gaps.append((g, x.name[:40], y.name[:40]))
            by_next[y.name[:40]] += g
    span = (ev[-1].time_range.end - ev[0].time_range.start) if ev else 0
    g_tot = sum(g for g, _, _ in gaps)
    tot_gap += g_tot
    top = sorted(gaps, reverse=True)[:a.top]
    print(f"{q}: span {span / 1e3:.2f} ms, idle {g_tot / 1e3:.2f} ms in {len(gaps)} gaps | " +
          "; ".join(f"{g:.0f}us before {n2}" for g, _, n2 in top))
print(f"TOTAL idle inside queries {tot_gap / 1e3:.2f} ms")
for n, g in sorted(by_next.items(), key=lambda kv: -kv[1])[:15]:
    print(f"  {g / 1e3:7.2f} ms idle before {n}")

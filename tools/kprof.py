"""Per-query GPU kernel time vs wall time (torch.profiler / CUPTI sees the
driver-API launches of libscx too).  python tools/kprof.py --sf 10"""
import argparse
import os
import sys
import time
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2506_09226_b200 as P  # noqa: E402
from paper_2506_09226_b200.data import cached_generate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sf", type=float, default=10)
ap.add_argument("--queries", default=",".join(P.SUPPORTED_QUERIES))
a = ap.parse_args()
tables = P.load_tables(cached_generate(a.sf))
qs = a.queries.split(",")
for _ in range(2):
    for q in qs:
        P.reference_run(q, tables)
torch.cuda.synchronize()
tot_w = tot_k = 0.0
for q in qs:
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        P.reference_run(q, tables)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    per = defaultdict(lambda: [0, 0.0])
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            k = e.name[:48]
            per[k][0] += 1
            per[k][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    ktime = sum(v[1] for v in per.values()) / 1e3
    tot_w += wall * 1e3
    tot_k += ktime
    top = sorted(per.items(), key=lambda kv: -kv[1][1])[:6]
    print(f"{q}: wall {wall * 1e3:7.2f} ms  kernels {ktime:7.2f} ms  launches "
          f"{sum(v[0] for v in per.values())}  | " +
          "; ".join(f"{k} x{c} {t / 1e3:.2f}" for k, (c, t) in top))
print(f"TOTAL wall {tot_w:.2f} ms, kernel {tot_k:.2f} ms")

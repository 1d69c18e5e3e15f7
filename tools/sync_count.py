"""Host syncs per query at SF100 (relops._to_host calls and other D2H reads),
and each query's wall vs device time on one stream.
python tools/sync_count.py [--sf 100]"""
import argparse
import os
import sys
import time
from collections import Counter

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_09226_b200 as P  # noqa: E402
import paper_2506_09226_b200.relops as R  # noqa: E402
from paper_2506_09226_b200.data import cached_generate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sf", type=float, default=100)
a = ap.parse_args()
tables = P.load_tables(cached_generate(a.sf))
calls = Counter()
orig = R._to_host


def counted(t):
    import traceback
    fr = traceback.extract_stack(limit=3)[-2]
    calls[f"{os.path.basename(fr.filename)}:{fr.lineno}"] += 1
    return orig(t)


R._to_host = counted
for q in P.SUPPORTED_QUERIES:
    P.reference_run(q, tables)
torch.cuda.synchronize()
tot_w = tot_d = 0
for q in P.SUPPORTED_QUERIES:
    calls.clear()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    P.reference_run(q, tables)
    e1.record()
    torch.cuda.synchronize()
    w = (time.perf_counter() - t0) * 1e3
    d = e0.elapsed_time(e1)
    tot_w += w
    tot_d += d
    print(f"{q:4s} wall {w:6.2f} ms  device {d:6.2f} ms  syncs {sum(calls.values()):3d}  "
          + ", ".join(f"{k}x{v}" for k, v in calls.most_common(6)), flush=True)
print(f"total wall {tot_w:.1f} ms device {tot_d:.1f} ms")

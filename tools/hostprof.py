"""Host-side (Python) cost of the 22-query suite: cProfile over one warm pass,
top functions by own time and by cumulative time.  python tools/hostprof.py --sf 100"""
import argparse
import cProfile
import io
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_09226_b200 as P  # noqa: E402
from paper_2506_09226_b200.data import cached_generate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sf", type=float, default=100)
ap.add_argument("--top", type=int, default=45)
a = ap.parse_args()
tables = P.load_tables(cached_generate(a.sf))
for _ in range(2):
    for q in P.SUPPORTED_QUERIES:
        P.reference_run(q, tables)
torch.cuda.synchronize()
t0 = time.perf_counter()
for q in P.SUPPORTED_QUERIES:
    P.reference_run(q, tables)
torch.cuda.synchronize()
print(f"suite wall (no profiler): {1e3 * (time.perf_counter() - t0):.1f} ms")
pr = cProfile.Profile()
pr.enable()
for q in P.SUPPORTED_QUERIES:
    P.reference_run(q, tables)
torch.cuda.synchronize()
pr.disable()
for key in ("tottime", "cumulative"):
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats(key).print_stats(a.top)
    print(f"===== by {key}\n" + "\n".join(s.getvalue().splitlines()[:a.top + 12]))

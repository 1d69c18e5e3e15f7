"""cProfile of the host path of one query (repeated), by cumulative time.
python tools/pyprof_q.py --q Q1 --reps 50"""
import argparse
import cProfile
import io
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_09226_b200 as P  # noqa: E402
from paper_2506_09226_b200.data import cached_generate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sf", type=float, default=1)
ap.add_argument("--q", default="Q1")
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--top", type=int, default=40)
a = ap.parse_args()
tables = P.load_tables(cached_generate(a.sf))
for _ in range(3):
    P.reference_run(a.q, tables)
torch.cuda.synchronize()
import time  # noqa: E402
t0 = time.perf_counter()
for _ in range(a.reps):
    P.reference_run(a.q, tables)
torch.cuda.synchronize()
print(f"{a.q}: {(time.perf_counter() - t0) / a.reps * 1e3:.3f} ms wall per run (no profiler)")
pr = cProfile.Profile()
pr.enable()
for _ in range(a.reps):
    P.reference_run(a.q, tables)
torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(a.top)
print("\n".join(s.getvalue().splitlines()[:a.top + 12]))

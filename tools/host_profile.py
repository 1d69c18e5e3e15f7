"""Host-side profile of each query after warm-up (where the non-kernel time goes).
Usage: python tools/host_profile.py --sf 10 --queries Q3,Q19"""
import argparse
import cProfile
import io
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2506_09226_b200 as P
from paper_2506_09226_b200.data import cached_generate

ap = argparse.ArgumentParser()
ap.add_argument("--sf", type=float, default=10)
ap.add_argument("--queries", default="Q1,Q3,Q6,Q12,Q14,Q19")
ap.add_argument("--top", type=int, default=25)
a = ap.parse_args()
tables = P.load_tables(cached_generate(a.sf))
qs = a.queries.split(",")
for _ in range(3):
    for q in qs:
        P.reference_run(q, tables)
torch.cuda.synchronize()
for q in qs:
    t0 = time.perf_counter()
    P.reference_run(q, tables)
    torch.cuda.synchronize()
    print(f"{q}: {1e3 * (time.perf_counter() - t0):.2f} ms wall")
for q in qs:
    pr = cProfile.Profile()
    pr.enable()
    P.reference_run(q, tables)
    torch.cuda.synchronize()
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(a.top)
    print(f"===== {q}\n" + "\n".join(s.getvalue().splitlines()[:a.top + 12]))

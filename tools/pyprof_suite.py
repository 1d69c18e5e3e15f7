"""cProfile of the host path of the 22-query suite at a small SF (kernels are
tiny there, so wall ~ host time): per-query wall and the top functions.
python tools/pyprof_suite.py --sf 1 --reps 10"""
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
ap.add_argument("--sf", type=float, default=1)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--top", type=int, default=45)
a = ap.parse_args()
tables = P.load_tables(cached_generate(a.sf))
for _ in range(2):
    for q in P.SUPPORTED_QUERIES:
        P.reference_run(q, tables)
torch.cuda.synchronize()
per = {}
for q in P.SUPPORTED_QUERIES:
    t0 = time.perf_counter()
    for _ in range(a.reps):
        P.reference_run(q, tables)
    torch.cuda.synchronize()
    per[q] = (time.perf_counter() - t0) / a.reps * 1e3
print("wall ms per query:", {q: round(v, 2) for q, v in per.items()}, "sum", round(sum(per.values()), 1))
pr = cProfile.Profile()
pr.enable()
for _ in range(a.reps):
    for q in P.SUPPORTED_QUERIES:
        P.reference_run(q, tables)
torch.cuda.synchronize()
pr.disable()
for key in ("tottime", "cumulative"):
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats(key).print_stats(a.top)
    print(f"==== by {key} (per {a.reps} suite passes)")
    print("\n".join(s.getvalue().splitlines()[:a.top + 12]))

"""Host time stamps inside one query (no profiler): wall time spent in the
main relops steps.  python tools/stamps.py --sf 100 --q Q1"""
import argparse
import functools
import os
import sys
import time
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_09226_b200 as P  # noqa: E402
from paper_2506_09226_b200 import relops as R, _lib as L, expr as X  # noqa: E402
from paper_2506_09226_b200.data import cached_generate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sf", type=float, default=100)
ap.add_argument("--q", default="Q1")
a = ap.parse_args()
acc = defaultdict(float)
cnt = defaultdict(int)


def wrap(mod, name, label=None):
    f = getattr(mod, name)

    @functools.wraps(f)
    def g(*x, **k):
        t = time.perf_counter()
        try:
            return f(*x, **k)
        finally:
            acc[label or name] += time.perf_counter() - t
            cnt[label or name] += 1
    setattr(mod, name, g)


for n in ("_plan_aggs", "_to_host", "finish_dense", "_materialize", "group_aggregate",
          "local_hash_join", "filter_table", "_pack_budgets", "sort_table"):
    wrap(R, n)
wrap(X, "integerise")
wrap(L, "call", "ctypes call")
orig_init = R._Builder.__init__


def binit(self, *x, **k):
    t = time.perf_counter()
    orig_init(self, *x, **k)
    acc["_Builder.__init__"] += time.perf_counter() - t
    cnt["_Builder.__init__"] += 1


R._Builder.__init__ = binit
tables = P.load_tables(cached_generate(a.sf))
for _ in range(3):
    P.reference_run(a.q, tables)
torch.cuda.synchronize()
acc.clear(); cnt.clear()
reps = 5
t0 = time.perf_counter()
for _ in range(reps):
    P.reference_run(a.q, tables)
    torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / reps
print(f"{a.q}: wall {wall * 1e3:.2f} ms per run")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:22s} {v / reps * 1e3:7.3f} ms  x{cnt[k] // reps}")

"""Time each query (wall, after warm-up) and show JIT cache stats + a cProfile
of the slowest.  python tools/qprof.py --sf 10 [--queries Q16,Q9]"""
import argparse
import cProfile
import ctypes as C
import io
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_09226_b200 as P  # noqa: E402
from paper_2506_09226_b200 import _lib  # noqa: E402
from paper_2506_09226_b200.data import cached_generate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sf", type=float, default=10)
ap.add_argument("--queries", default=",".join(P.SUPPORTED_QUERIES))
ap.add_argument("--top", type=int, default=30)
ap.add_argument("--profile", default="")
a = ap.parse_args()
lib = _lib.load()


def stats():
    v = [C.c_int64() for _ in range(3)]
    lib.scx_jit_stats(*[C.byref(x) for x in v])
    return tuple(x.value for x in v)


tables = P.load_tables(cached_generate(a.sf))
qs = a.queries.split(",")
for _ in range(2):
    for q in qs:
        P.reference_run(q, tables)
torch.cuda.synchronize()
print("jit stats after warm-up (compiled, disk, mem):", stats())
times = {}
for q in qs:
    s0 = stats()
    t0 = time.perf_counter()
    P.reference_run(q, tables)
    torch.cuda.synchronize()
    times[q] = time.perf_counter() - t0
    print(f"{q}: {1e3 * times[q]:.2f} ms wall  jit delta {tuple(b - c for b, c in zip(stats(), s0))}")
for q in (a.profile.split(",") if a.profile else [max(times, key=times.get)]):
    pr = cProfile.Profile()
    pr.enable()
    P.reference_run(q, tables)
    torch.cuda.synchronize()
    pr.disable()
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(a.top)
    print(f"===== {q}\n" + "\n".join(s.getvalue().splitlines()[:a.top + 12]))

"""Run one query repeatedly inside full-suite passes and report per-pass times
plus allocator retries (to chase timing outliers).  python tools/q_repeat.py --q Q21"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_09226_b200 as P  # noqa: E402
from paper_2506_09226_b200 import _lib  # noqa: E402
from paper_2506_09226_b200.data import cached_generate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sf", type=float, default=100)
ap.add_argument("--q", default="Q21")
ap.add_argument("--passes", type=int, default=8)
a = ap.parse_args()
lib = _lib.load()
tables = P.load_tables(cached_generate(a.sf))


def jit():
    import ctypes as C
    v = [C.c_int64() for _ in range(3)]
    lib.scx_jit_stats(*[C.byref(x) for x in v])
    return tuple(x.value for x in v)


for i in range(a.passes):
    for q in P.SUPPORTED_QUERIES:
        torch.cuda.synchronize()
        s0, r0 = jit(), torch.cuda.memory_stats().get("num_alloc_retries", 0)
        t0 = time.perf_counter()
        P.reference_run(q, tables)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        s1, r1 = jit(), torch.cuda.memory_stats().get("num_alloc_retries", 0)
        if q == a.q or dt > 30 or s1[0] != s0[0] or r1 != r0:
            print(f"pass {i} {q}: {dt:.2f} ms  jit compiled {s1[0] - s0[0]}  alloc retries {r1 - r0}"
                  f"  reserved {torch.cuda.memory_reserved() / 2**30:.1f} GiB")

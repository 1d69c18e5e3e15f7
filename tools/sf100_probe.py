"""Generate SF-x once (cached in /tmp/scx_data), report host time / RSS, and
time the 22 queries.  python tools/sf100_probe.py --sf 100"""
import argparse
import os
import resource
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--sf", type=float, default=100)
a = ap.parse_args()
t0 = time.time()
from paper_2506_09226_b200.data import cached_generate  # noqa: E402
ds = cached_generate(a.sf)
print(f"generate+cache SF{a.sf}: {time.time() - t0:.1f} s, host bytes {ds.nbytes / 1e9:.2f} GB, "
      f"max RSS {resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6:.1f} GB", flush=True)
import torch  # noqa: E402
import paper_2506_09226_b200 as P  # noqa: E402
t0 = time.time()
tables = P.load_tables(ds)
torch.cuda.synchronize()
print(f"load_tables: {time.time() - t0:.1f} s, device alloc {torch.cuda.memory_allocated() / 1e9:.1f} GB",
      flush=True)
for rep in range(3):
    tot = 0
    line = []
    for q in P.SUPPORTED_QUERIES:
        t0 = time.perf_counter()
        P.reference_run(q, tables)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        tot += dt
        line.append(f"{q}={dt * 1e3:.1f}")
    print(f"pass {rep}: total {tot * 1e3:.1f} ms | " + " ".join(line), flush=True)
print(f"peak device memory {torch.cuda.max_memory_allocated() / 1e9:.1f} GB")

"""Warm up, then run the 22-query suite once (for ncu launch lists):
ncu --metrics gpu__time_duration.sum ... python tools/suite_once.py --sf 100"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_09226_b200 as P  # noqa: E402
from paper_2506_09226_b200.data import cached_generate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sf", type=float, default=100)
ap.add_argument("--warm", type=int, default=1)
a = ap.parse_args()
tables = P.load_tables(cached_generate(a.sf))
for _ in range(a.warm):
    for q in P.SUPPORTED_QUERIES:
        P.reference_run(q, tables)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("timed_suite")
for q in P.SUPPORTED_QUERIES:
    torch.cuda.nvtx.range_push(q)
    P.reference_run(q, tables)
    torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("suite done")

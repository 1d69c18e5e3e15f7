"""Profiling driver: load SF data once, run chosen queries a few times.
Usage: python tools/prof_queries.py --sf 10 --queries Q1,Q6 --reps 3"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2506_09226_b200 as P
from paper_2506_09226_b200.data import cached_generate

ap = argparse.ArgumentParser()
ap.add_argument("--sf", type=float, default=10)
ap.add_argument("--queries", default="Q1,Q6")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
tables = P.load_tables(cached_generate(a.sf))
for _ in range(a.reps):
    for q in a.queries.split(","):
        P.reference_run(q, tables)
torch.cuda.synchronize()
print("done")

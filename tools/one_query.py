"""Run one query once (after `--warm` warm-up passes) -- for ncu captures.
python tools/one_query.py --sf 10 --query Q17 --warm 1"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_09226_b200 as P  # noqa: E402
from paper_2506_09226_b200.data import cached_generate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sf", type=float, default=10)
ap.add_argument("--query", default="Q17")
ap.add_argument("--warm", type=int, default=1)
a = ap.parse_args()
tables = P.load_tables(cached_generate(a.sf))
for q in a.query.split(","):
    for _ in range(a.warm + 1):
        P.reference_run(q, tables)
torch.cuda.synchronize()

"""Per-query device time of the probe-heavy queries at SF100 under several
codegen configurations (env knobs of csrc/jit.cu), one process, the launch-
plan memo cleared between configurations (scx_jit_clear_plans).

    python tools/chunk_sweep.py --configs "SCX_CHUNK=0;SCX_CHUNK=1;SCX_CHUNK=1,SCX_CHUNK_U0=2"
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_09226_b200 as P  # noqa: E402
from paper_2506_09226_b200 import _lib  # noqa: E402
from paper_2506_09226_b200.data import cached_generate  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sf", type=float, default=100)
ap.add_argument("--queries", default="Q3,Q5,Q7,Q8,Q9,Q10,Q12,Q17,Q19,Q20,Q21,Q2,Q16,Q11")
ap.add_argument("--configs", required=True)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
lib = _lib.load()
tables = P.load_tables(cached_generate(a.sf))
qs = a.queries.split(",")
knobs = set()
cfgs = a.configs.split(";")
best = {c: {} for c in cfgs}


def apply(cfg):
    global knobs
    env = dict(kv.split("=") for kv in cfg.split(",") if kv)
    for k in knobs | set(env):
        os.environ.pop(k, None)
    os.environ.update(env)
    knobs |= set(env)
    lib.scx_jit_clear_plans()


for cfg in cfgs:                       # compile + warm every configuration once
    apply(cfg)
    for q in qs:
        P.reference_run(q, tables)
for r in range(a.reps):                # interleaved rounds: min over rounds per query
    for cfg in (cfgs if r % 2 == 0 else cfgs[::-1]):
        apply(cfg)
        for q in qs:
            P.reference_run(q, tables)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            P.reference_run(q, tables)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            best[cfg][q] = min(best[cfg].get(q, 1e9), round(t, 3))
for cfg in cfgs:
    print(cfg, "sum", round(sum(best[cfg].values()), 2), best[cfg], flush=True)
print(json.dumps(best))

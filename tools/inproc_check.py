"""All 22 queries at N in-process virtual ranks vs the oracle; lists every
mismatch instead of stopping at the first.  python tools/inproc_check.py --n 2,3,8 --sf 0.1"""
import argparse
import os
import sys
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2506_09226_b200 as P  # noqa: E402
from oracle import ref as O  # noqa: E402
from test_gpu_tpch22 import assert_same  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", default="2,3,8")
ap.add_argument("--sf", type=float, default=0.1)
ap.add_argument("--skew", type=float, default=0.0)
ap.add_argument("--q", default="")
a = ap.parse_args()
ds = P.generate(a.sf, a.skew, 0)
ref = ds.to_reference()
qs = a.q.split(",") if a.q else [f"Q{i}" for i in range(1, 23)]
exp = {q: O.reference_run(q, ref) for q in qs}
bad = []
for n in [int(x) for x in a.n.split(",")]:
    per = P.partition_tables(ds, n)
    cl = P.create_cluster(P.Topology(k=n, v=1), P.MODE_IN_PROCESS)
    for q in qs:
        try:
            res, rep = P.run_query(q, "default", cl, per)
            assert_same(res, exp[q], f"{q}@N{n}")
            print(f"ok   {q}@N{n} exchanges={rep.exchange_counts}", flush=True)
        except Exception as e:  # noqa: BLE001
            bad.append((q, n))
            print(f"FAIL {q}@N{n}: {type(e).__name__}: {str(e)[:300]}", flush=True)
            if os.environ.get("TB"):
                traceback.print_exc()
print("failures:", bad)

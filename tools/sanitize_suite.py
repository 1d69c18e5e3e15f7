"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): the
22 TPC-H queries at SF0.01 through reference_run on one rank, the same at
N=3 virtual ranks (partition kernel + fused scatter shuffles + broadcasts),
and a large stable partition.

    compute-sanitizer --tool memcheck python tools/sanitize_suite.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_09226_b200 as P  # noqa: E402

sf = float(os.environ.get("SAN_SF", "0.01"))
ds = P.generate(sf, 0.0, 0)
tables = P.load_tables(ds)
for q in P.SUPPORTED_QUERIES:
    P.reference_run(q, tables)
torch.cuda.synchronize()
print("N=1 suite ok", flush=True)
if os.environ.get("SAN_N3", "1") == "1":
    per = P.partition_tables(ds, 3)
    cl = P.create_cluster(P.Topology(k=3, v=1, bg_gbps=900, bn_gbps=900), P.MODE_IN_PROCESS)
    for q in P.SUPPORTED_QUERIES:
        P.run_query(q, "default", cl, per)
    torch.cuda.synchronize()
    print("N=3 suite ok", flush=True)
rng = np.random.default_rng(0)
t = P.ColumnTable({"k": P.Column("int64", rng.integers(0, 1 << 40, 300_001)),
                   "v": P.Column("int64", rng.integers(0, 1 << 20, 300_001))})
parts = P.hash_partition(t, ["k"], 5)
torch.cuda.synchronize()
print("partition ok", sum(p.row_count for p in parts), flush=True)
print("kernels launched:", P._lib.load().scx_launch_count())

"""Time the partition kernel on 1 GiB of 16-byte rows (config 5 shape) at N parts.
python tools/part_bench.py [--gib 1] [--parts 1,2,8]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_09226_b200 import exchange as X  # noqa: E402
from paper_2506_09226_b200.table import Column, ColumnTable  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--gib", type=float, default=1.0)
ap.add_argument("--parts", default="1,2,4,8")
a = ap.parse_args()
rows = int(a.gib * (1 << 30)) // 16
key = torch.from_numpy(np.random.default_rng(0).integers(0, 2 ** 62, size=rows, dtype=np.int64)).cuda()
pay = torch.arange(rows, dtype=torch.int64, device="cuda")
t = ColumnTable({"key": Column("int64", key, 0, None, 0, 2 ** 62),
                 "payload": Column("int64", pay, 0, None, 0, rows)})
for n in [int(x) for x in a.parts.split(",")]:
    ms = []
    for i in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        outs, cnt = X.partition_device(t, ["key"], n)
        e1.record()
        torch.cuda.synchronize()
        if i:
            ms.append(e0.elapsed_time(e1))
        del outs
    m = sum(ms) / len(ms)
    alg = rows * 16 * 2 + rows * 8
    print(f"parts={n} {m:.3f} ms  {alg / m / 1e6:.0f} GB/s (alg {alg / 1e9:.2f} GB)")

"""Trace Q15 / Q16 intermediates per virtual rank at N=2."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2506_09226_b200 as P
from paper_2506_09226_b200 import queries as Qm
from paper_2506_09226_b200.engine import DeviceContext
from paper_2506_09226_b200.table import date_to_days
from oracle import ref as O

ds = P.generate(0.1, 0.0, 0)
per = P.partition_tables(ds, 2)
cl = P.create_cluster(P.Topology(k=2, v=1), P.MODE_IN_PROCESS)


def w(ep):
    q = DeviceContext(ep, per[ep.rank], "default", "default_keys", timed=False)
    li = q.table("lineitem")
    sd = li["l_shipdate"]
    lf = q.filter(li, (sd >= date_to_days("1996-01-01")) & (sd < date_to_days("1996-04-01")))
    lf0 = lf.select(["l_suppkey"]).materialize()
    lf = q.shuffle(lf.select(["l_suppkey", "l_extendedprice", "l_discount"]), ["l_suppkey"])
    lf = q.add_column(lf, "rev", lf["l_extendedprice"] * (1.0 - lf["l_discount"]))
    rev = q.group(lf, ["l_suppkey"], {"total_revenue": ("sum", "rev")}, sort=False).materialize()
    mx = q.global_group_all(rev, [], {"m": ("max", "total_revenue")}).column("m")
    tr = rev.column("total_revenue")
    print(f"rank {ep.rank}: lf rows {lf0.row_count} -> shuffled {lf.select(["l_suppkey"]).materialize().row_count}; "
          f"rev rows {rev.row_count} scale {tr.scale} dtype {tr.np_dtype} lo/hi {tr.lo}/{tr.hi} "
          f"max-local {tr.host().max() if rev.row_count else None}; mx raw {mx.host()} scale "
          f"{mx.scale} exact {Qm.exact(mx)}", flush=True)
    best = q.filter(rev, rev["total_revenue"] == Qm.exact(mx)).materialize()
    print(f"rank {ep.rank}: best rows {best.row_count}", flush=True)
    s = q.table("supplier").select(["s_suppkey"])
    out = q.join(best, s, on=[("l_suppkey", "s_suppkey")], how="semi").materialize()
    print(f"rank {ep.rank}: out rows {out.row_count}", flush=True)
    return None


P.run_workers(cl, w)
ref = ds.to_reference()
print("oracle Q15:", O.reference_run("Q15", ref))

# Q16 / Q17 at N=2 / N=8: first differing rows
for qid, n in (("Q16", 2), ("Q17", 8)):
    per_n = P.partition_tables(ds, n)
    cln = P.create_cluster(P.Topology(k=n, v=1), P.MODE_IN_PROCESS)
    try:
        res, _ = P.run_query(qid, "default", cln, per_n)
    except Exception as e:  # noqa: BLE001
        import traceback
        traceback.print_exc()
        continue
    got = res.materialize().to_reference()
    exp = O.reference_run(qid, ref)
    for name, (k, v, d) in exp.items():
        gv = got[name][1]
        if len(gv) != len(v) or not np.array_equal(np.asarray(gv).astype(np.float64), np.asarray(v).astype(np.float64)):
            idx = [i for i in range(min(len(gv), len(v))) if gv[i] != v[i]][:5]
            print(qid, name, "len", len(gv), len(v), "first diffs", idx,
                  [(gv[i], v[i]) for i in idx], "dict eq", got[name][2] == d)

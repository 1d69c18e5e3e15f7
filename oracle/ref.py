"""CPU oracle: numpy restatement of the reference's relational path.

TEST INFRASTRUCTURE (see oracle/__init__.py).  A table here is a plain
``dict[name -> (kind, values, dictionary)]`` in the reference's storage
dtypes (int64 / float64 / int32 dates / int32 dict codes, table.py:25-30).
Every routine reproduces the reference's numpy operations in the same order
so float64 results are bit-identical to ``shufflecast.reference_run`` (the
pinning test checks this against golden vectors from the real reference).
"""

from __future__ import annotations

from datetime import date

import numpy as np

EPOCH = date(1970, 1, 1)
FIB = np.uint64(0x9E3779B97F4A7C15)


def days(iso: str) -> int:
    y, m, d = (int(x) for x in iso.split("-"))
    return (date(y, m, d) - EPOCH).days


# ---- table helpers (table.py:171-214) --------------------------------------

def nrows(t) -> int:
    return len(next(iter(t.values()))[1]) if t else 0


def take(t, idx):
    return {n: (k, v[idx], d) for n, (k, v, d) in t.items()}


def select(t, names):
    return {n: t[n] for n in names}


def vals(t, name):
    return t[name][1]


def isin(t, name, wanted):
    """table.py:185-192"""
    k, v, d = t[name]
    codes = [i for i, s in enumerate(d) if s in set(wanted)]
    return np.isin(v, np.asarray(codes, dtype=np.int32))


def codes_where(t, name, pred):
    """queries.py:23-29"""
    k, v, d = t[name]
    return np.isin(v, np.asarray([i for i, s in enumerate(d) if pred(s)], dtype=np.int32))


def sort_by(t, names, descending=()):
    """Stable lexsort, dict by string rank, desc by negation (table.py:198-214)."""
    keys = []
    for name in reversed(names):
        k, v, d = t[name]
        if k == "dict":
            rank = np.empty(len(d), dtype=np.int64)
            rank[np.argsort(np.asarray(d, dtype=object))] = np.arange(len(d))
            key = rank[v]
        else:
            key = v
        keys.append(-key if name in descending else key)
    idx = np.lexsort(keys) if keys else np.arange(nrows(t))
    return take(t, idx)


def head(t, n):
    return take(t, np.arange(min(n, nrows(t))))


# ---- relops (relops.py:20-160) ---------------------------------------------

def filter_(t, mask):
    return take(t, np.flatnonzero(np.asarray(mask, dtype=bool)))


def _codes(left, right, on):
    """Dense join codes consistent across both sides (relops.py:32-56)."""
    lc = rc = None
    for ln, rn in on:
        lv = left[ln][1].astype(np.int64)
        rv = right[rn][1].astype(np.int64)
        uniq, inv = np.unique(np.concatenate([lv, rv]), return_inverse=True)
        a, b = inv[:len(lv)], inv[len(lv):]
        if lc is None:
            lc, rc = a, b
        else:
            lc, rc = lc * len(uniq) + a, rc * len(uniq) + b
    return lc.astype(np.int64), rc.astype(np.int64)


def join(left, right, on, how="inner"):
    """relops.py:59-94: semi/anti via isin, inner via stable argsort+searchsorted."""
    lc, rc = _codes(left, right, on)
    if how in ("semi", "anti"):
        m = np.isin(lc, rc)
        return filter_(left, m if how == "semi" else ~m)
    order = np.argsort(rc, kind="stable")
    rs = rc[order]
    lo = np.searchsorted(rs, lc, side="left")
    hi = np.searchsorted(rs, lc, side="right")
    cnt = hi - lo
    tot = int(cnt.sum())
    lidx = np.repeat(np.arange(len(lc)), cnt)
    start = np.repeat(lo, cnt)
    within = np.arange(tot) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    ridx = order[start + within]
    out = take(left, lidx)
    out.update(take(right, ridx))
    return out


def group(t, keys, aggs):
    """relops.py:97-160 (np.unique codes, bincount, add.at, sort by keys)."""
    n = nrows(t)
    if keys:
        codes = None
        for k in keys:
            u, c = np.unique(t[k][1].astype(np.int64), return_inverse=True)
            codes = c if codes is None else codes * len(u) + c
        uc, first, inv = np.unique(codes, return_index=True, return_inverse=True)
        ng = len(uc)
        out = {k: (t[k][0], t[k][1][first], t[k][2]) for k in keys}
    else:
        ng = 1
        inv = np.zeros(n, dtype=np.int64)
        out = {}
    counts = np.bincount(inv, minlength=ng).astype(np.int64)
    for name, (op, col) in aggs.items():
        if op == "count":
            out[name] = ("int64", counts, None)
            continue
        kind, v, _ = t[col]
        if op == "sum" and kind != "float64":
            acc = np.zeros(ng, dtype=np.int64)
            np.add.at(acc, inv, v.astype(np.int64))
            out[name] = ("int64", acc, None)
        elif op in ("sum", "avg"):
            acc = np.zeros(ng, dtype=np.float64)
            np.add.at(acc, inv, v.astype(np.float64))
            if op == "avg":
                acc = acc / np.maximum(counts, 1)
            out[name] = ("float64", acc, None)
        else:
            if np.issubdtype(v.dtype, np.floating):
                init = np.inf if op == "min" else -np.inf
            else:
                info = np.iinfo(v.dtype)
                init = info.max if op == "min" else info.min
            acc = np.full(ng, init, dtype=v.dtype)
            (np.minimum if op == "min" else np.maximum).at(acc, inv, v)
            out[name] = ("float64" if np.issubdtype(v.dtype, np.floating) else kind, acc, None)
    return sort_by(out, keys) if keys else out


# ---- exchange hash (exchange.py:35-70) --------------------------------------

def hash_keys(t, keys):
    acc = np.zeros(nrows(t), dtype=np.uint64)
    with np.errstate(over="ignore"):
        for k in keys:
            acc = (acc ^ (t[k][1].astype(np.uint64) * FIB)) * FIB
    return acc


def hash_partition(t, keys, n):
    b = hash_keys(t, keys) % np.uint64(n)
    order = np.argsort(b, kind="stable")
    cuts = np.searchsorted(b[order], np.arange(n + 1, dtype=b.dtype))
    return [take(t, order[cuts[i]:cuts[i + 1]]) for i in range(n)]


# ---- query drivers, single context (queries.py:32-238, engine.py:221-258) ----

def q1(T):
    li = T["lineitem"]
    f = filter_(li, vals(li, "l_shipdate") <= days("1998-09-02"))
    rf, ls = f["l_returnflag"], f["l_linestatus"]
    ncell = len(rf[2]) * len(ls[2])
    cell = rf[1].astype(np.int64) * len(ls[2]) + ls[1]
    ext, dsc, tax = vals(f, "l_extendedprice"), vals(f, "l_discount"), vals(f, "l_tax")
    dp = ext * (1.0 - dsc)
    ch = dp * (1.0 + tax)
    ms = [vals(f, "l_quantity").astype(np.float64), ext, dp, ch, dsc, np.ones(nrows(f))]
    grid = np.zeros((len(ms), ncell))
    for i, m in enumerate(ms):
        np.add.at(grid[i], cell, m)
    tot = grid        # all_reduce_sum is the identity in one context
    cnt = tot[5]
    live = np.flatnonzero(cnt > 0)
    out = {
        "l_returnflag": ("dict", (live // len(ls[2])).astype(np.int32), rf[2]),
        "l_linestatus": ("dict", (live % len(ls[2])).astype(np.int32), ls[2]),
        "sum_qty": ("float64", tot[0][live], None),
        "sum_base_price": ("float64", tot[1][live], None),
        "sum_disc_price": ("float64", tot[2][live], None),
        "sum_charge": ("float64", tot[3][live], None),
        "avg_qty": ("float64", tot[0][live] / cnt[live], None),
        "avg_price": ("float64", tot[1][live] / cnt[live], None),
        "avg_disc": ("float64", tot[4][live] / cnt[live], None),
        "count_order": ("int64", cnt[live].astype(np.int64), None),
    }
    return sort_by(out, ["l_returnflag", "l_linestatus"])


def q3(T):
    cust = T["customer"]
    ck = select(filter_(cust, isin(cust, "c_mktsegment", ["BUILDING"])), ["c_custkey"])
    o = T["orders"]
    of = filter_(o, vals(o, "o_orderdate") < days("1995-03-15"))
    oj = join(of, ck, [("o_custkey", "c_custkey")], "semi")
    li = T["lineitem"]
    lf = filter_(li, vals(li, "l_shipdate") > days("1995-03-15"))
    j = join(select(lf, ["l_orderkey", "l_extendedprice", "l_discount"]),
             select(oj, ["o_orderkey", "o_orderdate", "o_shippriority"]),
             [("l_orderkey", "o_orderkey")])
    j["revenue"] = ("float64", vals(j, "l_extendedprice") * (1.0 - vals(j, "l_discount")), None)
    g = group(j, ["l_orderkey", "o_orderdate", "o_shippriority"], {"revenue": ("sum", "revenue")})
    top = head(sort_by(g, ["revenue", "o_orderdate"], {"revenue"}), 10)
    return select(top, ["l_orderkey", "revenue", "o_orderdate", "o_shippriority"])


def q6(T):
    li = T["lineitem"]
    sd, dsc = vals(li, "l_shipdate"), vals(li, "l_discount")
    m = ((sd >= days("1994-01-01")) & (sd < days("1995-01-01")) & (dsc >= 0.05)
         & (dsc <= 0.07) & (vals(li, "l_quantity") < 24))
    f = filter_(li, m)
    rev = float((vals(f, "l_extendedprice") * vals(f, "l_discount")).sum())
    return {"revenue": ("float64", np.asarray([rev]), None)}


def q12(T):
    li = T["lineitem"]
    sd, cd, rd = vals(li, "l_shipdate"), vals(li, "l_commitdate"), vals(li, "l_receiptdate")
    m = (isin(li, "l_shipmode", ["MAIL", "SHIP"]) & (cd < rd) & (sd < cd)
         & (rd >= days("1994-01-01")) & (rd < days("1995-01-01")))
    lf = select(filter_(li, m), ["l_orderkey", "l_shipmode"])
    o = select(T["orders"], ["o_orderkey", "o_orderpriority"])
    j = join(lf, o, [("l_orderkey", "o_orderkey")])
    high = codes_where(j, "o_orderpriority", lambda s: s in ("1-URGENT", "2-HIGH"))
    j["high"] = ("int64", high.astype(np.int64), None)
    j["low"] = ("int64", (~high).astype(np.int64), None)
    g = group(j, ["l_shipmode"], {"high_line_count": ("sum", "high"),
                                  "low_line_count": ("sum", "low")})
    return group(g, ["l_shipmode"], {"high_line_count": ("sum", "high_line_count"),
                                     "low_line_count": ("sum", "low_line_count")})


def q14(T):
    li = T["lineitem"]
    sd = vals(li, "l_shipdate")
    lf = select(filter_(li, (sd >= days("1995-09-01")) & (sd < days("1995-10-01"))),
                ["l_partkey", "l_extendedprice", "l_discount"])
    j = join(lf, select(T["part"], ["p_partkey", "p_type"]), [("l_partkey", "p_partkey")])
    dp = vals(j, "l_extendedprice") * (1.0 - vals(j, "l_discount"))
    promo = np.where(codes_where(j, "p_type", lambda s: s.startswith("PROMO")), dp, 0.0)
    tot = float(np.asarray([dp.sum()]).sum())
    ps = float(np.asarray([promo.sum()]).sum())
    v = 100.0 * ps / tot if tot else 0.0
    return {"promo_revenue": ("float64", np.asarray([v]), None)}


Q19_BRANCHES = (
    ("Brand#12", ("SM CASE", "SM BOX", "SM PACK", "SM PKG"), 1, 11, 1, 5),
    ("Brand#23", ("MED BAG", "MED BOX", "MED PKG", "MED PACK"), 10, 20, 1, 10),
    ("Brand#34", ("LG CASE", "LG BOX", "LG PACK", "LG PKG"), 20, 30, 1, 15),
)


def q19(T):
    p = T["part"]
    brands = [b for b, *_ in Q19_BRANCHES]
    pf = filter_(p, isin(p, "p_brand", brands) & (vals(p, "p_size") >= 1)
                 & (vals(p, "p_size") <= 15))
    pb = select(pf, ["p_partkey", "p_brand", "p_size", "p_container"])
    li = T["lineitem"]
    lf = select(filter_(li, isin(li, "l_shipmode", ["AIR", "AIR REG"])
                        & isin(li, "l_shipinstruct", ["DELIVER IN PERSON"])),
                ["l_partkey", "l_quantity", "l_extendedprice", "l_discount"])
    j = join(lf, pb, [("l_partkey", "p_partkey")])
    qty, size = vals(j, "l_quantity"), vals(j, "p_size")
    keep = np.zeros(nrows(j), dtype=bool)
    for brand, cont, qlo, qhi, slo, shi in Q19_BRANCHES:
        keep |= (isin(j, "p_brand", [brand]) & isin(j, "p_container", list(cont))
                 & (qty >= qlo) & (qty <= qhi) & (size >= slo) & (size <= shi))
    mt = filter_(j, keep)
    rev = float((vals(mt, "l_extendedprice") * (1.0 - vals(mt, "l_discount"))).sum())
    return {"revenue": ("float64", np.asarray([float(np.asarray([rev]).sum())]), None)}


QUERIES = {"Q1": q1, "Q3": q3, "Q6": q6, "Q12": q12, "Q14": q14, "Q19": q19}


def all_queries() -> dict:
    """The reference's six drivers + the builder-written 16 (oracle/tpch_ext.py)."""
    from . import tpch_ext
    return {**QUERIES, **tpch_ext.QUERIES}


def reference_run(qid: str, tables):
    """Single-context ground truth (engine.py:463-469)."""
    return all_queries()[qid](tables)


def to_jsonable(t) -> dict:
    """Exact serialisation: floats as hex, ints as ints, dict as codes+dict."""
    out = {}
    for n, (k, v, d) in t.items():
        if k == "float64":
            out[n] = {"kind": k, "hex": [float(x).hex() for x in v]}
        else:
            out[n] = {"kind": k, "values": [int(x) for x in v],
                      **({"dictionary": list(d)} if d is not None else {})}
    return out


def from_jsonable(j: dict):
    t = {}
    for n, c in j.items():
        if c["kind"] == "float64":
            t[n] = ("float64", np.asarray([float.fromhex(x) for x in c["hex"]]), None)
        else:
            dt = {"int64": np.int64, "date32": np.int32, "dict": np.int32}[c["kind"]]
            t[n] = (c["kind"], np.asarray(c["values"], dtype=dt),
                    tuple(c["dictionary"]) if "dictionary" in c else None)
    return t

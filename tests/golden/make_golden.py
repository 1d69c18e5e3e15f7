"""Generate golden fixtures by running the REAL reference (shufflecast).

Run in the dev container (the only place /root/reference exists):

    python tests/golden/make_golden.py

Writes small JSON fixtures next to this file.  They pin (a) our generator to
the reference's data, (b) the CPU oracle (oracle/ref.py) to the reference's
outputs, and (c) the GPU path through the oracle.  The GPU box never reads
/root/reference -- only these committed files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ser_table(t) -> dict:
    out = {}
    for name in t.column_names:
        c = t.column(name)
        if c.kind == "float64":
            out[name] = {"kind": c.kind, "hex": [float(x).hex() for x in c.values]}
        else:
            out[name] = {"kind": c.kind, "values": [int(x) for x in c.values],
                         **({"dictionary": list(c.dictionary)} if c.dictionary else {})}
    return out


def _col_digest(v: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()


def main() -> None:
    sys.path.insert(0, REF)
    import shufflecast as s
    from shufflecast.table import Column, ColumnTable

    # ---- 1. generator digests + 2. reference_run results --------------------
    gens = {}
    results = {}
    for sf, skew in [(0.01, 0.0), (0.01, 1.5), (0.1, 0.0), (1.0, 0.0)]:
        ds = s.generate(sf, skew=skew, seed=0)
        key = f"sf{sf}_skew{skew}"
        gens[key] = {name: {"rows": t.row_count,
                            "columns": {c: {"kind": t.column(c).kind,
                                            "dtype": str(t.column(c).values.dtype),
                                            "sha256": _col_digest(t.column(c).values)}
                                        for c in t.column_names}}
                     for name, t in ds.tables.items()}
        results[key] = {q: _ser_table(s.reference_run(q, ds)) for q in s.SUPPORTED_QUERIES}
        print("done", key, flush=True)
    with open(os.path.join(HERE, "generator_digests.json"), "w") as fh:
        json.dump(gens, fh, indent=1)
    with open(os.path.join(HERE, "query_results.json"), "w") as fh:
        json.dump(results, fh, indent=1)

    # ---- 3. hash KATs + partition assignments --------------------------------
    keys = [0, 1, 2, 3, 1 << 40, -1, 123456789, -987654321]
    t1 = ColumnTable({"k": Column("int64", np.asarray(keys, dtype=np.int64))})
    rng = np.random.default_rng(7)
    a = rng.integers(-(1 << 40), 1 << 40, size=2000)
    b = rng.integers(0, 50, size=2000).astype(np.int32)
    t2 = ColumnTable({"a": Column("int64", a), "b": Column("date32", b)})
    parts = {}
    for n in (1, 2, 3, 4, 5, 8, 16):
        p1 = s.hash_partition(t2, ["a"], n)
        p2 = s.hash_partition(t2, ["a", "b"], n)
        parts[str(n)] = {"single": [[int(x) for x in p.column("a").values] for p in p1],
                         "multi_sizes": [p.row_count for p in p2],
                         "multi_first": [[int(x) for x in p.column("a").values[:5]] for p in p2]}
    kat = {
        "keys": keys,
        "hash_single": [str(int(x)) for x in s.hash_keys(t1, ["k"])],
        "pair_keys": [[1, 2], [1, 3]],
        "hash_pairs": [str(int(x)) for x in s.hash_keys(
            ColumnTable({"x": Column("int64", np.asarray([1, 1])),
                         "y": Column("int64", np.asarray([2, 3]))}), ["x", "y"])],
        "partition_input_seed": 7,
        "partitions": parts,
    }
    with open(os.path.join(HERE, "hash_kats.json"), "w") as fh:
        json.dump(kat, fh, indent=1)

    # ---- 4. relops semantics on small random tables --------------------------
    rng = np.random.default_rng(11)
    n_l, n_r = 400, 120
    dict_ = ("SHIP", "AIR", "MAIL", "RAIL", "FOB")
    left = ColumnTable({
        "lk": Column("int64", rng.integers(0, 150, size=n_l)),
        "lv": Column("float64", np.round(rng.uniform(0, 1000, size=n_l), 2)),
        "ld": Column("date32", rng.integers(8000, 8100, size=n_l).astype(np.int32)),
        "lc": Column("dict", rng.integers(0, len(dict_), size=n_l).astype(np.int32), dict_),
        "li": Column("int64", rng.integers(-50, 50, size=n_l)),
    })
    right_u = ColumnTable({
        "rk": Column("int64", rng.permutation(200)[:n_r].astype(np.int64)),
        "rv": Column("int64", rng.integers(0, 9, size=n_r)),
    })
    right_d = ColumnTable({
        "rk": Column("int64", rng.integers(0, 150, size=n_r)),
        "rv": Column("int64", rng.integers(0, 9, size=n_r)),
    })
    rel = {"left": _ser_table(left), "right_unique": _ser_table(right_u),
           "right_dup": _ser_table(right_d)}
    for how in ("inner", "semi", "anti"):
        rel[f"join_unique_{how}"] = _ser_table(s.local_hash_join(left, right_u, [("lk", "rk")], how))
        rel[f"join_dup_{how}"] = _ser_table(s.local_hash_join(left, right_d, [("lk", "rk")], how))
    aggs = {"n": ("count", None), "s_f": ("sum", "lv"), "s_i": ("sum", "li"), "a_f": ("avg", "lv"),
            "mn_i": ("min", "li"), "mx_i": ("max", "li"), "mn_f": ("min", "lv"),
            "mx_d": ("max", "ld"), "s_d": ("sum", "ld")}
    rel["group_lc"] = _ser_table(s.group_aggregate(left, ["lc"], aggs))
    rel["group_lc_ld"] = _ser_table(s.group_aggregate(left, ["lc", "ld"], aggs))
    rel["group_lk"] = _ser_table(s.group_aggregate(left, ["lk"], aggs))
    rel["group_none"] = _ser_table(s.group_aggregate(left, [], aggs))
    rel["sort_lc_desc_lv"] = _ser_table(left.sort_by(["lc", "lv"], {"lv"}))
    rel["sort_li_ld"] = _ser_table(left.sort_by(["li", "ld"], {"li"}))
    with open(os.path.join(HERE, "relops.json"), "w") as fh:
        json.dump(rel, fh, indent=1)

    # ---- 5. exchange semantics (in-process cluster) ---------------------------
    topo = s.Topology(k=3, v=1, bg_gbps=900, bn_gbps=900)
    cl = s.create_cluster(topo, s.MODE_IN_PROCESS)
    base = [ColumnTable({"k": Column("int64", np.arange(r * 10, r * 10 + 7 + r)),
                         "v": Column("date32", np.arange(7 + r, dtype=np.int32) + 100 * r)})
            for r in range(3)]

    def w(ep):
        sh = s.shuffle_table(ep, base[ep.rank], ["k"])
        bc = s.broadcast_table(ep, base[ep.rank])
        return _ser_table(sh), _ser_table(bc)

    outs = s.run_workers(cl, w)
    ex = {"inputs": [_ser_table(t) for t in base],
          "shuffle": [o[0] for o in outs], "broadcast": [o[1] for o in outs]}
    with open(os.path.join(HERE, "exchange.json"), "w") as fh:
        json.dump(ex, fh, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()

"""GPU parity: the CUDA path vs the oracle / golden reference outputs.

Bar: keys, counts, integer/date/dict columns and row order
bit-exact; float64 columns within rtol 1e-9 (the tolerance north_star
states).  Fixed-point aggregates are additionally checked bit-exact against
an exact integer restatement.
"""

import numpy as np
import pytest

from conftest import load_golden, parse_key
from oracle import ref as O

pytestmark = pytest.mark.gpu

RTOL = 1e-9


def _dev():
    import paper_2506_09226_b200 as P
    return P


def assert_table_matches(got, expected: dict, ctx=""):
    """got: device ColumnTable; expected: oracle-jsonable dict."""
    got = got.materialize()
    assert got.column_names == list(expected), (ctx, got.column_names, list(expected))
    for name, exp in expected.items():
        c = got.column(name)
        assert c.kind == exp["kind"], (ctx, name, c.kind, exp["kind"])
        v = c.values
        if exp["kind"] == "float64":
            e = np.asarray([float.fromhex(x) for x in exp["hex"]])
            assert len(v) == len(e), (ctx, name, len(v), len(e))
            np.testing.assert_allclose(v, e, rtol=RTOL, atol=0, err_msg=f"{ctx}:{name}")
        else:
            e = np.asarray(exp["values"])
            assert len(v) == len(e), (ctx, name, len(v), len(e))
            assert np.array_equal(v.astype(np.int64), e.astype(np.int64)), (ctx, name, v[:10], e[:10])
            if "dictionary" in exp:
                assert list(c.dictionary) == exp["dictionary"]


RES = load_golden("query_results.json")
_DS = {}


def device_tables(key):
    if key not in _DS:
        from paper_2506_09226_b200.data import generate
        from paper_2506_09226_b200.engine import load_tables
        sf, skew = parse_key(key)
        _DS.clear()
        _DS[key] = load_tables(generate(sf, skew, 0))
    return _DS[key]


@pytest.mark.parametrize("key", sorted(RES))
@pytest.mark.parametrize("qid", ["Q1", "Q3", "Q6", "Q12", "Q14", "Q19"])
def test_query_matches_reference(key, qid):
    P = _dev()
    tables = device_tables(key)
    got = P.reference_run(qid, tables)
    assert_table_matches(got, RES[key][qid], f"{key}/{qid}")


@pytest.mark.parametrize("variant", ["default", "pa", "pb"])
def test_q12_variants_single_gpu(variant):
    P = _dev()
    key = "sf0.01_skew0.0"
    res, rep = P.run_query("Q12", variant, tables=device_tables(key),
                           scheme="default_keys" if variant == "default" else "unpartitioned")
    assert_table_matches(res, RES[key]["Q12"], variant)
    assert rep.exchange_counts == P.get_plan("Q12", variant).expected_exchanges


def test_q6_fixed_point_exact():
    """Q6 revenue as an exact integer (cents x percent) == integer restatement."""
    from paper_2506_09226_b200.data import generate
    from paper_2506_09226_b200.engine import load_tables
    import paper_2506_09226_b200.relops as R
    from paper_2506_09226_b200.table import date_to_days as d
    ds = generate(0.1, 0.0, 0)
    li = ds.tables["lineitem"]
    sd = li.column("l_shipdate").to_int64()
    dc = li.column("l_discount").to_int64()
    qt = li.column("l_quantity").to_int64()
    ex = li.column("l_extendedprice").to_int64()
    m = (sd >= d("1994-01-01")) & (sd < d("1995-01-01")) & (dc >= 5) & (dc <= 7) & (qt < 24)
    exact = int((ex[m] * dc[m]).sum())                 # units of 1e-4 dollars
    t = load_tables(ds)["lineitem"]
    f = R.filter_table(t, (t["l_shipdate"] >= d("1994-01-01")) & (t["l_shipdate"] < d("1995-01-01"))
                       & (t["l_discount"] >= 0.05) & (t["l_discount"] <= 0.07)
                       & (t["l_quantity"] < 24))
    f = f.with_column("rev", f["l_extendedprice"] * f["l_discount"])
    g = R.group_aggregate(f, [], {"revenue": ("sum", "rev")})
    c = g.column("revenue")
    assert c.scale == 4
    assert int(c.host()[0]) == exact


REL = load_golden("relops.json")


def _rel_tables():
    from paper_2506_09226_b200.table import Column, ColumnTable

    def up(j):
        t = O.from_jsonable(j)
        return ColumnTable({n: Column.from_numpy(k, v, d) for n, (k, v, d) in t.items()})
    return up(REL["left"]), up(REL["right_unique"]), up(REL["right_dup"])


@pytest.mark.parametrize("how", ["inner", "semi", "anti"])
def test_join_semantics(how):
    P = _dev()
    left, ru, rd = _rel_tables()
    assert_table_matches(P.local_hash_join(left, ru, [("lk", "rk")], how), REL[f"join_unique_{how}"], how)
    assert_table_matches(P.local_hash_join(left, rd, [("lk", "rk")], how), REL[f"join_dup_{how}"],
                         how + "_dup")


def _oracle_join_check(got, lt, rt, on):
    exp = O.join(lt, rt, on, "inner")
    got = got.materialize()
    assert got.column_names == list(exp)
    for name, (kind, v, _) in exp.items():
        g = got.column(name).values
        assert len(g) == len(v), (name, len(g), len(v))
        assert np.array_equal(g.astype(np.int64), v.astype(np.int64)), name


@pytest.mark.parametrize("n,m,keyspan,seed", [(200_000, 50_000, 3_000, 0),
                                              (100_000, 300_000, 20_000, 1),
                                              (50_000, 40_000, 7, 2),        # heavy duplicates
                                              (1, 100_000, 1, 3),            # one left row, all match
                                              (10_000, 10_000, 10 ** 9, 4)])  # mostly no match
def test_inner_join_duplicates_vs_oracle(n, m, keyspan, seed):
    """Inner join with duplicate build keys (relops.py:81-93): left row order,
    matches in right row order -- at sizes with heavy duplicate runs."""
    from paper_2506_09226_b200.table import Column, ColumnTable
    P = _dev()
    rng = np.random.default_rng(seed)
    lt = {"lk": ("int64", rng.integers(-5, keyspan, size=n).astype(np.int64), None),
          "lv": ("int64", np.arange(n, dtype=np.int64) * 3, None)}
    rt = {"rk": ("int64", rng.integers(0, keyspan + 5, size=m).astype(np.int64), None),
          "rv": ("date32", rng.integers(0, 20000, size=m).astype(np.int32), None)}
    up = lambda t: ColumnTable({k: Column.from_numpy(a, b, c) for k, (a, b, c) in t.items()})
    got = P.local_hash_join(up(lt), up(rt), [("lk", "rk")], "inner")
    _oracle_join_check(got, lt, rt, [("lk", "rk")])


def test_inner_join_duplicates_multikey():
    from paper_2506_09226_b200.table import Column, ColumnTable
    P = _dev()
    rng = np.random.default_rng(7)
    n, m = 30_000, 20_000
    lt = {"a": ("int64", rng.integers(0, 50, size=n), None),
          "b": ("dict", rng.integers(0, 3, size=n).astype(np.int32), ("X", "Y", "Z")),
          "lv": ("int64", np.arange(n), None)}
    rt = {"c": ("int64", rng.integers(0, 50, size=m), None),
          "d": ("dict", rng.integers(0, 3, size=m).astype(np.int32), ("X", "Y", "Z")),
          "rv": ("int64", np.arange(m) * 7, None)}
    up = lambda t: ColumnTable({k: Column.from_numpy(a, np.asarray(b), c) for k, (a, b, c) in t.items()})
    on = [("a", "c"), ("b", "d")]
    got = P.local_hash_join(up(lt), up(rt), on, "inner")
    _oracle_join_check(got, {k: (a, np.asarray(b), c) for k, (a, b, c) in lt.items()},
                       {k: (a, np.asarray(b), c) for k, (a, b, c) in rt.items()}, on)


AGGS = {"n": ("count", None), "s_f": ("sum", "lv"), "s_i": ("sum", "li"), "a_f": ("avg", "lv"),
        "mn_i": ("min", "li"), "mx_i": ("max", "li"), "mn_f": ("min", "lv"),
        "mx_d": ("max", "ld"), "s_d": ("sum", "ld")}


@pytest.mark.parametrize("keys,name", [(["lc"], "group_lc"), (["lc", "ld"], "group_lc_ld"),
                                       (["lk"], "group_lk"), ([], "group_none")])
def test_group_semantics(keys, name):
    P = _dev()
    left, _, _ = _rel_tables()
    assert_table_matches(P.group_aggregate(left, keys, AGGS), REL[name], name)


def test_sort_semantics():
    left, _, _ = _rel_tables()
    assert_table_matches(left.sort_by(["lc", "lv"], {"lv"}), REL["sort_lc_desc_lv"], "sort1")
    assert_table_matches(left.sort_by(["li", "ld"], {"li"}), REL["sort_li_ld"], "sort2")


def test_filter_then_materialize_keeps_order():
    P = _dev()
    left, _, _ = _rel_tables()
    ref = O.from_jsonable(REL["left"])
    m = (ref["li"][1] > 3) & (ref["lv"][1] <= 500.0)
    got = P.filter_table(left, (left["li"] > 3) & (left["lv"] <= 500.0)).materialize()
    assert_table_matches(got, O.to_jsonable(O.filter_(ref, m)), "filter")
    # numpy-mask filtering (reference spelling) goes through the same kernel
    got2 = P.filter_table(left, m).materialize()
    assert np.array_equal(got2.column("lk").values, ref["lk"][1][m])


def test_hash_keys_and_partition_match_reference():
    P = _dev()
    from paper_2506_09226_b200.table import Column, ColumnTable
    k = load_golden("hash_kats.json")
    t = ColumnTable({"k": Column.from_numpy("int64", np.asarray(k["keys"], dtype=np.int64))})
    h = P.hash_keys(t, ["k"]).cpu().numpy()
    assert [str(int(x)) for x in h] == k["hash_single"]
    rng = np.random.default_rng(k["partition_input_seed"])
    a = rng.integers(-(1 << 40), 1 << 40, size=2000)
    b = rng.integers(0, 50, size=2000).astype(np.int32)
    t2 = ColumnTable({"a": Column.from_numpy("int64", a), "b": Column.from_numpy("date32", b)})
    for n, exp in k["partitions"].items():
        parts = P.hash_partition(t2, ["a"], int(n))
        assert [[int(x) for x in p.column("a").values] for p in parts] == exp["single"], n
        parts2 = P.hash_partition(t2, ["a", "b"], int(n))
        assert [p.row_count for p in parts2] == exp["multi_sizes"], n
        assert [[int(x) for x in p.column("a").values[:5]] for p in parts2] == exp["multi_first"]


@pytest.mark.parametrize("n", [1, 2, 3, 8, 16, 17, 64])
def test_partition_large_stable(n):
    """Partition of SF1 lineitem on l_orderkey == oracle stable partition."""
    P = _dev()
    from paper_2506_09226_b200.data import generate
    ds = generate(1.0, 0.0, 0)
    t = ds.tables["lineitem"].select(["l_orderkey", "l_partkey", "l_shipdate"]).to_device()
    parts = P.hash_partition(t, ["l_orderkey"], n)
    ref = ds.tables["lineitem"].select(["l_orderkey", "l_partkey", "l_shipdate"]).to_reference()
    oparts = O.hash_partition(ref, ["l_orderkey"], n)
    assert sum(p.row_count for p in parts) == t.row_count
    for p, o in zip(parts, oparts):
        for c in ("l_orderkey", "l_partkey", "l_shipdate"):
            assert np.array_equal(p.column(c).values, o[c][1])


def test_radix_sort_large_and_edge_cases():
    P = _dev()
    import torch
    from paper_2506_09226_b200.table import Column, ColumnTable
    rng = np.random.default_rng(3)
    for n in (0, 1, 5, 700, 2048, 2049, 4097, 300_000):
        a = rng.integers(-1000, 1000, size=n)
        b = rng.integers(0, 3, size=n)
        t = ColumnTable({"a": Column.from_numpy("int64", a), "b": Column.from_numpy("int64", b)})
        s = t.sort_by(["b", "a"], {"a"})
        idx = np.lexsort([-a, b]) if n else np.arange(0)
        assert np.array_equal(s.column("a").values, a[idx])
        assert np.array_equal(s.column("b").values, b[idx])
    # keys wider than 64 bits: two LSD words, each pass must keep the order
    # of the previous one for ties (small single-CTA sort and radix path)
    for n in (1500, 6000):
        c = rng.integers(0, 4, size=n)
        d = rng.integers(-(1 << 40), 1 << 40, size=n) // (1 << 38) * (1 << 38)   # many ties
        e = rng.integers(-(1 << 40), 1 << 40, size=n)
        t = ColumnTable({"c": Column.from_numpy("int64", c), "d": Column.from_numpy("int64", d),
                         "e": Column.from_numpy("int64", e)})
        s = t.sort_by(["c", "d", "e"], {"d"})
        idx = np.lexsort([e, -d, c])
        for name, ref in (("c", c), ("d", d), ("e", e)):
            assert np.array_equal(s.column(name).values, ref[idx]), (n, name)


@pytest.mark.parametrize("layout", ["sorted_sparse", "unsorted_sparse", "sorted_filtered"])
def test_group_by_clustered_key(layout):
    """Group-by on a sparse key whose domain is >> rows: a non-decreasing key
    column takes the dense-rank path (scx_sorted_rank + direct table), an
    unsorted one the hash path; both must equal the oracle's group
    (relops.py:97-160: output sorted by key, int sums exact)."""
    from paper_2506_09226_b200.table import Column, ColumnTable
    rng = np.random.default_rng(7)
    n = 200_000
    k = np.cumsum(rng.integers(0, 3, size=n)) * 997 + 5      # runs of equal keys, sparse
    if layout == "unsorted_sparse":
        k = rng.permutation(k)
    x = rng.integers(-1000, 1000, size=n)
    d = rng.integers(8000, 9000, size=n)
    ref = {"k": ("int64", k, None), "x": ("int64", x, None), "d": ("date32", d.astype(np.int32), None)}
    aggs = {"n": ("count", None), "sx": ("sum", "x"), "mn": ("min", "x"), "mx": ("max", "d")}
    t = ColumnTable({n_: Column.from_numpy(kd, v) for n_, (kd, v, _) in ref.items()})
    P = _dev()
    if layout == "sorted_filtered":
        got = P.group_aggregate(P.filter_table(t, t["x"] > 0), ["k"], aggs)
        exp = O.group(O.filter_(ref, x > 0), ["k"], aggs)
    else:
        got = P.group_aggregate(t, ["k"], aggs)
        exp = O.group(ref, ["k"], aggs)
    assert_table_matches(got, O.to_jsonable(exp), layout)


@pytest.mark.parametrize("with_count", [True, False])
@pytest.mark.parametrize("dense_keys", [True, False])
def test_group_having(dense_keys, with_count):
    """group_aggregate(..., having=(name, lo, hi)) == filter(group_aggregate).
    Dense keys take the direct table with HAVING folded into its compaction;
    sparse keys the generic post-filter."""
    from paper_2506_09226_b200.table import Column, ColumnTable
    rng = np.random.default_rng(11)
    n = 200_000
    k = rng.integers(0, 50_000, size=n) * (1 if dense_keys else 1_000_003)
    x = rng.integers(0, 100, size=n)
    ref = {"k": ("int64", k, None), "x": ("int64", x, None)}
    # without a count the HAVING sum itself marks live groups (lo > 0)
    aggs = {"n": ("count", None), "sx": ("sum", "x")} if with_count else {"sx": ("sum", "x")}
    t = ColumnTable({n_: Column.from_numpy(kd, v) for n_, (kd, v, _) in ref.items()})
    got = _dev().group_aggregate(t, ["k"], aggs, having=("sx", 300, 400))
    exp = O.group(ref, ["k"], aggs)
    sx = exp["sx"][1]
    exp = O.filter_(exp, (sx >= 300) & (sx <= 400))
    assert_table_matches(got, O.to_jsonable(exp), f"having dense={dense_keys}")


@pytest.mark.parametrize("how", ["semi", "anti"])
@pytest.mark.parametrize("frac", [0.001, 0.3])
def test_bitmap_semi_join_big_probe(how, frac):
    """Semi / anti joins of a >4M-row probe side against a bitmap build: the
    kernel prefilters with a coarse bitmap staged in shared memory
    (scx_bitmap_coarsen) and must still equal np.isin (relops.py:73-76)."""
    from paper_2506_09226_b200.table import Column, ColumnTable
    rng = np.random.default_rng(5)
    n, dom = 5_000_000, 20_000_000
    k = rng.integers(1, dom + 1, size=n)
    v = rng.integers(0, 100, size=n)
    build = np.unique(rng.integers(1, dom + 1, size=int(dom * frac)))
    left = ColumnTable({"k": Column.from_numpy("int64", k), "v": Column.from_numpy("int64", v)})
    right = ColumnTable({"b": Column.from_numpy("int64", build)})
    got = _dev().local_hash_join(left, right, [("k", "b")], how).materialize()
    keep = np.isin(k, build)
    if how == "anti":
        keep = ~keep
    assert np.array_equal(got.column("k").values.astype(np.int64), k[keep])
    assert np.array_equal(got.column("v").values.astype(np.int64), v[keep])


@pytest.mark.parametrize("k", [1, 10, 100, 3000])
def test_top_k_equals_sort_head(k):
    """ColumnTable.top (radix select + sort of the candidates) == sort_by().head(k),
    ties kept in input order (table.py:198-214 stable lexsort)."""
    from paper_2506_09226_b200.table import Column, ColumnTable
    rng = np.random.default_rng(17)
    n = 200_000
    a = rng.integers(0, 5000, size=n)           # many ties on the leading key
    b = rng.integers(-50, 50, size=n)
    t = ColumnTable({"a": Column.from_numpy("int64", a), "b": Column.from_numpy("int64", b)})
    got = t.top(["a", "b"], {"a"}, k)
    idx = np.lexsort([b, -a])[:k]
    assert np.array_equal(got.column("a").values, a[idx])
    assert np.array_equal(got.column("b").values, b[idx])


@pytest.mark.parametrize("sorted_keys", [True, False])
def test_group_having_unsorted_output(sorted_keys):
    """sort=False + HAVING: a clustered key takes the stream aggregation
    (scx_sorted_group_agg, unordered output), an unclustered one the table
    path; as a set of groups both equal the oracle's group + filter."""
    from paper_2506_09226_b200.table import Column, ColumnTable
    rng = np.random.default_rng(23)
    n = 300_000
    k = np.sort(rng.integers(0, 80_000, size=n)) * 13 + 7
    if not sorted_keys:
        k = rng.permutation(k)
    x = rng.integers(0, 100, size=n)
    ref = {"k": ("int64", k, None), "x": ("int64", x, None)}
    aggs = {"sx": ("sum", "x"), "n": ("count", None), "mx": ("max", "x")}
    t = ColumnTable({n_: Column.from_numpy(kd, v) for n_, (kd, v, _) in ref.items()})
    from paper_2506_09226_b200 import relops as R
    saved, R._STREAM_AGG = R._STREAM_AGG, True     # exercise the opt-in kernel too
    try:
        got = _dev().group_aggregate(t, ["k"], aggs, sort=False,
                                     having=("sx", 250, 10 ** 9)).materialize()
    finally:
        R._STREAM_AGG = saved
    got = got.sort_by(["k"])
    exp = O.group(ref, ["k"], aggs)
    exp = O.filter_(exp, exp["sx"][1] >= 250)
    assert_table_matches(got, O.to_jsonable(exp), f"having-unsorted sorted_keys={sorted_keys}")


@pytest.mark.parametrize("k", [7, 100])
def test_top_k_wide_keys(k):
    """top(...) with sort keys wider than 64 bits: radix select on the most
    significant word, full LSD sort of the candidates (ties stay in order)."""
    from paper_2506_09226_b200.table import Column, ColumnTable
    rng = np.random.default_rng(29)
    n = 150_000
    a = rng.integers(0, 300, size=n)                       # many ties at the top word
    b = rng.integers(-(1 << 40), 1 << 40, size=n)
    c = rng.integers(-(1 << 40), 1 << 40, size=n) // 1000 * 1000
    t = ColumnTable({"a": Column.from_numpy("int64", a), "b": Column.from_numpy("int64", b),
                     "c": Column.from_numpy("int64", c)})
    got = t.top(["a", "c", "b"], {"a", "b"}, k)
    idx = np.lexsort([-b, c, -a])[:k]
    for name, ref in (("a", a), ("b", b), ("c", c)):
        assert np.array_equal(got.column(name).values, ref[idx]), name


@pytest.mark.parametrize("qid", ["Q1", "Q6"])
def test_dense_graph_replay_matches_golden(qid):
    """relops.DenseGraph (bench config 1/2): the query's device work captured
    as one CUDA graph replays to the reference's result, repeatedly."""
    import paper_2506_09226_b200 as P
    import paper_2506_09226_b200.relops as R
    key = "sf0.1_skew0.0"
    tables = device_tables(key)
    R.GRAPH_CAPTURE = []
    try:
        eager = P.reference_run(qid, tables)
        graphs = R.GRAPH_CAPTURE
    finally:
        R.GRAPH_CAPTURE = None
    assert len(graphs) == 1
    assert_table_matches(eager, RES[key][qid], f"{qid}/eager")
    for i in range(3):
        assert_table_matches(graphs[0].replay(), RES[key][qid], f"{qid}/graph{i}")


@pytest.mark.parametrize("parts", [1, 3, 8, 17])
def test_partition_direct_equals_staged(parts, monkeypatch):
    """partition.cu: the direct scatter (<= 8 parts by default) and the
    shared-memory-staged scatter produce the same stable partition."""
    import paper_2506_09226_b200 as P
    rng = np.random.default_rng(parts)
    n = 300_017
    t = P.ColumnTable({"k": P.Column("int64", rng.integers(0, 1 << 40, n)),
                       "v": P.Column("int64", np.arange(n)),
                       "b": P.Column("int64", rng.integers(0, 200, n))})
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("SCX_PART_DIRECT", mode)
        parts_t = P.hash_partition(t, ["k"], parts)
        outs[mode] = [(p.column("k").values.copy(), p.column("v").values.copy(),
                       p.column("b").values.copy()) for p in parts_t]
    for a, b in zip(outs["1"], outs["0"]):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("qid", ["Q3", "Q5", "Q7", "Q9", "Q14", "Q17", "Q19", "Q20", "Q21"])
def test_chunk_mode_equals_row_owner(qid, monkeypatch):
    """jit.cu: the chunked dense kernels (selection queues) and the row-owner
    kernels return identical results (SF0.1)."""
    import paper_2506_09226_b200 as P
    from paper_2506_09226_b200 import _lib
    tables = device_tables("sf0.1_skew0.0")
    got = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("SCX_CHUNK", mode)
        _lib.load().scx_jit_clear_plans()
        got[mode] = P.result_digest(P.reference_run(qid, tables))
    monkeypatch.delenv("SCX_CHUNK")
    _lib.load().scx_jit_clear_plans()
    assert got["1"] == got["0"], qid

"""Pin the CPU oracle (and our generator) to the real reference's outputs.

Golden fixtures come from tests/golden/make_golden.py, which ran the
unmodified reference (shufflecast) in the dev container.
"""

import hashlib

import numpy as np
import pytest

from conftest import load_golden, parse_key
from oracle import ref as O
from paper_2506_09226_b200.data import generate, partition_dataset

GEN = load_golden("generator_digests.json")
RES = load_golden("query_results.json")


@pytest.mark.parametrize("key", sorted(GEN))
def test_generator_bit_identical(key):
    """data.py:161-268: every widened column hashes to the reference's bytes."""
    sf, skew = parse_key(key)
    ds = generate(sf, skew, 0)
    for tname, tab in GEN[key].items():
        ref = ds.tables[tname].to_reference()
        assert ds.tables[tname].row_count == tab["rows"]
        for cname, info in tab["columns"].items():
            kind, v, _ = ref[cname]
            assert kind == info["kind"]
            assert str(v.dtype) == info["dtype"], (tname, cname)
            digest = hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()
            assert digest == info["sha256"], (tname, cname)


@pytest.mark.parametrize("key", sorted(RES))
def test_oracle_matches_reference_bit_exact(key):
    sf, skew = parse_key(key)
    T = generate(sf, skew, 0).to_reference()
    for q, expected in RES[key].items():
        assert O.to_jsonable(O.reference_run(q, T)) == expected, (key, q)


def test_narrowed_layout_is_smaller():
    ds = generate(0.1, 0.0, 0)
    li = ds.tables["lineitem"]
    ref_bytes = sum(v.nbytes for _, v, _ in li.to_reference().values())
    assert li.nbytes * 2.5 < ref_bytes        # ~25 B/row vs 76 B/row
    assert li.column("l_discount").values.dtype == np.int8
    assert li.column("l_shipdate").values.dtype == np.int16
    assert li.column("l_shipmode").values.dtype == np.uint8
    assert li.column("l_extendedprice").scale == 2


def test_hash_kats():
    """exchange.py:35-49 Fibonacci hash, u64 wraparound."""
    k = load_golden("hash_kats.json")
    t = {"k": ("int64", np.asarray(k["keys"], dtype=np.int64), None)}
    assert [str(int(x)) for x in O.hash_keys(t, ["k"])] == k["hash_single"]
    t2 = {"x": ("int64", np.asarray([1, 1]), None), "y": ("int64", np.asarray([2, 3]), None)}
    assert [str(int(x)) for x in O.hash_keys(t2, ["x", "y"])] == k["hash_pairs"]
    # SURVEY.md §8c derived KATs
    assert int(O.hash_keys({"k": ("int64", np.asarray([1]), None)}, ["k"])[0]) == 0xdf442d22ce4859b9


def test_hash_partition_matches_reference():
    k = load_golden("hash_kats.json")
    rng = np.random.default_rng(k["partition_input_seed"])
    a = rng.integers(-(1 << 40), 1 << 40, size=2000)
    b = rng.integers(0, 50, size=2000).astype(np.int32)
    t = {"a": ("int64", a, None), "b": ("date32", b, None)}
    for n, exp in k["partitions"].items():
        parts = O.hash_partition(t, ["a"], int(n))
        assert [[int(x) for x in p["a"][1]] for p in parts] == exp["single"]
        parts2 = O.hash_partition(t, ["a", "b"], int(n))
        assert [O.nrows(p) for p in parts2] == exp["multi_sizes"]


def test_host_partition_matches_oracle():
    ds = generate(0.01, 0.0, 0)
    pd = partition_dataset(ds, 3)
    ref_li = ds.tables["lineitem"].to_reference()
    parts = O.hash_partition(ref_li, ["l_orderkey"], 3)
    for r in range(3):
        got = pd.worker_tables(r)["lineitem"].to_reference()["l_orderkey"][1]
        assert np.array_equal(got, parts[r]["l_orderkey"][1])


def test_relops_oracle_matches_reference():
    rel = load_golden("relops.json")
    left = O.from_jsonable(rel["left"])
    ru = O.from_jsonable(rel["right_unique"])
    rd = O.from_jsonable(rel["right_dup"])
    for how in ("inner", "semi", "anti"):
        assert O.to_jsonable(O.join(left, ru, [("lk", "rk")], how)) == rel[f"join_unique_{how}"]
        assert O.to_jsonable(O.join(left, rd, [("lk", "rk")], how)) == rel[f"join_dup_{how}"]
    aggs = {"n": ("count", None), "s_f": ("sum", "lv"), "s_i": ("sum", "li"), "a_f": ("avg", "lv"),
            "mn_i": ("min", "li"), "mx_i": ("max", "li"), "mn_f": ("min", "lv"),
            "mx_d": ("max", "ld"), "s_d": ("sum", "ld")}
    assert O.to_jsonable(O.group(left, ["lc"], aggs)) == rel["group_lc"]
    assert O.to_jsonable(O.group(left, ["lc", "ld"], aggs)) == rel["group_lc_ld"]
    assert O.to_jsonable(O.group(left, ["lk"], aggs)) == rel["group_lk"]
    assert O.to_jsonable(O.group(left, [], aggs)) == rel["group_none"]
    assert O.to_jsonable(O.sort_by(left, ["lc", "lv"], {"lv"})) == rel["sort_lc_desc_lv"]
    assert O.to_jsonable(O.sort_by(left, ["li", "ld"], {"li"})) == rel["sort_li_ld"]


def test_exchange_fixture_semantics():
    """Shuffle = hash_partition of the concatenation, rank-ordered sources;
    broadcast = rank-ordered concatenation."""
    ex = load_golden("exchange.json")
    ins = [O.from_jsonable(t) for t in ex["inputs"]]
    n = len(ins)
    for r in range(n):
        parts_by_src = [O.hash_partition(t, ["k"], n)[r] for t in ins]
        exp = np.concatenate([p["k"][1] for p in parts_by_src])
        assert [int(x) for x in exp] == ex["shuffle"][r]["k"]["values"]
        allk = np.concatenate([t["k"][1] for t in ins])
        assert [int(x) for x in allk] == ex["broadcast"][r]["k"]["values"]

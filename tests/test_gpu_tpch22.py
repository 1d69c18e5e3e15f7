"""GPU parity for the 16 TPC-H queries the reference lacks (+ all 22 through
run_query).

The oracle for these is builder-written (oracle/tpch_ext.py: numpy in the
reference's style, exact decimal arithmetic); the bar is the same as for the
reference's six: keys, counts, integer / date / dict columns and row order
bit-exact, float64 within rtol 1e-9.
"""

import numpy as np
import pytest

from oracle import ref as O
from oracle import tpch_ext as E

pytestmark = pytest.mark.gpu

RTOL = 1e-9
EXT = sorted(E.QUERIES, key=lambda q: int(q[1:]))
_CACHE = {}


def _datasets(key):
    """(device tables, reference tables) for a dataset key, cached."""
    if key not in _CACHE:
        import paper_2506_09226_b200 as P
        from paper_2506_09226_b200.data import generate
        sf, variant = key
        ds = generate(sf, 0.0, 0)
        if variant == "sparse_orders":
            ds = drop_orders(ds)
        _CACHE.clear()
        _CACHE[key] = (P.load_tables(ds), ds.to_reference())
    return _CACHE[key]


def drop_orders(ds):
    """dbgen gives a third of the customers no orders (custkey % 3 == 0); the
    reference generator does not, which leaves Q13's zero bucket and Q22
    empty.  This variant removes those customers' orders (and their lines)."""
    from paper_2506_09226_b200.data import Dataset
    o = ds.tables["orders"]
    keep = np.flatnonzero(o.column("o_custkey").values.astype(np.int64) % 3 != 0)
    kept = o.column("o_orderkey").values.astype(np.int64)[keep]
    li = ds.tables["lineitem"]
    lk = np.flatnonzero(np.isin(li.column("l_orderkey").values.astype(np.int64), kept))
    tables = dict(ds.tables)
    tables["orders"] = o.take(keep)
    tables["lineitem"] = li.take(lk)
    return Dataset(tables, ds.sf, ds.skew, ds.seed)


def assert_same(got, exp, ctx=""):
    got = got.materialize().to_reference()
    assert list(got) == list(exp), (ctx, list(got), list(exp))
    for name, (kind, v, d) in exp.items():
        gk, gv, gd = got[name]
        assert gk == kind, (ctx, name, gk, kind)
        assert len(gv) == len(v), (ctx, name, len(gv), len(v))
        if kind == "float64":
            np.testing.assert_allclose(gv, v, rtol=RTOL, atol=0, err_msg=f"{ctx}:{name}")
        else:
            assert np.array_equal(np.asarray(gv).astype(np.int64), np.asarray(v).astype(np.int64)), \
                (ctx, name, gv[:10], v[:10])
            if kind == "dict":
                assert tuple(gd) == tuple(d), (ctx, name)


@pytest.mark.parametrize("sf", [0.01, 0.1])
@pytest.mark.parametrize("qid", EXT)
def test_extended_query_matches_oracle(qid, sf):
    import paper_2506_09226_b200 as P
    dev, ref = _datasets((sf, "plain"))
    assert_same(P.reference_run(qid, dev), O.reference_run(qid, ref), f"{qid}@SF{sf}")


@pytest.mark.parametrize("qid", ["Q13", "Q22", "Q4", "Q18", "Q21"])
def test_sparse_orders_variant(qid):
    import paper_2506_09226_b200 as P
    dev, ref = _datasets((0.1, "sparse_orders"))
    exp = O.reference_run(qid, ref)
    if qid == "Q22":
        assert O.nrows(exp) > 0          # the variant makes Q22 non-trivial
    assert_same(P.reference_run(qid, dev), exp, f"{qid}@sparse")


@pytest.mark.parametrize("qid", ["Q2", "Q5", "Q9", "Q11", "Q16", "Q20"])
def test_extended_query_sf1(qid):
    import paper_2506_09226_b200 as P
    dev, ref = _datasets((1.0, "plain"))
    assert_same(P.reference_run(qid, dev), O.reference_run(qid, ref), f"{qid}@SF1")


def test_all_22_through_run_query_with_exchange_counts():
    """run_query checks each plan's executed (shuffle, broadcast) counts
    against EXCHANGE_PLANS (engine.py:433-439 semantics)."""
    import paper_2506_09226_b200 as P
    dev, ref = _datasets((0.01, "plain"))
    for qid in P.SUPPORTED_QUERIES:
        res, rep = P.run_query(qid, "default", None, dev)
        assert rep.exchange_counts == P.get_plan(qid, "default").expected_exchanges
        assert_same(res, O.reference_run(qid, ref), qid)

"""Host logic of the e2e pass (bench.e2e_order / e2e_assignment): the
column-level upload order and the worker queues, no GPU."""
import numpy as np

import bench
from paper_2506_09226_b200 import codec
from paper_2506_09226_b200.data import cached_generate


def _host(sf=0.01):
    ds = cached_generate(sf)
    return {t: {c: (hc, pc) for (c, hc), pc in zip(ds.tables[t].columns.items(),
                                                    codec.pack_table(ds.tables[t]).values())}
            for t in ds.tables}


def test_order_covers_every_column_once_and_every_query():
    host = _host()
    order, qorder, rel, cost = bench.e2e_order(host, rate_gbs=0.01)
    assert sorted(order) == sorted((t, c) for t in host for c in host[t])
    assert sorted(qorder) == sorted(bench.QUERIES)
    # a query is released once its last column has landed: release times
    # are the running byte totals of the columns in order
    landed, t = {}, 0.0
    for tn, c in order:
        t += bench._src_bytes(host[tn][c][1]) / (0.01 * 1e6)
        landed[c] = t
    qcols = bench.query_columns({c for tn in host for c in host[tn]})
    for q in qorder:
        assert np.isclose(rel[q], max([landed[c] for c in qcols[q]] + [0.0]))


def test_search_never_worse_than_descending_cost():
    host = _host()
    owner = {c: t for t in host for c in host[t]}
    nb = {c: bench._src_bytes(host[t][c][1]) for c, t in owner.items()}
    qcols = bench.query_columns(set(owner))
    cost = dict(bench.Q_COST)
    rate = 0.01 * 1e6
    base = bench._e2e_schedule(sorted(bench.QUERIES, key=lambda q: -cost[q]), qcols, nb, cost,
                               rate)[1]
    _, qorder, _, _ = bench.e2e_order(host, cost, rate_gbs=0.01)
    assert bench._e2e_schedule(qorder, qcols, nb, cost, rate)[1] <= base + 1e-9


def test_assignment_is_a_partition_in_release_order():
    qorder = list(bench.QUERIES)
    rel = {q: float(i) for i, q in enumerate(qorder)}
    out = bench.e2e_assignment(qorder, rel, bench.Q_COST, 5)
    assert sorted(q for w in out for q in w) == sorted(qorder)
    for w in out:
        assert [q for q in qorder if q in w] == w

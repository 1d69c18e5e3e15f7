"""Bit-packed transfer encoding (codec.py / csrc/codec.cu).

CPU: the threaded host packer (scx_pack_host, libscx.so host code) round-
trips through the numpy restatement of the device unpacker for every column
of the generated dataset and for edge cases.  GPU: scx_unpack on the device
reproduces the narrowed columns bit for bit, and tables uploaded packed run
the queries to the same results.
"""

import numpy as np
import pytest

from paper_2506_09226_b200 import _lib as L
from paper_2506_09226_b200 import codec
from paper_2506_09226_b200.table import HostColumn


@pytest.fixture(scope="module")
def ds():
    from paper_2506_09226_b200.data import generate
    return generate(0.05, 0.0, 0)


def test_dataset_columns_round_trip_and_shrink(ds):
    narrow = packed = 0
    for t, ht in ds.tables.items():
        pt = codec.pack_table(ht, threads=3)
        for c, hc in ht.columns.items():
            pc = pt[c]
            got = codec.unpack_host(pc, ht.columns[pc.ref].values if pc.ref else None)
            assert got.dtype == hc.values.dtype, (t, c)
            assert np.array_equal(got, hc.values), (t, c, pc.encoding, pc.k)
            narrow += hc.values.nbytes
            packed += pc.nbytes
    assert packed < 0.6 * narrow, (packed, narrow)


def test_column_relative_dates(ds):
    li = ds.tables["lineitem"]
    pt = codec.pack_table(li, threads=2)
    dates = ["l_shipdate", "l_commitdate", "l_receiptdate"]
    diffs = [c for c in dates if pt[c].encoding == codec.DIFF]
    assert len(diffs) == 2 and min(pt[c].k for c in diffs) <= 5
    for c in diffs:
        assert pt[pt[c].ref].encoding != codec.DIFF          # no chains
        got = codec.unpack_host(pt[c], li.columns[pt[c].ref].values)
        assert np.array_equal(got, li.columns[c].values)


def test_sorted_orderkey_uses_one_bit_deltas(ds):
    pc = codec.pack_column(ds.tables["lineitem"].columns["l_orderkey"])
    assert pc.encoding == L.PACK_DELTA and pc.k == 1
    assert codec.pack_column(ds.tables["orders"].columns["o_orderkey"]).encoding == L.PACK_IOTA


@pytest.mark.parametrize("n", [0, 1, 31, 32, 33, 2047, 2048, 2049, 100_003])
@pytest.mark.parametrize("bits", [0, 1, 7, 17, 31, 32])
def test_for_edges(n, bits):
    rng = np.random.default_rng(n * 64 + bits)
    lo = -12345
    hi = lo + (1 << bits) - 1 if bits else lo
    v = rng.integers(lo, hi + 1, size=n, dtype=np.int64)
    if n:
        v[0] = hi                                     # the top of the range is used
    hc = HostColumn("int64", v, 0, None, lo, hi)
    pc = codec.pack_column(hc, threads=4)
    assert np.array_equal(codec.unpack_host(pc), v)
    if n and 0 < bits < 32:
        assert pc.encoding == L.PACK_FOR and pc.k == bits


@pytest.mark.parametrize("n", [1, 2048, 5000, 70_001])
def test_delta_edges(n):
    rng = np.random.default_rng(n)
    v = np.cumsum(rng.integers(0, 9, size=n)).astype(np.int64) + 7
    hc = HostColumn("int64", v, 0, None, int(v.min()), int(v.max()), False, True)
    pc = codec.pack_column(hc, threads=2)
    assert pc.encoding in (L.PACK_DELTA, L.PACK_FOR)
    assert np.array_equal(codec.unpack_host(pc), v)


def test_unsorted_flag_falls_back_to_for():
    v = np.array([5, 3, 9, 1], dtype=np.int32)
    pc = codec.pack_column(HostColumn("int64", v, 0, None, 1, 9, False, True))
    assert pc.encoding == L.PACK_FOR
    assert np.array_equal(codec.unpack_host(pc), v)


def test_raw_float_passthrough():
    v = np.array([0.1, 2.5, -3.25])
    pc = codec.pack_column(HostColumn("float64", v, -1))
    assert pc.encoding == codec.RAW and pc.nbytes == v.nbytes


@pytest.mark.gpu
def test_device_unpack_matches(ds):
    import torch
    for t, ht in ds.tables.items():
        for c, hc in ht.columns.items():
            pc = codec.pack_column(hc)
            if pc.encoding == codec.RAW:
                continue
            w = codec._pin(pc.words) if pc.words is not None else None
            b = codec._pin(pc.bases) if pc.bases is not None else None
            s = torch.cuda.Stream()
            buf = codec.upload_packed(pc, w, b, s)
            torch.cuda.synchronize()
            assert np.array_equal(buf.cpu().numpy(), hc.values), (t, c, pc.encoding, pc.k)


@pytest.mark.gpu
def test_packed_upload_runs_queries_identically(ds):
    import paper_2506_09226_b200 as P
    from paper_2506_09226_b200.engine import DeviceContext, load_tables, upload_tables_async
    from paper_2506_09226_b200.cluster import Endpoint
    from paper_2506_09226_b200.queries import PLAN_FUNCTIONS
    host = codec.pin_tables(ds.tables, packed=True)
    dev, ready = upload_tables_async(host)
    plain = load_tables(ds)
    ep = Endpoint(0, 1, "nccl")
    for q in ("Q1", "Q3", "Q5", "Q9", "Q18", "Q21"):
        a = PLAN_FUNCTIONS[q](DeviceContext(ep, dev, "default", "default_keys", timed=False,
                                            ready=ready))
        b = P.reference_run(q, plain)
        assert P.result_digest(a) == P.result_digest(b), q


@pytest.mark.gpu
def test_column_ordered_upload_on_worker_streams(ds):
    """Column-level upload order (bench.e2e_order) with per-column events:
    queries issued on other streams while the columns are in flight wait for
    exactly the columns they read and give the device-resident results."""
    import threading
    import torch
    import paper_2506_09226_b200 as P
    from paper_2506_09226_b200.engine import DeviceContext, load_tables, upload_tables_async
    from paper_2506_09226_b200.cluster import Endpoint
    from paper_2506_09226_b200.queries import PLAN_FUNCTIONS
    import bench
    host = codec.pin_tables(ds.tables, packed=True)
    order, qorder, _, _ = bench.e2e_order(host)
    assert sorted(order) == sorted((t, c) for t in host for c in host[t])
    assert sorted(qorder) == sorted(PLAN_FUNCTIONS)
    plain = load_tables(ds)
    ep = Endpoint(0, 1, "nccl")
    dev, ready = upload_tables_async(host, order)
    assert all(getattr(t, "column_ready", False) for t in dev.values())
    got, errs = {}, []

    def work(qs):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for q in qs:
                    got[q] = PLAN_FUNCTIONS[q](DeviceContext(ep, dev, "default", "default_keys",
                                                             timed=False, ready=ready))
                    got[q] = got[q].materialize() if got[q] is not None else None
            s.synchronize()
        except BaseException as e:      # re-raised below
            errs.append(e)

    th = [threading.Thread(target=work, args=(qorder[i::3],)) for i in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    for q in qorder:
        assert P.result_digest(got[q]) == P.result_digest(P.reference_run(q, plain)), q


def test_key_relative_dates_roundtrip(ds):
    """pack_tables: child dates stored against the parent row's date through
    the dense foreign key (FKDIFF) where >= 2 bits narrower, l_suppkey as its
    index among l_partkey's partsupp suppliers (FKIDX); a same-row DIFF may
    reference a key-relative column; every column round-trips."""
    packs = codec.pack_tables(ds.tables)
    li, od = ds.tables["lineitem"], ds.tables["orders"]
    fk = [c for c, pc in packs["lineitem"].items() if pc.encoding == codec.FKDIFF]
    assert fk, "no key-relative date column chosen"
    dec = {}
    for c in fk:
        pc = packs["lineitem"][c]
        assert pc.k + 2 <= codec.pack_column(li.columns[c]).k
        dec[c] = codec.unpack_host(pc, od.columns[pc.ref].values, li.columns[pc.fk].values)
    ix = packs["lineitem"]["l_suppkey"]
    assert ix.encoding == codec.FKIDX and ix.k == 2 and ix.fanout == 4
    dec["l_suppkey"] = codec.unpack_host(ix, ds.tables["partsupp"].columns["ps_suppkey"].values,
                                         li.columns["l_partkey"].values)
    for t, ht in ds.tables.items():
        for c, pc in packs[t].items():
            if pc.encoding in (codec.FKDIFF, codec.FKIDX):
                got = dec[c]
            elif pc.encoding == codec.DIFF:
                got = codec.unpack_host(pc, ht.columns[pc.ref].values)
            else:
                got = codec.unpack_host(pc)
            assert np.array_equal(got, ht.columns[c].values), (t, c, pc.encoding)
    assert sum(pc.nbytes for p in packs.values() for pc in p.values()) < \
        sum(codec.pack_table(ht)[c].nbytes for ht in ds.tables.values() for c in ht.columns)

"""Parity at BASELINE config 2's scale: all 22 TPC-H queries at SF10 on the
GPU against committed golden results (tests/golden/results_sf10.json).

The fixture was produced in the dev container by
tests/golden/make_scale_results.py: the six reference queries by the REAL
reference (`shufflecast.reference_run`, engine.py:463-469) on the
reference's own generate(10, 0, 0) -- checked equal to the oracle
restatement -- and the builder-written 16 by oracle/tpch_ext.py.  It also
holds the sha256 of every reference-generator column, so this test first
proves the GPU box regenerated the same SF10 data (60M lineitem rows).

Bar: keys, counts, integer / date / dict columns and row order bit-exact;
float64 within rtol 1e-9 (exact fixed-point sums rounded once).
"""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import ref as O
from test_gpu_tpch22 import assert_same

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
FIX = os.path.join(HERE, "golden", "results_sf10.json")
QUERIES = [f"Q{i}" for i in range(1, 23)]


@pytest.fixture(scope="module")
def sf10():
    import paper_2506_09226_b200 as P
    from paper_2506_09226_b200.data import cached_generate
    with open(FIX) as fh:
        fix = json.load(fh)
    ds = cached_generate(fix["sf"], 0.0, 0)
    dev = P.load_tables(ds)
    yield fix, ds, dev
    del dev


def test_sf10_data_is_the_references(sf10):
    fix, ds, _ = sf10
    digests = fix["reference_digests"]
    assert len(digests) >= 30          # every column of the reference generator
    for key, want in digests.items():
        tname, cname = key.split(".", 1)
        _, v, _ = ds.tables[tname].column(cname).to_reference()
        got = hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()
        assert got == want, key


@pytest.mark.parametrize("qid", QUERIES)
def test_query_sf10_matches_golden(sf10, qid):
    import paper_2506_09226_b200 as P
    fix, _, dev = sf10
    exp = O.from_jsonable(fix["results"][qid])
    assert_same(P.reference_run(qid, dev), exp, f"{qid}@SF10")

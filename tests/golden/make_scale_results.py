"""Golden query results at a larger scale factor (test infrastructure).

    python tests/golden/make_scale_results.py --sf 10 [--out results_sf10.json]

For the reference's six queries (Q1 Q3 Q6 Q12 Q14 Q19) the expected result is
produced by the REAL reference (`shufflecast.reference_run`,
engine.py:463-469, imported from /root/reference in the dev container) on the
reference's own `generate(sf, 0, 0)`; the oracle restatement (oracle/ref.py)
is run on our generator's data and must agree bit for bit (this pins both the
generator and the oracle at this scale).  For the builder-written 16 the
expected result is the oracle (oracle/tpch_ext.py).  Also records, per
table, sha256 digests of the reference generator's columns so the GPU box
(which has no /root/reference) can check that it regenerated the same data.

The GPU box never runs this: it reads the committed JSON.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)

REF_QUERIES = ("Q1", "Q3", "Q6", "Q12", "Q14", "Q19")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--sf", type=float, default=10.0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-reference", action="store_true",
                    help="skip the real reference (oracle only)")
    a = ap.parse_args()
    out_path = a.out or os.path.join(HERE, f"results_sf{a.sf:g}.json")

    from oracle import ref as O
    from paper_2506_09226_b200.data import generate

    t0 = time.time()
    T = generate(a.sf, 0.0, 0).to_reference()
    print(f"generated SF{a.sf} in {time.time() - t0:.1f}s", flush=True)
    results, timing = {}, {}
    for qid in sorted(O.all_queries(), key=lambda q: int(q[1:])):
        t1 = time.time()
        results[qid] = O.to_jsonable(O.reference_run(qid, T))
        timing[qid] = round(time.time() - t1, 2)
        print(qid, timing[qid], "s", flush=True)
    out = {"sf": a.sf, "skew": 0.0, "seed": 0, "results": results,
           "oracle_s_1core": timing, "reference_checked": []}

    if not a.no_reference and os.path.isdir(REF):
        sys.path.insert(0, REF)
        import shufflecast as s
        del T
        ds = s.generate(a.sf, skew=0.0, seed=0)
        ours = generate(a.sf, 0.0, 0)
        digests = {}
        for tname, tab in ds.tables.items():
            mine = ours.tables[tname].to_reference()
            for c in tab.column_names:
                v = tab.column(c).values
                d = hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest()
                m = hashlib.sha256(np.ascontiguousarray(mine[c][1]).tobytes()).hexdigest()
                assert d == m, ("generator differs from the reference", tname, c)
                digests[f"{tname}.{c}"] = d
        del ours
        out["reference_digests"] = digests
        for qid in REF_QUERIES:
            t1 = time.time()
            got = s.reference_run(qid, ds)
            ser = {}
            for name in got.column_names:
                col = got.column(name)
                ser[name] = O.to_jsonable({name: (col.kind, col.values, col.dictionary)})[name]
            assert ser == results[qid], f"oracle differs from the reference at SF{a.sf}: {qid}"
            out["reference_checked"].append(qid)
            print("reference", qid, round(time.time() - t1, 2), "s (matches the oracle)", flush=True)
    with open(out_path, "w") as fh:
        json.dump(out, fh, indent=0)
    print("wrote", out_path)


if __name__ == "__main__":
    main()

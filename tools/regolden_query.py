"""Recompute one query's entry in a committed golden results file with the
oracle (test infrastructure), e.g. after a plan's SQL changed:

    python tools/regolden_query.py --sf 10 --query Q11
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("--sf", type=float, required=True)
ap.add_argument("--query", required=True)
ap.add_argument("--src", default=None, help="oracle_<Q>.json written by tools/sf100_cpu.py")
a = ap.parse_args()
path = os.path.join(ROOT, "tests", "golden", f"results_sf{a.sf:g}.json")
with open(path) as fh:
    gold = json.load(fh)
if a.src:
    with open(a.src) as fh:
        rec = json.load(fh)
    res, dt = rec["result"], rec["seconds_1core"]
else:
    from oracle import ref as O
    from paper_2506_09226_b200.data import generate
    T = generate(a.sf, 0.0, 0).to_reference()
    t0 = time.time()
    res = O.to_jsonable(O.reference_run(a.query, T))
    dt = time.time() - t0
gold["results"][a.query] = res
if "oracle_s_1core" in gold:
    gold["oracle_s_1core"][a.query] = round(dt, 2)
with open(path, "w") as fh:
    json.dump(gold, fh, indent=0)
print(a.query, {k: len(v.get("values", v.get("hex", []))) for k, v in res.items()})

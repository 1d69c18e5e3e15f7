"""Collect the SF100 CPU-path records written on the GPU box's host by
tools/sf100_cpu.py (gpurun_out/cpu_sf100/{oracle,reference}_Q*.json) into

* tests/golden/results_sf100.json -- the expected results of all 22 queries
  at SF100 (bench.py's `parity` check of the timed step, outside the timed
  region), in the results_sf10.json format; the reference's six are checked
  equal to the unmodified reference's own results (`reference_checked`);
* profiles/r2_cpu_sf100.json -- the measured single-core CPU time per query
  (oracle port for all 22, the unmodified reference for its six), which
  bench.py reports as `measured_at_headline_sf`.

    python tools/sf100_collect.py [gpurun_out/cpu_sf100]
"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "cpu_sf100")
REF_QUERIES = ("Q1", "Q3", "Q6", "Q12", "Q14", "Q19")


def qnum(q):
    return int(q[1:])


oracle, reference = {}, {}
for p in glob.glob(os.path.join(src, "oracle_Q*.json")):
    with open(p) as fh:
        r = json.load(fh)
    oracle[r["qid"]] = r
for p in glob.glob(os.path.join(src, "reference_Q*.json")):
    with open(p) as fh:
        r = json.load(fh)
    reference[r["qid"]] = r
qs = sorted(oracle, key=qnum)
print(f"oracle records: {len(qs)}; reference records: {sorted(reference, key=qnum)}")
checked = []
for q, r in reference.items():
    if q in oracle:
        ok = r["result"] == oracle[q]["result"]
        print(f"  {q}: reference == oracle: {ok}")
        if not ok:
            sys.exit(f"{q}: the oracle differs from the reference at SF100")
        checked.append(q)
host = ""
hp = os.path.join(src, "host.txt")
if os.path.exists(hp):
    host = open(hp).read()
sf = oracle[qs[0]]["sf"] if qs else 100.0
gold = {"sf": sf, "skew": 0.0, "seed": 0,
        "against": "oracle restatement of the CPU path (numpy, oracle/), run on the B200 box's "
                   "host at SF100 (tools/sf100_cpu.py); the reference's six queries equal the "
                   "unmodified reference's own results (reference_checked)",
        "results": {q: oracle[q]["result"] for q in qs},
        "oracle_s_1core": {q: round(oracle[q]["seconds_1core"], 2) for q in qs},
        "reference_checked": sorted(checked, key=qnum)}
with open(os.path.join(ROOT, "tests", "golden", f"results_sf{sf:g}.json"), "w") as fh:
    json.dump(gold, fh, indent=0)
prof = {"sf": sf, "n_queries": len(qs),
        "suite_s_1core": round(sum(oracle[q]["seconds_1core"] for q in qs), 1),
        "per_query_s_1core": {q: round(oracle[q]["seconds_1core"], 2) for q in qs},
        "kind": "port (oracle/, numpy) for all 22; the unmodified reference for its six below",
        "reference_s_1core": {q: round(reference[q]["seconds_1core"], 2)
                              for q in sorted(reference, key=qnum)},
        "reference_matches_oracle": sorted(checked, key=qnum),
        "host": host.strip().splitlines()[:12],
        "method": "tools/sf100_cpu.py on the B200 box's host, one query at a time on one core "
                  "(OMP_NUM_THREADS=1), data generated once and widened to the reference dtypes"}
with open(os.path.join(ROOT, "profiles", "r2_cpu_sf100.json"), "w") as fh:
    json.dump(prof, fh, indent=1)
print(f"suite {prof['suite_s_1core']} s on 1 core over {len(qs)} queries")

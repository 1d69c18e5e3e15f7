"""CPU path at SF100 on the GPU box's host (test / measurement infrastructure).

    python tools/sf100_cpu.py --phase oracle --queries Q1,Q6 [--sf 100]
    python tools/sf100_cpu.py --phase reference [--sf 100]

oracle:    the oracle restatement (oracle/ref.py + oracle/tpch_ext.py, numpy,
           one core) on our generator's SF data widened to the reference's
           dtypes; per query: the exact result (golden fixture for the GPU's
           SF100 parity check in bench.py) and its single-core time.
reference: the REAL reference (`shufflecast` installed under baseline/_ref,
           unmodified) -- its own generate(sf) and reference_run for its six
           queries, single core; the result must equal the oracle's.

Each query's record is written to gpurun_out/cpu_sf<sf>/<phase>_<qid>.json as
soon as it finishes.  A watchdog exits the process if host memory runs low
(the oracle at SF100 peaks around 130 GB; the box has ~196 GB).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("OMP_NUM_THREADS", "1")


def _mem_available_gb() -> float:
    with open("/proc/meminfo") as fh:
        for line in fh:
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) / 1e6
    return 1e9


def _watchdog(limit_gb: float, log) -> None:
    def run():
        while True:
            if _mem_available_gb() < limit_gb:
                log(f"watchdog: MemAvailable < {limit_gb} GB, exiting")
                os._exit(3)
            time.sleep(0.5)
    threading.Thread(target=run, daemon=True).start()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--phase", choices=["oracle", "reference"], required=True)
    ap.add_argument("--sf", type=float, default=100.0)
    ap.add_argument("--queries", default="")
    ap.add_argument("--out", default=None)
    ap.add_argument("--min-free-gb", type=float, default=12.0)
    a = ap.parse_args()
    out_dir = a.out or os.path.join(ROOT, "gpurun_out", f"cpu_sf{a.sf:g}")
    os.makedirs(out_dir, exist_ok=True)
    logf = open(os.path.join(out_dir, f"{a.phase}.log"), "a")

    def log(msg):
        line = f"[{time.strftime('%H:%M:%S')}] {msg}"
        print(line, flush=True)
        logf.write(line + "\n")
        logf.flush()

    _watchdog(a.min_free_gb, log)
    from oracle import ref as O
    t0 = time.time()
    if a.phase == "oracle":
        from paper_2506_09226_b200.data import cached_generate
        ds = cached_generate(a.sf, 0.0, 0)
        T = {}
        for name in list(ds.tables):
            T[name] = ds.tables[name].to_reference()
            del ds.tables[name]
            gc.collect()
        del ds
        log(f"SF{a.sf:g} generated + widened in {time.time() - t0:.0f}s, "
            f"MemAvailable {_mem_available_gb():.0f} GB")
        qs = a.queries.split(",") if a.queries else sorted(O.all_queries(), key=lambda q: int(q[1:]))
        for qid in qs:
            if os.path.exists(os.path.join(out_dir, f"oracle_{qid}.json")):
                continue
            t1 = time.perf_counter()
            res = O.reference_run(qid, T)
            dt = time.perf_counter() - t1
            with open(os.path.join(out_dir, f"oracle_{qid}.json"), "w") as fh:
                json.dump({"qid": qid, "sf": a.sf, "seconds_1core": dt,
                           "result": O.to_jsonable(res)}, fh)
            del res
            gc.collect()
            log(f"{qid} {dt:.1f}s (1 core), MemAvailable {_mem_available_gb():.0f} GB")
    else:
        sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
        import shufflecast as s
        ds = s.generate(a.sf, skew=0.0, seed=0)
        log(f"reference generate(SF{a.sf:g}) {time.time() - t0:.0f}s, "
            f"MemAvailable {_mem_available_gb():.0f} GB")
        for qid in (a.queries.split(",") if a.queries else s.SUPPORTED_QUERIES):
            t1 = time.perf_counter()
            got = s.reference_run(qid, ds)
            dt = time.perf_counter() - t1
            ser = {n: O.to_jsonable({n: (got.column(n).kind, got.column(n).values,
                                         got.column(n).dictionary)})[n] for n in got.column_names}
            rec = {"qid": qid, "sf": a.sf, "seconds_1core": dt, "result": ser}
            op = os.path.join(out_dir, f"oracle_{qid}.json")
            if os.path.exists(op):
                with open(op) as fh:
                    rec["matches_oracle"] = json.load(fh)["result"] == ser
            with open(os.path.join(out_dir, f"reference_{qid}.json"), "w") as fh:
                json.dump(rec, fh)
            log(f"reference {qid} {dt:.1f}s (1 core) matches_oracle={rec.get('matches_oracle')}")
            del got
            gc.collect()
    log(f"done in {time.time() - t0:.0f}s")


if __name__ == "__main__":
    np.seterr(all="ignore")
    main()

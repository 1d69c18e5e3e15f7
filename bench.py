"""Benchmark: TPC-H 22-query suite on B200 vs the reference's CPU path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--sf SF] [--impl ours|reference]

One "step" = one pass of all 22 TPC-H queries (the reference's six drivers
plus the builder-written 16, queries.py) over HBM-resident SF-`sf` data,
results materialised on the root.  `value` = device-timed suite
seconds (CUDA events on the launching stream, barrier + synchronize on both
sides, max over ranks).  `e2e` = the same suite through the public API with
the touched base columns copied H2D from pinned host memory inside the timed
region, results copied back.  `roofline` = the longest fused-scan launch of a
single-stream suite pass (the kernel with the largest share of the step) vs the
measured HBM copy bandwidth; `roofline_q1_scan` = Q1's scan + group-by.  `cpu_baseline` = the oracle
port of the reference (oracle/ref.py, numpy, 1 core) on a bounded SF sample,
scaled linearly to `sf`.

Under torchrun (N>1) every rank holds its default_keys partition and runs
the same plans with NCCL exchanges (weak scaling in data per GPU is NOT
claimed: total work is fixed, so scaling is "strong").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
# grow the caching allocator by remapping one expandable segment instead of
# cudaMalloc'ing new multi-GB segments (a new segment inside a timed pass cost
# 30-130 ms in Q21); must be set before torch initialises CUDA
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
sys.path.insert(0, ROOT)

METRIC = "TPC-H 22-query total time (s) at SF100, 1/2/4/8 B200; shuffle GB/s vs NVLink"
QUERIES = tuple(f"Q{i}" for i in range(1, 23))
# e2e at N=1: upload order (by first use, biggest consumers first) and the
# query order that follows table arrival (all 22 queries, each exactly once)
E2E_TABLE_ORDER = ("lineitem", "orders", "customer", "nation", "region", "supplier", "part",
                   "partsupp")
E2E_QUERY_ORDER = ("Q1", "Q6", "Q12", "Q4", "Q18", "Q3", "Q13", "Q22", "Q10", "Q5", "Q7", "Q21",
                   "Q15", "Q14", "Q19", "Q17", "Q8", "Q9", "Q2", "Q11", "Q16", "Q20")
assert sorted(E2E_QUERY_ORDER) == sorted(QUERIES)
# single-stream per-query device times at SF100 (ms, round 1): the static
# longest-first assignment of queries to worker streams and the e2e order
Q_COST = {'Q1': 2.3, 'Q2': 4.0, 'Q3': 5.3, 'Q4': 1.9, 'Q5': 4.8, 'Q6': 1.0, 'Q7': 5.5, 'Q8': 4.5,
          'Q9': 9.9, 'Q10': 3.3, 'Q11': 2.0, 'Q12': 2.3, 'Q13': 3.8, 'Q14': 2.2, 'Q15': 2.1,
          'Q16': 4.9, 'Q17': 4.0, 'Q18': 2.9, 'Q19': 3.0, 'Q20': 5.5, 'Q21': 7.8, 'Q22': 1.8}


def query_columns(names) -> dict:
    """Base columns each plan reads, read off its source: the column-name
    literals of the plan function and of the queries.py helpers it calls.
    Only orders the e2e upload (a column a plan reads but this misses is
    still waited for: Column.data waits on its own upload event)."""
    import inspect
    import re
    from paper_2506_09226_b200 import queries as QM
    from paper_2506_09226_b200.queries import PLAN_FUNCTIONS
    funcs = {n: f for n, f in vars(QM).items()
             if inspect.isfunction(f) and f.__module__ == QM.__name__}

    def lits(f, seen):
        if f.__name__ in seen:
            return set()
        seen.add(f.__name__)
        src = inspect.getsource(f)
        out = {m for m in re.findall(r'"([a-z0-9_]+)"', src) if m in names}
        for n in re.findall(r"\b(_?[a-z0-9_]+)\(", src):
            if n in funcs:
                out |= lits(funcs[n], seen)
        return out
    return {q: lits(QM_f, set()) for q, QM_f in PLAN_FUNCTIONS.items()}


REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x100: "display_clock_setting"}


def _src_bytes(src) -> int:
    """Bytes one host column sends over PCIe (packed words or the raw array)."""
    nb = getattr(src, "nbytes", None)
    if nb is None:
        nb = src.numel() * src.element_size()
    return int(nb() if callable(nb) else nb)


def _e2e_schedule(qorder, qcols, nbytes, cost, rate):
    """Columns in first-use order of `qorder` and the modelled end of the pass:
    columns land back to back at `rate` bytes/ms (one copy stream), a query
    is released when its last column has landed, the GPU runs released work
    in release order.  Also returns each query's release time (ms)."""
    seq, landed, t, rel = [], {}, 0.0, {}
    for q in qorder:
        for c in sorted(qcols[q] - landed.keys()):
            seq.append(c)
            t += nbytes[c] / rate
            landed[c] = t
        rel[q] = max([landed[c] for c in qcols[q]] + [0.0])
    gpu = 0.0
    for q in sorted(qorder, key=lambda x: rel[x]):
        gpu = max(gpu, rel[q]) + cost[q]
    return seq, gpu, rel


def e2e_assignment(qorder, rel, cost, n_workers):
    """Queries to worker streams for the e2e pass: in release order, each to
    the worker that is free first (list scheduling on the modelled release
    times), so no released query queues behind a worker's unreleased one."""
    free = [0.0] * n_workers
    out = [[] for _ in range(n_workers)]
    for q in qorder:
        j = min(range(n_workers), key=lambda w: free[w])
        out[j].append(q)
        free[j] = max(free[j], rel.get(q, 0.0)) + cost.get(q, 1.0)
    return out


def e2e_order(host: dict, cost: dict | None = None, rate_gbs: float = 54.0):
    """Column-level upload order and the matching query order for the e2e
    pass.  A query starts once the columns it reads have landed, so the pass
    ends at (upload) + (work released by the last columns): the order is a
    local search over query orders (adjacent swaps and moves, from the
    descending-cost order) minimising the modelled end of the pass
    (_e2e_schedule), with `cost` the queries' measured single-stream device
    times (ms) and each column's packed bytes over PCIe at `rate_gbs`."""
    owner = {c: t for t in host for c in host[t]}
    nbytes = {c: _src_bytes(host[t][c][1]) for c, t in owner.items()}
    qcols = query_columns(set(owner))
    # a packed column relative to others (codec DIFF / FKDIFF / FKIDX) lands
    # only after them: a query reading it waits for its whole dependency closure
    deps = {}
    for c, t in owner.items():
        pc = getattr(host[t][c][1], "col", None)
        d = set()
        if pc is not None and pc.ref is not None:
            d.add(pc.ref)
        if pc is not None and pc.fk is not None:
            d.add(pc.fk)
        deps[c] = {x for x in d if x in owner}

    def closure(cs):
        out, todo = set(), list(cs)
        while todo:
            x = todo.pop()
            if x not in out:
                out.add(x)
                todo.extend(deps.get(x, ()))
        return out
    qcols = {q: closure(cs) for q, cs in qcols.items()}
    cost = {q: (cost or {}).get(q) or Q_COST.get(q, 1.0) for q in QUERIES}
    rate = rate_gbs * 1e6                  # bytes per ms
    best = sorted(QUERIES, key=lambda x: -cost[x])
    best_t = _e2e_schedule(best, qcols, nbytes, cost, rate)[1]
    improved = True
    while improved:
        improved = False
        for i in range(len(best)):
            for j in range(len(best)):
                if i == j:
                    continue
                cand = best[:i] + best[i + 1:]
                cand.insert(j, best[i])
                t = _e2e_schedule(cand, qcols, nbytes, cost, rate)[1]
                if t < best_t - 1e-9:
                    best, best_t, improved = cand, t, True
    seq, _, rel = _e2e_schedule(best, qcols, nbytes, cost, rate)
    # the queries in release order (stable): the order the workers run them
    best = sorted(best, key=lambda q: rel[q])
    return [(owner[c], c) for c in seq], best, rel, cost


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region.

    Default ``SCX_CLOCKS=steps``: NVML from the main thread once per timed
    step, issued after the step's kernels are queued (the GPU is still
    running them); ``nvml`` = background NVML thread, ``smi`` = an
    ``nvidia-smi -lms`` subprocess, ``off`` = none (A/B of sampler
    interference).
    """

    def __init__(self, device: int, period: float = 0.05):
        import threading
        # default: an nvidia-smi subprocess.  In-process NVML sampling stalled
        # one query of a timed pass by ~80 ms (driver lock) in 3 of 4 runs;
        # SCX_CLOCKS=nvml keeps it available for comparison
        self.mode = os.environ.get("SCX_CLOCKS", "steps")
        self._h = None
        self.samples: list[tuple[float, float, int]] = []
        self.max_mhz = None
        self.proc = None
        self._stop = threading.Event()
        self._thread = None
        if self.mode == "steps":
            # NVML queried from the main thread at the end of every timed step
            # (right after the step's last kernel, GPU still at load clocks):
            # a background sampler -- in-process NVML or an nvidia-smi
            # subprocess -- intermittently stalled one query of a timed pass
            # by 70-80 ms through the driver
            try:
                import pynvml as N
                N.nvmlInit()
                idx = device
                vis = os.environ.get("CUDA_VISIBLE_DEVICES")
                if vis and vis.split(",")[device].strip().isdigit():
                    idx = int(vis.split(",")[device])
                self._N = N
                self._h = N.nvmlDeviceGetHandleByIndex(idx)
                self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(self._h, N.NVML_CLOCK_SM))
            except Exception as exc:  # pragma: no cover
                self.mode = f"unavailable ({exc})"
        elif self.mode == "nvml":
            try:
                import pynvml as N
                N.nvmlInit()
                idx = device
                vis = os.environ.get("CUDA_VISIBLE_DEVICES")
                if vis and vis.split(",")[device].strip().isdigit():
                    idx = int(vis.split(",")[device])
                h = N.nvmlDeviceGetHandleByIndex(idx)
                self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))

                def run():
                    while not self._stop.is_set():
                        try:
                            self.samples.append((
                                float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)),
                                self.max_mhz,
                                int(N.nvmlDeviceGetCurrentClocksEventReasons(h))))
                        except Exception:
                            pass
                        self._stop.wait(period)

                self._thread = threading.Thread(target=run, daemon=True)
                self._thread.start()
            except Exception as exc:  # pragma: no cover
                self.mode = f"unavailable ({exc})"
        elif self.mode == "smi":
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(device),
                     "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                     "--format=csv,noheader,nounits", "-lms", "100"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except OSError:
                self.proc = None

    def sample(self) -> None:
        """One sample now (mode "steps": called at the end of each step)."""
        if self._h is None:
            return
        N = self._N
        try:
            self.samples.append((float(N.nvmlDeviceGetClockInfo(self._h, N.NVML_CLOCK_SM)),
                                 self.max_mhz,
                                 int(N.nvmlDeviceGetCurrentClocksEventReasons(self._h))))
        except Exception:
            pass

    def stop(self) -> dict:
        if self._thread is not None:
            self._stop.set()
            self._thread.join(timeout=5)
        elif self.proc is not None:
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=10)
            for line in out.strip().splitlines():
                parts = [x.strip() for x in line.split(",")]
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except (ValueError, IndexError):
                    continue
        sm = [x[0] for x in self.samples]
        mx = [x[1] for x in self.samples if x[1]]
        reasons = set()
        for _, _, r in self.samples:
            for bit, name in REASONS.items():
                if r & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else self.max_mhz, "reasons": sorted(reasons),
                "samples": len(sm), "sampler": self.mode}


# ---------------------------------------------------------------------------
# CPU baseline: the REAL reference (shufflecast, installed unmodified under
# baseline/_ref) for its six queries + the oracle port (oracle/tpch_ext.py)
# for the 16 it lacks.  Only here and in --impl reference.
# ---------------------------------------------------------------------------

REF_QUERIES = ("Q1", "Q3", "Q6", "Q12", "Q14", "Q19")
REF_PATH = os.path.join(ROOT, "baseline", "_ref")
CPU_SF100 = os.path.join(ROOT, "profiles", "r2_cpu_sf100.json")

_WORKER = {}


def _cpu_init(sample_sf):
    """Per process: the reference's own generate() for its queries, our
    generator (value-identical, widened) for the oracle's."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from paper_2506_09226_b200.data import cached_generate
    _WORKER["port"] = cached_generate(sample_sf).to_reference()
    if os.path.isdir(REF_PATH):
        sys.path.insert(0, REF_PATH)
        import shufflecast
        _WORKER["ref"] = (shufflecast, shufflecast.generate(sample_sf, skew=0.0, seed=0))


def _cpu_query(q):
    t0 = time.perf_counter()
    if q in REF_QUERIES and "ref" in _WORKER:
        s, ds = _WORKER["ref"]
        s.reference_run(q, ds)
        kind = "reference"
    else:
        from oracle import ref as O
        O.reference_run(q, _WORKER["port"])
        kind = "port"
    return q, time.perf_counter() - t0, kind


def _cpu_sf100_profile() -> dict | None:
    """The CPU path measured at SF100 on a B200 box's host (tools/sf100_cpu.py):
    one core per query, committed under profiles/."""
    if not os.path.exists(CPU_SF100):
        return None
    with open(CPU_SF100) as fh:
        d = json.load(fh)
    return {"source": "profiles/r2_cpu_sf100.json", "sf": d.get("sf"),
            "suite_s_1core": d.get("suite_s_1core"), "queries": d.get("n_queries"),
            "reference_queries_s_1core": d.get("reference_s_1core"), "host": d.get("host")}


def cpu_suite(sample_sf: float, processes: int, steps: int, warmup: int):
    """Wall time of one pass of the 22 queries at SF `sample_sf` on a pool of
    `processes` host processes (one query per task, longest first)."""
    import multiprocessing as mp
    from paper_2506_09226_b200.data import cached_generate
    cached_generate(sample_sf)          # materialise the cache before timing
    ctx = mp.get_context("fork")
    times, per, kinds = [], {}, {}
    with ctx.Pool(processes, initializer=_cpu_init, initargs=(sample_sf,)) as pool:
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            res = pool.map(_cpu_query, sorted(QUERIES, key=lambda q: -per.get(q, 0)), chunksize=1)
            dt = time.perf_counter() - t0
            per = {q: t for q, t, _ in res}
            kinds = {q: k for q, _, k in res}
            if i >= warmup:
                times.append(dt)
    return times, per, kinds


def run_reference_arm(args) -> None:
    """--impl reference: the reference's CPU path on all host cores -- the
    unmodified reference (baseline/_ref) for its six queries, the oracle port
    for the other 16 -- one pass of all 22 queries per step on a process pool.

    A step runs on a bounded SF sample (default SF1: an SF100 pass of the
    CPU path takes ~an hour of core time and ~130 GB of host RAM, see
    profiles/r2_cpu_sf100.json): `value` is that measured sample, NOT scaled
    to the headline SF, and `config` says so (same_config: false)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sample = min(args.sf, args.cpu_sample_sf)
    cores = min(len(QUERIES), os.cpu_count() or 1)
    times, per, kinds = cpu_suite(sample, cores, args.steps, max(1, args.warmup))
    value = statistics.mean(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(value * 1e3, 2), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"TPC-H Q1-Q22 at SF{sample:g} (bounded sample of the SF{args.sf:g} "
                               f"suite; value not scaled)",
                   "sf": sample, "headline_sf": args.sf, "same_config": sample == args.sf,
                   "queries": list(QUERIES), "parallelism": f"cpu x{cores} processes"},
        "cpu_baseline": {"value": round(value, 4), "unit": "s", "cores": cores,
                         "kind": "reference" if all(kinds.get(q) == "reference"
                                                    for q in QUERIES) else "port",
                         "kinds": kinds,
                         "sample": f"one pass of all 22 queries at SF{sample:g} on {cores} "
                                   f"processes (wall time, mean of {args.steps} steps): "
                                   f"{sum(k == 'reference' for k in kinds.values())} by the "
                                   f"unmodified reference, the rest by the oracle port",
                         "per_query_s": {q: round(t, 4) for q, t in per.items()}},
        "measured_at_headline_sf": _cpu_sf100_profile(),
        "e2e": {"value": round(value, 4), "unit": "s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# shuffle microbenchmark (BASELINE config 5): per GPU B bytes of
# 16-byte rows (int64 key from default_rng(rank), int64 payload), bucket =
# the reference's hash_keys % N; partition kernel + one all-to-all-v per column
# ---------------------------------------------------------------------------

def shuffle_bench(ep, gib: float, reps: int = 5) -> dict:
    import torch
    import torch.distributed as dist
    from paper_2506_09226_b200 import exchange as X
    from paper_2506_09226_b200.table import Column, ColumnTable, alloc
    rows = int(gib * (1 << 30)) // 16
    rng = np.random.default_rng(ep.rank)
    key = torch.from_numpy(rng.integers(0, 2 ** 62, size=rows, dtype=np.int64)).cuda()
    pay = torch.arange(rows, dtype=torch.int64, device="cuda")
    t = ColumnTable({"key": Column("int64", key, 0, None, 0, 2 ** 62),
                     "payload": Column("int64", pay, 0, None, 0, rows)})
    part_ms, ex_ms = [], []
    for i in range(reps + 1):
        torch.cuda.synchronize()
        if ep.n > 1:
            dist.barrier()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        outs, out_rows = X.partition_device(t, ["key"], ep.n)
        e1.record()
        if ep.n > 1:
            in_rows, _ = X.size_exchange(ep, out_rows)
            for nm in ("key", "payload"):
                X.alltoallv(ep, outs[nm], out_rows, in_rows)
        e2.record()
        torch.cuda.synchronize()
        if i:
            part_ms.append(e0.elapsed_time(e1))
            ex_ms.append(e1.elapsed_time(e2))
        del outs
    pm, xm = statistics.mean(part_ms), statistics.mean(ex_ms)
    if ep.n > 1:
        tt = torch.tensor([pm, xm], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        pm, xm = (float(x) for x in tt.cpu())
    pk = peaks()["hbm_gbs"]
    part_bytes = rows * 16 * 2 + rows * 8       # read key+payload, write both, re-read key
    out = {"bytes_per_gpu": rows * 16, "rows_per_gpu": rows, "n_gpus": ep.n,
           "partition_ms": round(pm, 4),
           "partition_gbs": round(part_bytes / (pm / 1e3) / 1e9, 1),
           "partition_frac_hbm": round(part_bytes / (pm / 1e3) / 1e9 / pk, 4),
           "partition_alg_bytes": part_bytes}
    if ep.n > 1:
        moved = rows * 16 * (ep.n - 1) / ep.n
        gbs = moved / (xm / 1e3) / 1e9
        out.update({"exchange_ms": round(xm, 4), "exchange_gbs_per_dir": round(gbs, 1),
                    "nvlink_frac_nominal_900": round(gbs / 900.0, 4),
                    "nvlink_frac_measured_770": round(gbs / 770.0, 4),
                    "total_ms": round(pm + xm, 4)})
    else:
        out["exchange_ms"] = None
        out["note"] = "N=1: no peer to exchange with; partition kernel only"
    return out



# ---------------------------------------------------------------------------
# parity at the benchmarked scale: the GPU's results vs committed golden
# results of the CPU path at the same SF (tests/golden/results_sf<sf>.json,
# produced by tools/sf100_cpu.py / tests/golden/make_scale_results.py)
# ---------------------------------------------------------------------------

def golden_results(sf: float) -> tuple[dict | None, str | None]:
    p = os.path.join(ROOT, "tests", "golden", f"results_sf{sf:g}.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as fh:
        d = json.load(fh)
    return d, os.path.relpath(p, ROOT)


def result_mismatch(got, exp: dict, rtol: float = 1e-9) -> str | None:
    """None when `got` (a device result table) equals the serialised
    expected result: names, kinds, row order, integer / date / dict values
    bit-exact, float64 within rtol."""
    if got is None:
        return "no result"
    ref = got.materialize().to_reference()
    if list(ref) != list(exp):
        return f"columns {list(ref)} != {list(exp)}"
    for name, c in exp.items():
        kind, v, d = ref[name]
        if kind != c["kind"]:
            return f"{name}: kind {kind} != {c['kind']}"
        if kind == "float64":
            e = np.asarray([float.fromhex(x) for x in c["hex"]])
            if len(v) != len(e) or not np.allclose(v, e, rtol=rtol, atol=0):
                return f"{name}: float values differ"
        else:
            e = np.asarray(c["values"], dtype=np.int64)
            if len(v) != len(e) or not np.array_equal(np.asarray(v).astype(np.int64), e):
                return f"{name}: values differ"
            if "dictionary" in c and tuple(d) != tuple(c["dictionary"]):
                return f"{name}: dictionary differs"
    return None


def parity_report(results: dict, sf: float) -> dict:
    fix, path = golden_results(sf)
    if fix is None:
        return {"sf": sf, "checked": False, "reason": f"no tests/golden/results_sf{sf:g}.json"}
    bad = {}
    for q in QUERIES:
        if q not in fix["results"]:
            bad[q] = "not in fixture"
            continue
        m = result_mismatch(results.get(q), fix["results"][q])
        if m:
            bad[q] = m
    return {"sf": sf, "queries": len(QUERIES), "ok": not bad, "mismatches": bad,
            "against": fix.get("against", "oracle restatement of the CPU path (numpy), same "
                                          "generator data"), "fixture": path}


# ---------------------------------------------------------------------------
# BASELINE configs 1 and 2 (single queries) and 5 (partition sweep)
# ---------------------------------------------------------------------------

def time_query(qid: str, tables, steps: int, warmup: int, flush_l2, lib) -> dict:
    import torch
    from paper_2506_09226_b200.engine import DeviceContext
    from paper_2506_09226_b200.queries import PLAN_FUNCTIONS
    import paper_2506_09226_b200.relops as R
    from paper_2506_09226_b200.cluster import Endpoint

    ep = Endpoint(0, 1, "nccl")

    def run():
        r = PLAN_FUNCTIONS[qid](DeviceContext(ep, tables, "default", "default_keys", timed=False))
        return r.materialize() if r is not None else None

    for _ in range(warmup):
        run()
    R.TRACE = set()
    res = run()
    alg = sum(nb for _, nb in R.TRACE)
    R.TRACE = None
    dev, wall = [], []
    l0 = lib.scx_launch_count()
    for _ in range(steps):
        flush_l2()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        wall.append((time.perf_counter() - t0) * 1e3)
        dev.append(e0.elapsed_time(e1))
    pk = peaks()["hbm_gbs"]
    d = statistics.mean(dev)
    out = {"device_ms": round(d, 4), "wall_ms": round(statistics.mean(wall), 4),
           "alg_bytes": alg, "roof_frac": round(alg / (d / 1e3) / 1e9 / pk, 4),
           "launches": int((lib.scx_launch_count() - l0) // max(1, steps)), "result": res}
    # the same query as one CUDA graph (relops.DenseGraph: accumulator fill +
    # fused scan + D2H of the exact cells, captured once; host plan building
    # is not repeated): device and wall time per replay incl. the host finish
    R.GRAPH_CAPTURE = []
    try:
        run()
        graphs = R.GRAPH_CAPTURE
    finally:
        R.GRAPH_CAPTURE = None
    if len(graphs) == 1:
        gph = graphs[0]
        gres = gph.replay()
        gdev, gwall = [], []
        for _ in range(steps):
            flush_l2()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record()
            gph.launch()
            e1.record()
            r = gph.finish()
            gwall.append((time.perf_counter() - t0) * 1e3)
            gdev.append(e0.elapsed_time(e1))
        gd = statistics.mean(gdev)
        out["cuda_graph"] = {
            "device_ms": round(gd, 4), "wall_ms": round(statistics.mean(gwall), 4),
            "roof_frac": round(alg / (gd / 1e3) / 1e9 / pk, 4),
            "same_result": result_mismatch(gres, _serialise(res)) is None,
            "note": "fill + fused scan + D2H captured once (relops.DenseGraph); wall = replay "
                    "+ host finish; eager wall - graph wall = per-launch host overhead"}
    return out


def _serialise(t) -> dict:
    """A device result table in the golden-fixture format (result_mismatch)."""
    out = {}
    for name, (kind, v, d) in t.materialize().to_reference().items():
        c = {"kind": kind}
        if kind == "float64":
            c["hex"] = [float(x).hex() for x in v]
        else:
            c["values"] = [int(x) for x in v]
            if d is not None:
                c["dictionary"] = list(d)
        out[name] = c
    return out


def partition_sweep(sizes_gib, parts_list, reps: int = 3) -> list[dict]:
    """Config 5 on one GPU: B bytes of 16-byte rows (int64 key uniform in
    [0, 2^62), int64 payload) hash-partitioned into N destination buffers --
    the exact data movement of the fused shuffle's send (scx_part_scatter
    writing each row into its receiver's buffer), with the N receivers being
    buffers on this GPU.  NVLink is not measurable with one GPU."""
    import torch
    from paper_2506_09226_b200 import exchange as X
    from paper_2506_09226_b200.table import Column, ColumnTable, alloc
    pk = peaks()["hbm_gbs"]
    out = []
    g = torch.Generator(device="cuda")
    for gib in sizes_gib:
        rows = int(gib * (1 << 30)) // 16
        torch.cuda.empty_cache()
        free, _ = torch.cuda.mem_get_info()
        if 2 * rows * 16 + (4 << 30) > free:
            out.append({"gib": gib, "skipped": f"needs {2 * gib:g} GiB + workspace, "
                                               f"{free / 2**30:.0f} GiB free"})
            continue
        g.manual_seed(0)
        key = torch.randint(0, 2 ** 62, (rows,), dtype=torch.int64, device="cuda", generator=g)
        pay = torch.arange(rows, dtype=torch.int64, device="cuda")
        t = ColumnTable({"key": Column("int64", key, 0, None, 0, 2 ** 62),
                         "payload": Column("int64", pay, 0, None, 0, rows)})
        for n in parts_list:
            hist_ms, scat_ms = [], []
            for i in range(reps + 1):
                torch.cuda.synchronize()
                e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                e[0].record()
                P = X._Partitioner(t, ["key"], n, fetch=False)   # pass 1
                e[1].record()
                P.fetch_counts()
                bufs = [[alloc(int(P.counts[p]), np.int64) for p in range(n)] for _ in range(2)]
                dst = np.array([[b.data_ptr() for b in row] for row in bufs], np.uint64)
                e[2].record()
                P.scatter(dst)                              # pass 2 into N receivers
                e[3].record()
                torch.cuda.synchronize()
                if i:
                    hist_ms.append(e[0].elapsed_time(e[1]))
                    scat_ms.append(e[2].elapsed_time(e[3]))
                del bufs, P
            h, sc = statistics.mean(hist_ms), statistics.mean(scat_ms)
            alg = rows * 8 + rows * 32                      # key read by pass 1 + read/write rows
            out.append({"gib": gib, "rows": rows, "n_dest": n, "hist_ms": round(h, 4),
                        "scatter_ms": round(sc, 4), "total_ms": round(h + sc, 4),
                        "alg_bytes": alg, "gbs": round(alg / ((h + sc) / 1e3) / 1e9, 1),
                        "frac_hbm": round(alg / ((h + sc) / 1e3) / 1e9 / pk, 4)})
        del key, pay, t
    return out

# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--sf", type=float, default=float(os.environ.get("SCX_BENCH_SF", "100")))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-sf", type=float, default=1.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--sweep", default="1,2,4,8,16,32,64",
                    help="config-5 partition sweep sizes (GiB per GPU); empty = skip")
    ap.add_argument("--table-order", action="store_true",
                    help="e2e: upload table by table (whole-table waits' order) instead of "
                         "the column-level first-use order")
    ap.add_argument("--no-pack", action="store_true",
                    help="e2e: send the narrowed columns unpacked")
    ap.add_argument("--shuffle-gib", type=float, default=1.0)
    ap.add_argument("--streams", type=int, default=int(os.environ.get("SCX_BENCH_STREAMS", "5")),
                    help="host threads / CUDA streams running the suite's queries concurrently")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    import torch.distributed as dist
    import paper_2506_09226_b200 as P
    from paper_2506_09226_b200 import _lib
    from paper_2506_09226_b200.data import cached_generate, load_dataset
    from paper_2506_09226_b200.engine import (DeviceContext, load_tables, reserve_device_pool,
                                              upload_tables_async)
    from paper_2506_09226_b200.queries import PLAN_FUNCTIONS

    ep = P.create_cluster("nccl")
    dev = torch.cuda.current_device()
    lib = _lib.load()

    # ---- data: generated once (rank 0), cached, mmapped by every rank ----
    path = f"/tmp/scx_data/sf{args.sf}_skew0.0_seed0"
    if ep.rank == 0:
        ds = cached_generate(args.sf)
    if ep.n > 1:
        dist.barrier()
        if ep.rank != 0:
            ds = load_dataset(path)
    names = sorted(ds.tables)
    tables = load_tables(ds, ep, "default_keys", names=names)
    torch.cuda.synchronize()

    dbg = os.environ.get("SCX_BENCH_DEBUG") == "1"

    def jit_compiled():
        v = [_lib.C.c_int64() for _ in range(3)]
        lib.scx_jit_stats(*[_lib.C.byref(x) for x in v])
        return v[0].value

    def suite(tabs, per_query=None, concurrent=True):
        if n_streams > 1 and concurrent:
            return suite_concurrent(tabs, per_query)
        results = {}
        for q in QUERIES:
            if dbg:
                c0, t0 = jit_compiled(), time.perf_counter()
            if per_query is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record()
            ctx = DeviceContext(ep, tabs, "default", "default_keys", timed=False)
            r = PLAN_FUNCTIONS[q](ctx)
            if r is not None:
                r = r.materialize()
            results[q] = r
            if dbg:
                dt = (time.perf_counter() - t0) * 1e3          # host time, no sync
                if jit_compiled() != c0 or dt > 15:
                    print(f"  {q}: {dt:.1f} ms, jit compiled {jit_compiled() - c0}", file=sys.stderr)
            if per_query is not None:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record()
                per_query.append((q, e0, e1))
        return results

    def suite_concurrent(tabs, per_query=None, ready=None, order=None, assign=None):
        """The same 22 queries, pulled in order by `n_streams` host threads,
        each issuing on its own CUDA stream: one query's plan building and
        result finishing overlap another's kernels.  The step's end event
        waits for every worker stream."""
        import threading
        start = torch.cuda.Event()
        start.record()
        results, errors, lock = {}, [], threading.Lock()
        pending = list(order or QUERIES)
        done = [torch.cuda.Event() for _ in worker_streams]

        def work(i):
            try:
                torch.cuda.set_device(dev)
                s = worker_streams[i]
                with torch.cuda.stream(s):
                    s.wait_event(start)
                    if assign == "dynamic":
                        # a shared queue in `order`: each worker takes the next
                        # query as soon as it is free
                        def mine_iter():
                            while True:
                                with lock:
                                    if not pending:
                                        return
                                    q = pending.pop(0)
                                yield q
                        mine = mine_iter()
                    else:
                        mine = [q for q in (order or QUERIES) if q in (assign or assignment)[i]]
                    for q in mine:
                        if per_query is not None:
                            e0 = torch.cuda.Event(enable_timing=True)
                            e0.record()
                        ctx = DeviceContext(ep, tabs, "default", "default_keys", timed=False,
                                            ready=ready)
                        r = PLAN_FUNCTIONS[q](ctx)
                        results[q] = r.materialize() if r is not None else None
                        if per_query is not None:
                            e1 = torch.cuda.Event(enable_timing=True)
                            e1.record()
                            with lock:
                                per_query.append((q, e0, e1))
                    done[i].record(s)
            except BaseException as exc:     # re-raised on the main thread
                errors.append(exc)

        threads = [threading.Thread(target=work, args=(i,)) for i in range(n_streams)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            raise errors[0]
        cur = torch.cuda.current_stream()
        for ev in done:
            cur.wait_event(ev)
        return {q: results[q] for q in QUERIES}

    # collectives on one communicator must be issued in the same order on every
    # rank, which concurrent host threads cannot promise: N > 1 runs one stream
    n_streams = max(1, args.streams) if ep.n == 1 else 1
    # static longest-first assignment of queries to streams (by the round-1
    # single-stream per-query times, ms) so every step repeats the same
    # per-stream allocation pattern the warm-up passes already cached
    q_cost = Q_COST
    assignment = [[] for _ in range(n_streams)]
    load = [0.0] * n_streams
    for q in sorted(QUERIES, key=lambda x: -q_cost.get(x, 1.0)):
        j = load.index(min(load))
        assignment[j].append(q)
        load[j] += q_cost.get(q, 1.0)
    assignment = [[q for q in QUERIES if q in a] for a in assignment]
    worker_streams = [torch.cuda.Stream() for _ in range(n_streams)] if n_streams > 1 else []
    # cached segments for the queries' intermediates (no cudaMalloc inside the
    # timed region).  The caching allocator reuses a block only on the stream
    # that allocated it, so the budget is reserved on every stream that runs
    # queries (the worker streams, and the default stream of the single-stream
    # and e2e passes)
    budget = int(min(96, max(8, args.sf * 0.6)) * (1 << 30))
    for st in worker_streams:
        with torch.cuda.stream(st):
            reserve_device_pool(budget // (len(worker_streams) + 1))
    # the default stream runs the single-stream pass, whose largest query
    # (Q9) needs more than a worker's share (with 1/6 of the budget its
    # intermediates were cudaMalloc'ed inside the pass: Q9 10 -> 68 ms)
    reserve_device_pool(budget // 2 if worker_streams else budget)
    flush = P.table.alloc(64 << 20, np.int64)    # 512 MB > 126 MB L2

    def flush_l2():
        lib.scx_fill_i64(_lib.C.c_void_p(flush.data_ptr()), flush.numel(), 1, 0,
                         _lib.stream_ptr())

    def sync_all():
        torch.cuda.synchronize()
        if ep.n > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if ep.n == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up (the first pass also compiles / loads the plan kernels) ----
    import paper_2506_09226_b200.relops as R
    for _ in range(args.warmup):
        suite(tables)
    sync_all()
    # algorithmic bytes per query: distinct base-column bytes its scans read
    q_bytes = {}
    for q in QUERIES:
        R.TRACE = set()
        ctx = DeviceContext(ep, tables, "default", "default_keys", timed=False)
        r = PLAN_FUNCTIONS[q](ctx)
        if r is not None:
            r.materialize()
        q_bytes[q] = sum(nb for _, nb in R.TRACE)
        R.TRACE = None
    sync_all()

    # ---- timed region (device events, L2 flushed between steps) ----
    sampler = ClockSampler(dev)
    launches0 = lib.scx_launch_count()
    step_ms = []
    q_ms = {q: [] for q in QUERIES}
    import gc
    for _ in range(args.steps):
        flush_l2()
        gc.collect()          # a cyclic-GC pass inside the region showed up as
        gc.disable()          # a single 80 ms host stall in one step of Q21
        sync_all()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        per = []
        results = None          # the previous step's results are not needed now
        e0.record()
        results = suite(tables, per)
        e1.record()
        sampler.sample()        # GPU still finishing the step: load clocks + reasons
        sync_all()
        gc.enable()
        step_ms.append(e0.elapsed_time(e1))
        ms_ = torch.cuda.memory_stats()
        print(f"step {len(step_ms)}: {step_ms[-1]:.2f} ms, alloc retries "
              f"{ms_.get('num_alloc_retries', 0)}, reserved "
              f"{ms_.get('reserved_bytes.all.current', 0) / 2**30:.2f} GiB, peak "
              f"{ms_.get('allocated_bytes.all.peak', 0) / 2**30:.2f} GiB, "
              f"slowest {max(per, key=lambda x: x[1].elapsed_time(x[2]))[0] if per else '-'}",
              file=sys.stderr)
        for q, a, b in per:
            q_ms[q].append(a.elapsed_time(b))
    launches = lib.scx_launch_count() - launches0
    clocks = sampler.stop()
    ms = max_over_ranks(statistics.mean(step_ms))
    value = ms / 1e3

    # ---- parity of the timed step's results at this SF (outside the region) ----
    parity = parity_report(results, args.sf) if ep.rank == 0 else None

    # ---- the same suite on ONE stream: per-query device times that add up ----
    ss_ms = []
    q_ms1 = {q: [] for q in QUERIES}
    for _ in range(args.steps if n_streams > 1 else 0):
        flush_l2()
        gc.collect()
        gc.disable()
        sync_all()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        per = []
        e0.record()
        suite(tables, per, concurrent=False)
        e1.record()
        sync_all()
        gc.enable()
        ss_ms.append(e0.elapsed_time(e1))
        for q, a, b in per:
            q_ms1[q].append(a.elapsed_time(b))
    if n_streams == 1:
        ss_ms, q_ms1 = step_ms, q_ms

    # ---- e2e: same suite, base columns H2D from pinned host inside the region ----
    # N > 1: each rank's own rows (the default_keys hash partition, selected on
    # the host outside the timed region); only those cross PCIe per rank
    from paper_2506_09226_b200.data import REPLICATED_TABLES, worker_rows
    rank_rows = {}
    if ep.n > 1:
        for tname in names:
            if tname not in REPLICATED_TABLES:
                rank_rows[tname] = worker_rows(tname, ds.tables[tname], "default_keys",
                                               ep.n)[ep.rank]
    host_tables = {t: (ds.tables[t].take(rank_rows[t]) if t in rank_rows else ds.tables[t])
                   for t in names}
    # the host copy of each column is bit-packed once, outside the timed
    # region (codec.py: FOR / delta / iota); its words cross PCIe and are
    # unpacked on the device right behind their copy
    from paper_2506_09226_b200 import codec
    host = codec.pin_tables({t: host_tables[t] for t in names}, packed=not args.no_pack)
    h2d_bytes = codec.h2d_bytes(host)
    narrow_bytes = sum(hc.values.nbytes for t in names for hc in host_tables[t].columns.values())
    # N=1: tables stream in on a copy stream (largest / most-used first) and
    # the queries run in the order their tables arrive, each waiting only for
    # its own tables -- PCIe transfer overlapped with query execution
    copy_order = [t for t in E2E_TABLE_ORDER if t in names] + \
        [t for t in names if t not in E2E_TABLE_ORDER]
    e2e_query_order = E2E_QUERY_ORDER
    e2e_assign = None
    if ep.n == 1 and not args.table_order:
        copy_order, e2e_query_order, rel, qcost = e2e_order(
            host, {q: statistics.mean(v) for q, v in q_ms1.items() if v})
        if n_streams > 1:
            # SCX_E2E_QUEUE=dynamic: workers pull from one queue in release
            # order instead of the modelled static queues
            # (SCX_E2E_COST_SCALE: query time under contention / single-stream time)
            cs = float(os.environ.get("SCX_E2E_COST_SCALE", "1"))
            e2e_assign = ("dynamic" if os.environ.get("SCX_E2E_QUEUE") == "dynamic" else
                          e2e_assignment(e2e_query_order, rel,
                                         {q: c * cs for q, c in qcost.items()}, n_streams))
    e2e_ms, e2e_up_ms = [], []
    e2e_qdone, e2e_landed = {}, {}
    d2h_bytes = 0
    n_e2e = max(3, min(args.steps, 5))
    for i in range(n_e2e + 2):
        gc.collect()
        gc.disable()
        sync_all()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        if ep.n == 1:
            dev_tables, ready = upload_tables_async(host, copy_order)
            up_events = [ev for evs in ready.values() for ev in evs]
            if n_streams > 1:
                # the same worker streams as the device-resident suite, each
                # query waiting only for its own tables' upload events
                pq = []
                res = suite_concurrent(dev_tables, per_query=pq, ready=ready,
                                       order=e2e_query_order, assign=e2e_assign)
            else:
                res = {}
                for q in e2e_query_order:
                    ctx = DeviceContext(ep, dev_tables, "default", "default_keys", timed=False,
                                        ready=ready)
                    r = PLAN_FUNCTIONS[q](ctx)
                    res[q] = r.materialize() if r is not None else None
        else:
            dev_tables, ready = upload_tables_async(host, copy_order)
            for evs in ready.values():
                for ev in evs:
                    torch.cuda.current_stream().wait_event(ev)
            res = suite(dev_tables)
        out = {q: (r.to_reference() if r is not None else None) for q, r in res.items()}
        if ep.n == 1:
            # every uploaded column is inside the timed region, read or not
            for ev in up_events:
                torch.cuda.current_stream().wait_event(ev)
        e1.record()
        sync_all()
        if i > 1:            # two untimed passes warm the pinned path and the pools
            e2e_ms.append(e0.elapsed_time(e1))
            if ep.n == 1 and n_streams > 1:     # when each query's last kernel ended
                e2e_qdone = {q: round(e0.elapsed_time(b), 2) for q, _, b in pq}
            if ep.n == 1:                       # when each column (and its unpack) landed
                e2e_landed = {f"{t}.{c}": round(e0.elapsed_time(col._ready[0]), 2)
                              for t, tab in dev_tables.items() for c, col in tab.columns.items()
                              if col._ready is not None}
            if ep.n == 1 and up_events:   # when the last column (and its unpack) landed
                e2e_up_ms.append(max(e0.elapsed_time(ev) for ev in up_events))
        d2h_bytes = sum(v.nbytes for r in out.values() if r for _, v, _ in r.values())
        del dev_tables
        gc.enable()
    # median over the timed passes (one pass of a run occasionally stalls its
    # whole upload for ~2 s -- passes_ms keeps every pass)
    e2e_s = max_over_ranks(statistics.median(e2e_ms)) / 1e3
    # the streamed e2e pass must reproduce the device-resident results
    e2e_match = all(P.result_digest(results[q]) == P.result_digest(res[q]) if results[q] is not None
                    else res[q] is None for q in QUERIES)

    # ---- roofline: Q1's fused scan kernel timed alone (dominant single launch) ----
    pk = peaks()
    li = tables["lineitem"]
    q1_bytes = q_bytes["Q1"]
    from paper_2506_09226_b200.table import date_to_days

    f = R.filter_table(li, li["l_shipdate"] <= date_to_days("1998-09-02"))
    dp = f["l_extendedprice"] * (1.0 - f["l_discount"])
    f = f.with_column("qty_f", f["l_quantity"].astype("float64"))
    f = f.with_column("dp", dp).with_column("ch", dp * (1.0 + f["l_tax"]))
    q1_aggs = {"a": ("sum", "qty_f"), "b": ("sum", "l_extendedprice"), "c": ("sum", "dp"),
               "d": ("sum", "ch"), "e": ("sum", "l_discount"), "n": ("count", None)}
    rl_ms = []
    for i in range(8):          # events bracket exactly the one pipeline launch
        flush_l2()
        torch.cuda.synchronize()
        tm = []
        R.group_aggregate(f, ["l_returnflag", "l_linestatus"], q1_aggs, timing=tm)
        torch.cuda.synchronize()
        if i >= 2:
            rl_ms.append(tm[0][0].elapsed_time(tm[0][1]))
    k_ms = statistics.median(rl_ms)
    achieved = q1_bytes / (k_ms / 1e3) / 1e9
    traffic = None      # dram read+write of this kernel from the committed ncu capture
    tp = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tp):
        with open(tp) as fh:
            tr = json.load(fh)
        if float(tr.get("sf", -1)) == float(args.sf):
            traffic = int(tr["dram_bytes_read"]) + int(tr["dram_bytes_write"])
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"],
                "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4),
                "traffic": traffic, "kernel": "scx_pipe (Q1 fused scan + dense group-by, JIT)",
                "alg_bytes_per_launch": q1_bytes, "launch_ms": round(k_ms, 4),
                "peak_source": pk["source"]}

    # ---- the dominant kernel: every fused-scan launch of one single-stream
    # suite pass timed with CUDA events (L2 flushed before each query); the
    # longest launch is the kernel with the largest share of the step ----
    dom = None
    if ep.n == 1:
        scans = []
        for q in QUERIES:
            flush_l2()
            torch.cuda.synchronize()
            R.LAUNCH_LOG, R.LAUNCH_BYTES = [], []
            try:
                ctx = DeviceContext(ep, tables, "default", "default_keys", timed=False)
                r = PLAN_FUNCTIONS[q](ctx)
                if r is not None:
                    r.materialize()
                torch.cuda.synchronize()
                for i, ((a0, a1), nb) in enumerate(zip(R.LAUNCH_LOG, R.LAUNCH_BYTES)):
                    scans.append((a0.elapsed_time(a1), nb, q, i))
            finally:
                R.LAUNCH_LOG = None
        if scans:
            dms, nb, dq, di = max(scans)
            tot_ms = sum(x[0] for x in scans)
            dtr = dl2 = None
            tp = os.path.join(ROOT, "profiles", "roofline_traffic_dominant.json")
            if os.path.exists(tp):
                with open(tp) as fh:
                    tr = json.load(fh)
                if float(tr.get("sf", -1)) == float(args.sf) and tr.get("query") == dq:
                    dtr = int(tr["dram_bytes_read"]) + int(tr["dram_bytes_write"])
                    dl2 = tr.get("l2")
            dom = {"bound": "hbm", "achieved": round(nb / (dms / 1e3) / 1e9, 1),
                   "peak": pk["hbm_gbs"], "unit": "GB/s",
                   "frac": round(nb / (dms / 1e3) / 1e9 / pk["hbm_gbs"], 4), "traffic": dtr,
                   "kernel": f"scx_pipe: {dq}'s fused-scan launch #{di} (the longest of the suite)",
                   "alg_bytes_per_launch": nb, "launch_ms": round(dms, 4),
                   "share_of_fused_scan_time": round(dms / tot_ms, 4),
                   "peak_source": pk["source"]}
            if dl2:
                dom["l2"] = dl2      # the same launch's L2 counters (ncu --set full)

    shuffle = shuffle_bench(ep, args.shuffle_gib) if args.shuffle_gib > 0 else None

    per_query = {}
    roof_total = sum(q_bytes.values()) / (pk["hbm_gbs"] * 1e9)
    for q in QUERIES:
        t = statistics.mean(q_ms1[q]) / 1e3 if q_ms1[q] else None
        b = q_bytes[q]
        t_roof = b / (pk["hbm_gbs"] * 1e9)
        per_query[q] = {"s": round(t, 6) if t else None, "alg_bytes": b,
                        "roof_frac": round(t_roof / t, 4) if t else None,
                        "s_min": round(min(q_ms1[q]) / 1e3, 6) if q_ms1[q] else None,
                        "s_max": round(max(q_ms1[q]) / 1e3, 6) if q_ms1[q] else None,
                        "s_concurrent": round(statistics.mean(q_ms[q]) / 1e3, 6)
                        if q_ms[q] else None}

    # ---- BASELINE configs 1 / 2 and the config-5 partition sweep (1 GPU) ----
    configs = None
    if ep.n == 1 and not args.no_configs:
        from paper_2506_09226_b200.engine import load_tables as _lt
        configs = {}
        for key, qid, csf in (("config1_q6_sf1", "Q6", 1.0), ("config2_q1_sf10", "Q1", 10.0)):
            ctab = _lt(cached_generate(csf))
            r = time_query(qid, ctab, max(5, args.steps), 3, flush_l2, lib)
            fix, fpath = golden_results(csf)
            if fix is None and csf == 1.0:
                # SF1: the reference-made fixture of the six reference queries
                with open(os.path.join(ROOT, "tests", "golden", "query_results.json")) as fh:
                    fix = {"results": json.load(fh)["sf1.0_skew0.0"]}
                fpath = "tests/golden/query_results.json[sf1.0_skew0.0]"
            res = r.pop("result")
            r["parity"] = (None if fix is None else
                           {"ok": result_mismatch(res, fix["results"][qid]) is None,
                            "fixture": fpath})
            r["workload"] = f"TPC-H {qid} at SF{csf:g}, 1 GPU, L2 flushed"
            configs[key] = r
            del ctab
        if args.sweep:
            del tables, results, res
            gc.collect()
            torch.cuda.empty_cache()
            configs["config5_partition_sweep"] = {
                "note": "hash partition of B GiB of 16-byte rows into N receiver buffers on one "
                        "GPU (the fused shuffle's send); NVLink not measurable with one GPU",
                "points": partition_sweep([float(x) for x in args.sweep.split(",")],
                                          [1, 2, 4, 8])}

    cpu = None
    if ep.rank == 0 and not args.no_cpu:
        sample = min(args.sf, args.cpu_sample_sf)
        times, per_cpu, kinds = cpu_suite(sample, 1, 1, 1)
        cpu = {"value": round(times[0], 4), "unit": "s", "cores": 1,
               "kind": "port", "kinds": kinds,
               "sample": f"one pass of all 22 queries at SF{sample:g}, 1 core (after a warm-up "
                         f"pass): the unmodified reference (baseline/_ref) for "
                         f"{sum(k == 'reference' for k in kinds.values())} queries, the oracle "
                         f"port for the rest; not scaled to SF{args.sf:g}",
               "per_query_s": {q: round(t, 4) for q, t in per_cpu.items()},
               "measured_at_headline_sf": _cpu_sf100_profile()}

    if ep.rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 6), "unit": "s", "n_gpus": ep.n,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic",
            "config": {"workload": f"TPC-H Q1-Q22 at SF{args.sf} (reference drivers Q1/3/6/12/"
                                   f"14/19 + builder-written 16, one pass = one step)",
                       "sf": args.sf, "queries": list(QUERIES),
                       "parallelism": f"dp{ep.n}", "l2": "flushed between steps (512 MB write)",
                       "layout": "narrowed fixed-point columns in HBM",
                       "streams": n_streams,
                       "execution": "concurrent: queries pulled by %d host threads, one CUDA "
                                    "stream each (single_stream holds the one-stream time)"
                                    % n_streams,
                       "descriptor_limit_fallbacks": dict(R.LIMIT_FALLBACKS)},
            "e2e": {"value": round(e2e_s, 6), "unit": "s", "statistic": "median of timed passes",
                    "results_match_device_run": e2e_match,
                    "h2d_bytes_per_step": h2d_bytes,
                    "d2h_bytes_per_step": d2h_bytes,
                    "narrowed_bytes": narrow_bytes,
                    "passes_ms": [round(x, 2) for x in e2e_ms],
                    "passes_upload_done_ms": [round(x, 2) for x in e2e_up_ms],
                    "query_order": list(e2e_query_order),
                    "worker_queues": e2e_assign,
                    "last_pass_query_done_ms": e2e_qdone,
                    "last_pass_column_landed_ms": e2e_landed,
                    "encoding": "bit-packed host columns (codec.py), unpacked on the device"
                                if not args.no_pack else "narrowed columns, unpacked"},
            "roofline": dom or roofline,
            "roofline_q1_scan": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": int(launches // max(1, args.steps)),
            "gpu_launches_total": int(launches),
            "parity": parity,
            "single_stream": {"value": round(max_over_ranks(statistics.mean(ss_ms)) / 1e3, 6)
                              if ss_ms else None, "unit": "s",
                              "note": "the same suite with every query on one stream, one "
                                      "after another (per_query.s comes from this pass)"},
            "per_query": per_query,
            "per_query_note": ("s / roof_frac: the single-stream pass (queries one after "
                               "another, so they add up); s_concurrent: first-to-last event "
                               "of the query inside the concurrent timed steps"),
            "configs": configs,
            "shuffle": shuffle,
            "suite_roofline": {"t_roof_s": round(roof_total, 6),
                               "frac": round(roof_total / value, 4),
                               "rule": "sum over queries of distinct scanned bytes / HBM peak"},
        }
        print(json.dumps(line), flush=True)
    if ep.n > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

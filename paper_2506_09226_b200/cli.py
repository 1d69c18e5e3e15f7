"""Thin command line: the reference's ``query`` and
``bench`` subcommands (`shufflecast/cli.py:130-210,230-275`) on the device
engine.

    python -m paper_2506_09226_b200.cli query --qid Q3 --sf 1 --out runs/q3
    torchrun --nproc-per-node 8 -m paper_2506_09226_b200.cli query --qid all --sf 100 --out runs/
    torchrun --nproc-per-node 8 -m paper_2506_09226_b200.cli bench --op shuffle \
        --sizes-mib 1,16,256 --reps 5 --out shuffle.csv

Writes ``<qid>_result.csv`` (decoded rows, floats as repr, like
`cli.py:149-161`) and ``<qid>_report.json`` (`RunReport.to_json`, engine.py:
166-179) per query and prints the reference's one-line summary
(`cli.py:164-174`).  Under torchrun every rank runs its partition; rank 0
writes.  Failures exit nonzero with a one-line error JSON on stderr.
The reference's ``model``/``project`` subcommands (analytic models) and its
virtual-time simulator are out of scope.
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys

import numpy as np

from .data import generate
from .engine import PlanError, load_tables, run_query
from .queries import SUPPORTED_QUERIES

MIB = 1 << 20


def _fmt(value) -> str:
    """CSV cell format of the reference (`cli.py:41-46`)."""
    if value is None:
        return ""
    if isinstance(value, float):
        return f"{value:.6f}"
    return str(value)


def _write_csv(path: str, fieldnames: list[str], rows: list[dict]) -> None:
    out = sys.stdout if path == "-" else open(path, "w", newline="")
    try:
        writer = csv.writer(out)
        writer.writerow(fieldnames)
        for row in rows:
            writer.writerow([_fmt(row[f]) for f in fieldnames])
    finally:
        if out is not sys.stdout:
            out.close()


def _int_list(text: str) -> list[int]:
    return [int(x) for x in text.split(",") if x.strip()]


def _write_result_csv(path: str, table) -> None:
    with open(path, "w", newline="") as fh:
        writer = csv.writer(fh)
        if table is None:
            return
        writer.writerow(table.column_names)
        decoded = [table.column(c).decoded() for c in table.column_names]
        kinds = [table.column(c).kind for c in table.column_names]
        for i in range(table.row_count):
            writer.writerow([repr(float(col[i])) if kind == "float64" else col[i]
                             for col, kind in zip(decoded, kinds)])


def _p80(xs) -> float:
    if not xs:
        return 0.0
    # linear interpolation, as np.percentile in the reference (bench.py:209-213)
    return float(np.percentile(np.asarray(xs, dtype=np.float64), 80))


def _summarize(qid: str, report) -> str:
    return (f"{qid} [{report.variant}/{report.mode}] exchanges={report.exchange_counts} "
            f"compute={report.compute_s:.6f}s shuffle={report.shuffle_s:.6f}s "
            f"broadcast={report.broadcast_s:.6f}s "
            f"p80_shuffle_msg={_p80(report.shuffle_msgs):.0f}B "
            f"p80_broadcast_msg={_p80(report.broadcast_msgs):.0f}B "
            f"peak_bytes_max={max(report.peak_bytes)}")


def cmd_query(args) -> int:
    from .cluster import create_cluster
    qids = list(SUPPORTED_QUERIES) if args.qid == "all" else [args.qid]
    if args.variant != "default" and args.qid != "Q12":
        raise PlanError("plan variants pa/pb exist only for Q12")
    scheme = "default_keys" if args.variant == "default" else "unpartitioned"
    ep = create_cluster()
    ds = generate(args.sf, args.skew, args.seed)
    tables = load_tables(ds, ep, scheme)
    if ep.rank == 0:
        os.makedirs(args.out, exist_ok=True)
    for qid in qids:
        result, report = run_query(qid, args.variant, ep, tables, scheme=scheme)
        if ep.rank == 0:
            _write_result_csv(os.path.join(args.out, f"{qid.lower()}_result.csv"), result)
            with open(os.path.join(args.out, f"{qid.lower()}_report.json"), "w") as fh:
                fh.write(report.to_json())
            print(_summarize(qid, report))
    return 0


def cmd_bench(args) -> int:
    from . import xbench as XB
    from .cluster import create_cluster
    ep = create_cluster()
    k, v = XB.parse_shorthand(args.topology) if args.topology else (ep.n, 1)
    topo = XB.Topology(k, v,
                       bg_gbps=args.bg_gbps if args.bg_gbps is not None else 450.0,
                       bn_gbps=args.bn_gbps if args.bn_gbps is not None else 50.0,
                       efficiency=args.efficiency if args.efficiency is not None else 0.8)
    spec = XB.BenchSpec(op=args.op, message_bytes=[m * MIB for m in _int_list(args.sizes_mib)],
                        topology=topo, repetitions=args.reps,
                        max_message_bytes=args.max_mib * MIB)
    rows = XB.run_bench(ep, spec)
    if ep.rank == 0:
        _write_csv(args.out, XB.ROW_FIELDS, rows)
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="shufflecast-gpu",
                                     description="TPC-H queries on the B200 engine")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("query", help="run one query (or all 22) on a generated dataset")
    p.add_argument("--qid", required=True, choices=list(SUPPORTED_QUERIES) + ["all"])
    p.add_argument("--variant", choices=["default", "pa", "pb"], default="default")
    p.add_argument("--sf", type=float, default=0.01, help="scale factor")
    p.add_argument("--skew", type=float, default=0.0, help="Zipf exponent (0=uniform)")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", required=True, help="output directory")
    p.set_defaults(func=cmd_query)

    p = sub.add_parser("bench", help="run an exchange microbenchmark sweep")
    p.add_argument("--topology", default=None,
                   help="KxV label (default: <world size>x1); K*V must equal the world size")
    p.add_argument("--bn-gbps", type=float, default=None, help="echoed: per-machine network GB/s")
    p.add_argument("--bg-gbps", type=float, default=None, help="echoed: per-GPU NVLink GB/s")
    p.add_argument("--efficiency", type=float, default=None, help="echoed: efficiency in (0,1]")
    p.add_argument("--op", choices=["shuffle", "broadcast", "broadcast_p2p"], required=True)
    p.add_argument("--sizes-mib", required=True,
                   help="strictly increasing per-GPU message sizes in MiB")
    p.add_argument("--reps", type=int, default=1)
    p.add_argument("--max-mib", type=int, default=1024, help="memory cap per buffer")
    p.add_argument("--out", default="-", help="CSV path or - for stdout")
    p.set_defaults(func=cmd_bench)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except Exception as exc:       # one-line error JSON, nonzero exit (cli.py contract)
        print(json.dumps({"error": {"type": type(exc).__name__, "message": str(exc)}}),
              file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())

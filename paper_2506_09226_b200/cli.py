"""Thin command line: the reference's ``query`` subcommand
(`shufflecast/cli.py:177-210`) on the device engine.

    python -m paper_2506_09226_b200.cli query --qid Q3 --sf 1 --out runs/q3
    torchrun --nproc-per-node 8 -m paper_2506_09226_b200.cli query --qid all --sf 100 --out runs/

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

from .data import generate
from .engine import PlanError, load_tables, run_query
from .queries import SUPPORTED_QUERIES


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
    s = sorted(xs)
    return float(s[min(len(s) - 1, int(0.8 * (len(s) - 1) + 0.5))])


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
        result, report = run_query(qid, args.variant, ep, tables, scheme)
        if ep.rank == 0:
            _write_result_csv(os.path.join(args.out, f"{qid.lower()}_result.csv"), result)
            with open(os.path.join(args.out, f"{qid.lower()}_report.json"), "w") as fh:
                fh.write(report.to_json())
            print(_summarize(qid, report))
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
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except Exception as exc:       # one-line error JSON, nonzero exit (cli.py contract)
        print(json.dumps({"error": type(exc).__name__, "message": str(exc)}), file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())

"""Thin CLI (reference cli.py:177-210 `query`): argument handling on CPU,
one real query on the GPU."""

import csv
import json
import os

import pytest

from paper_2506_09226_b200 import cli


def test_parser_accepts_all_22_queries_and_all():
    p = cli.build_parser()
    for q in ["Q1", "Q13", "Q22", "all"]:
        a = p.parse_args(["query", "--qid", q, "--out", "x"])
        assert a.qid == q and a.variant == "default" and a.sf == 0.01


def test_variant_error_is_one_line_json(tmp_path, capsys):
    rc = cli.main(["query", "--qid", "Q3", "--variant", "pa", "--out", str(tmp_path)])
    assert rc == 1
    err = capsys.readouterr().err.strip().splitlines()
    assert len(err) == 1 and json.loads(err[0])["error"] == "PlanError"


@pytest.mark.gpu
def test_query_writes_result_and_report(tmp_path, capsys):
    assert cli.main(["query", "--qid", "Q6", "--sf", "0.01", "--out", str(tmp_path)]) == 0
    rows = list(csv.reader(open(os.path.join(tmp_path, "q6_result.csv"))))
    assert rows[0] == ["revenue"] and abs(float(rows[1][0]) - 1151588.85) < 1e-6
    rep = json.loads(open(os.path.join(tmp_path, "q6_report.json")).read())
    assert rep["exchange_counts"] == [0, 0] and rep["result_digest"]
    assert "Q6 [default/" in capsys.readouterr().out

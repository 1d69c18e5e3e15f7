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
    assert len(err) == 1 and json.loads(err[0])["error"]["type"] == "PlanError"


@pytest.mark.gpu
def test_query_writes_result_and_report(tmp_path, capsys):
    assert cli.main(["query", "--qid", "Q6", "--sf", "0.01", "--out", str(tmp_path)]) == 0
    rows = list(csv.reader(open(os.path.join(tmp_path, "q6_result.csv"))))
    assert rows[0] == ["revenue"] and abs(float(rows[1][0]) - 1151588.85) < 1e-6
    rep = json.loads(open(os.path.join(tmp_path, "q6_report.json")).read())
    assert rep["exchange_counts"] == [0, 0] and rep["result_digest"]
    assert "Q6 [default/" in capsys.readouterr().out


# ---------------------------------------------------------------------------
# bench subcommand (reference cli.py:130-145, bench.py:41-159)
# ---------------------------------------------------------------------------

from paper_2506_09226_b200 import xbench as XB  # noqa: E402


@pytest.mark.parametrize("kw,msg", [
    (dict(op="gather"), "unknown bench op"),
    (dict(repetitions=0), "repetitions must be >= 1"),
    (dict(message_bytes=[]), "empty message size sweep"),
    (dict(message_bytes=[0, 4]), "message sizes must be positive"),
    (dict(message_bytes=[4, 4]), "strictly increasing"),
    (dict(message_bytes=[1, 1 << 31]), "exceed the configured memory cap"),
])
def test_bench_spec_validation(kw, msg):
    base = dict(op="shuffle", message_bytes=[1, 2], topology=XB.Topology(1, 1))
    base.update(kw)
    with pytest.raises(XB.BenchError, match=msg):
        XB.BenchSpec(**base)


def test_topology_shorthand():
    assert XB.parse_shorthand("8x5") == (8, 5)
    with pytest.raises(XB.BenchError):
        XB.parse_shorthand("eight")


def test_bench_topology_must_match_world(tmp_path, capsys):
    rc = cli.main(["bench", "--topology", "2x1", "--op", "shuffle", "--sizes-mib", "1",
                   "--out", str(tmp_path / "x.csv")])
    assert rc == 1
    err = json.loads(capsys.readouterr().err.strip())
    assert err["error"]["type"] == "BenchError"


@pytest.mark.parametrize("op", ["shuffle", "broadcast", "broadcast_p2p"])
def test_bench_one_rank_csv_schema(tmp_path, op):
    out = tmp_path / f"{op}.csv"
    assert cli.main(["bench", "--op", op, "--sizes-mib", "1,2", "--reps", "2",
                     "--out", str(out)]) == 0
    rows = list(csv.reader(open(out)))
    assert rows[0] == XB.ROW_FIELDS
    assert [r[1] for r in rows[1:]] == [str(1 << 20), str(2 << 20)]
    for r in rows[1:]:
        assert r[0] == op and r[2:4] == ["1", "1"] and float(r[7]) > 0
        assert r[8] == "" and r[9] == ""          # no model comparison with real bytes


def _bench_worker(rank, world, port, op, q):
    try:
        import os as _os
        _os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                           WORLD_SIZE=str(world))
        import torch
        import torch.distributed as dist
        from paper_2506_09226_b200 import xbench
        from paper_2506_09226_b200.cluster import create_cluster
        ep = create_cluster("gloo")
        msg = 1000 + 3 * world                  # uneven split for the shuffle
        buf = torch.full((msg,), rank + 1, dtype=torch.uint8)
        out = torch.empty(msg * world, dtype=torch.uint8)
        xbench._step(ep, op, buf, out)
        rows = xbench.run_bench(ep, xbench.BenchSpec(op, [64, 4096], xbench.Topology(world, 1), 2))
        q.put((rank, None if op == "shuffle" else out.tolist(), rows))
        dist.destroy_process_group()
    except Exception:                           # surfaced by the parent
        import traceback
        q.put((rank, "ERR", traceback.format_exc()))


@pytest.mark.parametrize("op", ["shuffle", "broadcast", "broadcast_p2p"])
def test_bench_gloo_world2(op):
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, op, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, payload, rows in got:
        assert payload != "ERR", rows
        assert [r["msg_bytes"] for r in rows] == [64, 4096]
        assert all(r["measured_thpt_gbps"] > 0 and r["k"] == 2 for r in rows)
        if op != "shuffle":                     # every rank ends with all buffers in rank order
            msg = len(payload) // 2
            assert payload == [1] * msg + [2] * msg


@pytest.mark.gpu
def test_bench_one_gpu_nccl_path(tmp_path):
    out = tmp_path / "s.csv"
    assert cli.main(["bench", "--op", "shuffle", "--sizes-mib", "16,64", "--reps", "3",
                     "--out", str(out)]) == 0
    rows = list(csv.reader(open(out)))
    assert len(rows) == 3 and all(float(r[7]) > 0 for r in rows[1:])


@pytest.mark.parametrize("k,v,bg,bn,eff,shuf,bcast", [
    (8, 1, 900, 900, 0.8, 6582.857142857143, 822.8571428571429),
    (4, 2, 900, 50, 0.8, 160.0, 76.8),
    (8, 4, 900, 400, 0.9, 1920.0, 345.6),
    (2, 1, 900, 900, 1.0, 3600.0, 1800.0)])
def test_model_overlay_matches_reference_models(k, v, bg, bn, eff, shuf, bcast):
    """xbench's model column == shufflecast.models (values computed by the
    reference's models.py:65-89 in the dev container)."""
    from paper_2506_09226_b200.cluster import Topology
    from paper_2506_09226_b200.xbench import model_throughput
    t = Topology(k, v, bg, bn, eff)
    assert model_throughput("shuffle", t) == pytest.approx(shuf, rel=1e-12)
    assert model_throughput("broadcast", t) == pytest.approx(bcast, rel=1e-12)
    assert model_throughput("broadcast_p2p", t) == pytest.approx(bcast, rel=1e-12)

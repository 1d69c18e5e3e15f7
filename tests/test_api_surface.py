"""The drop-in API: every in-scope name of the reference package
(`/root/reference/pkg/src/shufflecast/__init__.py:9-72`) is importable from
paper_2506_09226_b200 with the reference's positional parameters first.

Out of scope (tier framing): the analytic models, the topology
parser's string front ends, CSV I/O, the virtual-time simulator's
VirtualBytes, the CPU bench harness.  `Endpoint` is constructed by the
cluster, never by users, so only its `rank` / `n` attributes are checked.
"""

import inspect
import os

import numpy as np
import pytest

import paper_2506_09226_b200 as P

# name -> positional parameters of the reference callable (None = a
# constant / exception type); generated from the reference with
# inspect.signature and checked against it below when it is present
REFERENCE = {
    "Cluster": ["topology", "mode", "seed"],
    "Column": ["kind", "values", "dictionary"],
    "ColumnTable": ["columns"],
    "Dataset": ["tables", "sf", "skew", "seed"],
    "ExchangePlan": ["query_id", "variant", "steps", "expected_exchanges", "requires_co_partition"],
    "ExchangeStats": ["messages", "table_bytes"],
    "GroupOp": ["kind", "peer", "payload", "nbytes", "tag"],
    "PartitionedDataset": ["scheme", "n_workers", "workers", "source"],
    "Topology": ["k", "v", "bg_gbps", "bn_gbps", "efficiency", "bg_efficiency", "bn_efficiency"],
    "all_reduce": ["ep", "values", "op"],
    "barrier": ["ep"],
    "broadcast_collective": ["ep", "root", "payload", "nbytes"],
    "broadcast_p2p": ["ep", "root", "payload", "nbytes"],
    "broadcast_table": ["ep", "table", "stats", "use_p2p"],
    "concat_tables": ["tables"],
    "create_cluster": ["topo", "mode", "seed"],
    "filter_table": ["table", "predicate"],
    "generate": ["sf", "skew", "seed"],
    "group_aggregate": ["table", "group_keys", "aggs"],
    "group_execute": ["ep", "ops"],
    "hash_keys": ["table", "key_columns"],
    "hash_partition": ["table", "key_columns", "n_parts"],
    "local_hash_join": ["left", "right", "on", "how"],
    "partition_dataset": ["ds", "n_workers", "scheme"],
    "q12_variants": ["cluster", "dataset"],
    "reference_run": ["qid", "tables", "variant"],
    "result_digest": ["table"],
    "run_query": ["qid", "variant", "cluster", "dataset", "p2p_broadcast"],
    "run_workers": ["cluster", "fn", "args"],
    "shuffle_table": ["ep", "table", "key_columns", "stats"],
    "size_exchange": ["ep", "my_row"],
    "tables_equal": ["a", "b"],
    "RunReport": None, "SUPPORTED_QUERIES": None, "MODE_IN_PROCESS": None,
    "MODE_SIMULATED": None, "PlanError": None, "ProtocolError": None,
    "DeadlockError": None, "TopologyError": None, "Endpoint": None,
}
OUT_OF_SCOPE = {
    "BenchSpec", "percentile", "profile_from_reports", "run_bench", "run_suite", "load_csv",
    "load_csv_dir", "write_csv", "ExchangeChoice", "ModelDomainError", "WorkloadProfile",
    "broadcast_shuffle_ratio_threshold", "broadcast_throughput", "broadcast_time",
    "choose_exchange", "local_faster_holds", "model_rows", "project_workload",
    "shuffle_throughput", "shuffle_time", "parse_config", "parse_shorthand", "VirtualBytes",
}
REF_SRC = "/root/reference/pkg/src"


def _positional(obj):
    ps = inspect.signature(obj).parameters.values()
    return [p.name for p in ps if p.kind in (p.POSITIONAL_ONLY, p.POSITIONAL_OR_KEYWORD,
                                             p.VAR_POSITIONAL)]


@pytest.mark.parametrize("name", sorted(REFERENCE))
def test_name_exported_with_reference_positionals(name):
    assert hasattr(P, name), f"{name} missing from the drop-in package"
    want = REFERENCE[name]
    if want is None or name == "Column":
        return
    got = _positional(getattr(P, name))
    assert got[:len(want)] == want, (name, want, got)


def test_column_accepts_reference_call_shape():
    # Column(kind, values, dictionary): the B200 Column takes a device tensor
    # second; host values route through from_numpy, with a positional
    # dictionary in the third slot (table.py:289-300)
    src = inspect.getsource(P.Column.__init__)
    assert "isinstance(scale, (tuple, list))" in src and "from_numpy" in src


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree not present")
def test_table_is_current_with_the_reference():
    import subprocess
    import sys
    code = ("import inspect, json, shufflecast as R\n"
            "d = {}\n"
            "for n in dir(R):\n"
            "    o = getattr(R, n)\n"
            "    if n.startswith('_') or inspect.ismodule(o): continue\n"
            "    try: d[n] = [p.name for p in inspect.signature(o).parameters.values()]\n"
            "    except (TypeError, ValueError): d[n] = None\n"
            "print(json.dumps(d))\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         env={**os.environ, "PYTHONPATH": REF_SRC}, check=True).stdout
    import json
    ref = json.loads(out)
    for n, params in ref.items():
        if n in OUT_OF_SCOPE:
            continue
        assert n in REFERENCE, f"reference exports {n}, not classified here"
        if REFERENCE[n] is not None:
            assert params[:len(REFERENCE[n])] == REFERENCE[n], n


@pytest.mark.gpu
def test_column_positional_dictionary_on_device():
    c = P.Column("dict", np.array([1, 0, 1], dtype=np.int32), ("MAIL", "SHIP"))
    assert c.dictionary == ("MAIL", "SHIP")
    assert list(c.decoded()) == ["SHIP", "MAIL", "SHIP"]

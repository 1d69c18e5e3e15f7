"""In-process cluster + collectives: host protocol semantics on CPU
(transport.py:170-442, collectives.py:57-223 of the reference).

Payloads here are numpy arrays / bytes, handed over by reference exactly as
in the reference's in-process mode; no GPU is involved.
"""

import numpy as np
import pytest

from paper_2506_09226_b200 import cluster as CL
from paper_2506_09226_b200.collectives import (all_reduce, broadcast_collective, broadcast_p2p,
                                                group_execute)


def _cl(n):
    return CL.create_cluster(CL.Topology(k=n, v=1, bg_gbps=900, bn_gbps=900), CL.MODE_IN_PROCESS)


def test_create_cluster_shapes():
    cl = _cl(4)
    assert cl.n == 4 and [ep.rank for ep in cl.endpoints] == [0, 1, 2, 3]
    assert all(ep.in_process and ep.n == 4 for ep in cl.endpoints)
    assert CL.create_cluster(3).n == 3
    with pytest.raises(CL.ClusterConfigError):
        CL.create_cluster(CL.Topology(2, 1), CL.MODE_SIMULATED)
    with pytest.raises(CL.ClusterConfigError):
        CL.create_cluster(CL.Topology(2, 1), "carrier-pigeon")
    with pytest.raises(CL.TopologyError):
        CL.Topology(0, 1)
    t = CL.Topology(k=4, v=2)
    assert t.n == 8 and t.node_of(5) == 1 and t.local_index_of(5) == 1


def test_run_workers_results_in_rank_order():
    assert CL.run_workers(_cl(5), lambda ep, x: ep.rank * x, 3) == [0, 3, 6, 9, 12]


def test_point_to_point_ring():
    def w(ep):
        ep.send((ep.rank + 1) % ep.n, f"from {ep.rank}".encode())
        return ep.recv((ep.rank - 1) % ep.n)
    assert CL.run_workers(_cl(4), w) == [b"from 3", b"from 0", b"from 1", b"from 2"]


def test_group_execute_all_to_all():
    def w(ep):
        ops = [CL.GroupOp("send", d, payload=np.full(d + 1, ep.rank, np.int64))
               for d in range(ep.n) if d != ep.rank]
        ops += [CL.GroupOp("recv", s, nbytes=8 * (ep.rank + 1)) for s in range(ep.n) if s != ep.rank]
        res = group_execute(ep, ops)
        assert all(r is None for r, op in zip(res, ops) if op.kind == "send")
        return [r.tolist() for r, op in zip(res, ops) if op.kind == "recv"]
    out = CL.run_workers(_cl(3), w)
    assert out[0] == [[1], [2]]
    assert out[2] == [[0, 0, 0], [1, 1, 1]]


def test_group_unmatched_is_deadlock():
    def w(ep):
        ops = [CL.GroupOp("send", 1, payload=b"x")] if ep.rank == 0 else []
        return group_execute(ep, ops)
    with pytest.raises(CL.DeadlockError, match="rank 0 -> rank 1"):
        CL.run_workers(_cl(2), w)


def test_group_reservation_mismatch():
    def w(ep):
        if ep.rank == 0:
            return group_execute(ep, [CL.GroupOp("send", 1, payload=b"abc")])
        return group_execute(ep, [CL.GroupOp("recv", 0, nbytes=5)])
    with pytest.raises(CL.ProtocolError, match="reservation mismatch"):
        CL.run_workers(_cl(2), w)


def test_broadcasts():
    def w(ep, p2p):
        payload = np.arange(4) * 10 if ep.rank == 2 else None
        f = broadcast_p2p if p2p else broadcast_collective
        return f(ep, 2, payload, nbytes=32).tolist()
    for p2p in (False, True):
        assert CL.run_workers(_cl(4), w, p2p) == [[0, 10, 20, 30]] * 4


def test_broadcast_root_mismatch():
    def w(ep):
        return broadcast_collective(ep, ep.rank, b"x" if True else None, nbytes=1)
    with pytest.raises(CL.ProtocolError, match="root mismatch"):
        CL.run_workers(_cl(2), w)


def test_all_reduce_rank_order_fold():
    vals = [0.1, 0.2, 0.3]

    def w(ep, op):
        return all_reduce(ep, np.asarray([vals[ep.rank], ep.rank + 1.0]), op)
    s = CL.run_workers(_cl(3), w, "sum")
    assert s[0][0] == (0.1 + 0.2) + 0.3 and all((x == s[0]).all() for x in s)
    assert CL.run_workers(_cl(3), w, "max")[1].tolist() == [0.3, 3.0]
    assert CL.run_workers(_cl(3), w, "average")[0][1] == 2.0
    with pytest.raises(CL.ProtocolError, match="unsupported reduction"):
        CL.run_workers(_cl(2), w, "median")


def test_all_reduce_length_mismatch():
    def w(ep):
        return all_reduce(ep, np.zeros(ep.rank + 1))
    with pytest.raises(CL.ProtocolError, match="length mismatch"):
        CL.run_workers(_cl(2), w)


def test_collective_label_mismatch():
    def w(ep):
        if ep.rank == 0:
            return all_reduce(ep, [1.0])
        CL.barrier(ep)
    with pytest.raises(CL.ProtocolError, match="collective mismatch"):
        CL.run_workers(_cl(2), w)


def test_worker_failure_aborts_peers():
    def w(ep):
        if ep.rank == 1:
            raise ValueError("boom")
        CL.barrier(ep)            # would wait forever for rank 1
        return ep.rank
    with pytest.raises(ValueError, match="boom"):
        CL.run_workers(_cl(3), w)


def test_missing_peer_is_deadlock():
    def w(ep):
        if ep.rank == 0:
            CL.barrier(ep)
        return ep.rank
    with pytest.raises(CL.DeadlockError):
        CL.run_workers(_cl(2), w)


def test_cluster_reusable_across_runs():
    cl = _cl(3)
    for _ in range(3):
        assert CL.run_workers(cl, lambda ep: all_reduce(ep, [ep.rank])[0]) == [3, 3, 3]


def test_single_rank_endpoint_group():
    ep = CL.Endpoint(0, 1, CL.MODE_GLOO)
    assert broadcast_collective(ep, 0, b"abc") == b"abc"
    assert all_reduce(ep, [1, 2]).tolist() == [1, 2]
    assert CL.run_workers(ep, lambda e: e.rank) == [0]

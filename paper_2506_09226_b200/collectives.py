"""Group communication primitives (drop-in for
`/root/reference/pkg/src/shufflecast/collectives.py:57-223`).

Every operation is collective: all N workers call it in the same program
order.  A group completes as a unit whatever order each worker posted its
sends and receives in; an unmatched operation raises ``DeadlockError``
naming the ranks, a disagreement raises ``ProtocolError``.

In-process clusters (``MODE_IN_PROCESS``) match the group at one
rendezvous and hand payloads over by reference (collectives.py:113,143).
Process-per-GPU jobs run the same group as one NCCL (or gloo) group of
point-to-point operations / broadcasts; payloads there are device tensors
(bytes / numpy arrays are moved to the device first) and receives need the
``nbytes`` reservation the reference also requires.

The reference charges virtual time per group; that simulator is out of
scope (cluster.py docstring).
"""

from __future__ import annotations

import numpy as np

from .cluster import DeadlockError, Endpoint, GroupOp, ProtocolError, barrier  # noqa: F401

REDUCE_OPS = ("sum", "product", "min", "max", "average")


def _nbytes(payload) -> int:
    n = getattr(payload, "nbytes", None)
    if n is not None:
        return int(n)
    try:                                   # torch tensors
        return int(payload.numel() * payload.element_size())
    except AttributeError:
        return len(payload)


def _match(cluster, slots: list[list[GroupOp]]) -> list[list]:
    """Pair the i-th send src->dst(tag) with the i-th recv at dst for
    src(tag); the k-th bcast of every rank forms one broadcast."""
    sends: dict[tuple, list] = {}
    recvs: dict[tuple, list] = {}
    bcasts: dict[int, list] = {}
    for rank, ops in enumerate(slots):
        nb = 0
        for i, op in enumerate(ops):
            if op.kind == "send":
                cluster._check_rank(op.peer, "destination")
                sends.setdefault((rank, op.peer, op.tag), []).append(op)
            elif op.kind == "recv":
                cluster._check_rank(op.peer, "source")
                recvs.setdefault((op.peer, rank, op.tag), []).append((op, i))
            elif op.kind == "bcast":
                bcasts.setdefault(nb, []).append((rank, op, i))
                nb += 1
            else:
                raise ProtocolError(f"unknown group op kind {op.kind!r}")
    bad = []
    for key in sorted(set(sends) | set(recvs)):
        s, r = len(sends.get(key, ())), len(recvs.get(key, ()))
        if s != r:
            bad.append(f"rank {key[0]} -> rank {key[1]} (tag {key[2]}): {s} send(s) vs {r} recv(s)")
    if bad:
        raise DeadlockError("unmatched operations in group: " + "; ".join(bad))
    out = [[None] * len(ops) for ops in slots]
    for key, lst in sends.items():
        src, dst, _ = key
        for op, (rop, ri) in zip(lst, recvs[key]):
            n = _nbytes(op.payload)
            if rop.nbytes is not None and rop.nbytes != n:
                raise ProtocolError(f"receive reservation mismatch at rank {dst}: expected "
                                    f"{rop.nbytes} bytes from rank {src}, got {n}")
            out[dst][ri] = op.payload
    for pos in sorted(bcasts):
        entries = bcasts[pos]
        if len(entries) != cluster.n:
            raise ProtocolError(f"broadcast #{pos} posted by ranks {sorted(r for r, _, _ in entries)}"
                                f" only; collective broadcasts require all workers")
        roots = {op.peer for _, op, _ in entries}
        if len(roots) != 1:
            raise ProtocolError(f"root mismatch across workers for broadcast #{pos}: {sorted(roots)}")
        root = roots.pop()
        cluster._check_rank(root, "root")
        payload = next(op.payload for r, op, _ in entries if r == root)
        if payload is None:
            raise ProtocolError(f"root {root} posted no payload")
        n = _nbytes(payload)
        for r, op, i in entries:
            if r != root and op.nbytes is not None and op.nbytes != n:
                raise ProtocolError(f"broadcast reservation mismatch at rank {r}: expected "
                                    f"{op.nbytes}, root {root} sent {n}")
            out[r][i] = payload
    return out


def _as_device_bytes(ep: Endpoint, payload):
    import torch
    if isinstance(payload, torch.Tensor):
        return payload.contiguous().view(torch.uint8).reshape(-1).to(ep.device)
    arr = np.frombuffer(bytes(payload), np.uint8) if not isinstance(payload, np.ndarray) \
        else np.ascontiguousarray(payload).view(np.uint8).reshape(-1)
    return torch.from_numpy(arr.copy()).to(ep.device)


def _dist_group(ep: Endpoint, ops: list[GroupOp]) -> list:
    import torch
    import torch.distributed as dist
    res: list = [None] * len(ops)
    p2p = []
    for i, op in enumerate(ops):
        if op.kind == "send":
            p2p.append(dist.P2POp(dist.isend, _as_device_bytes(ep, op.payload), op.peer,
                                  group=ep.group, tag=op.tag))
        elif op.kind == "recv":
            if op.nbytes is None:
                raise ProtocolError("recv needs an nbytes reservation across processes")
            res[i] = torch.empty(op.nbytes, dtype=torch.uint8, device=ep.device)
            p2p.append(dist.P2POp(dist.irecv, res[i], op.peer, group=ep.group, tag=op.tag))
        elif op.kind != "bcast":
            raise ProtocolError(f"unknown group op kind {op.kind!r}")
    if p2p:
        for w in dist.batch_isend_irecv(p2p):
            w.wait()
    for i, op in enumerate(ops):
        if op.kind == "bcast":
            if ep.rank == op.peer:
                buf = _as_device_bytes(ep, op.payload)
                n = torch.tensor([buf.numel()], dtype=torch.int64, device=ep.device)
            else:
                n = torch.zeros(1, dtype=torch.int64, device=ep.device)
            dist.broadcast(n, src=op.peer, group=ep.group)
            if ep.rank != op.peer:
                if op.nbytes is not None and op.nbytes != int(n.item()):
                    raise ProtocolError(f"broadcast reservation mismatch at rank {ep.rank}: "
                                        f"expected {op.nbytes}, root {op.peer} sent {int(n.item())}")
                buf = torch.empty(int(n.item()), dtype=torch.uint8, device=ep.device)
            dist.broadcast(buf, src=op.peer, group=ep.group)
            res[i] = op.payload if ep.rank == op.peer else buf
    return res


def group_execute(ep: Endpoint, ops: list[GroupOp]) -> list:
    """One group of send / recv / bcast operations; returns, aligned with
    ``ops``, the received payload for recv and bcast entries and None for
    sends (collectives.py:57-165)."""
    if ep.in_process:
        return ep.cluster.rendezvous(ep.rank, "group", list(ops),
                                     lambda slots: _match(ep.cluster, slots))[ep.rank]
    if ep.n == 1:
        class _One:                       # a 1-rank job matches against itself
            n = 1

            @staticmethod
            def _check_rank(r, what):
                if r != 0:
                    from .cluster import ClusterConfigError
                    raise ClusterConfigError(f"{what} rank {r} outside [0, 1)")
        return _match(_One, [list(ops)])[0]
    return _dist_group(ep, ops)


def broadcast_collective(ep: Endpoint, root: int, payload=None, nbytes: int | None = None):
    """One-to-all broadcast; every worker returns the root's payload
    (collectives.py:168-180)."""
    op = GroupOp("bcast", root, payload=payload if ep.rank == root else None,
                 nbytes=None if ep.rank == root else nbytes)
    return group_execute(ep, [op])[0]


def broadcast_p2p(ep: Endpoint, root: int, payload=None, nbytes: int | None = None):
    """The same broadcast as N-1 grouped sends from the root
    (collectives.py:183-196)."""
    if ep.rank == root:
        group_execute(ep, [GroupOp("send", d, payload=payload) for d in range(ep.n) if d != root])
        return payload
    return group_execute(ep, [GroupOp("recv", root, nbytes=nbytes)])[0]


def _fold(op: str, slots: list[np.ndarray]) -> np.ndarray:
    if len({s.shape for s in slots}) > 1:
        raise ProtocolError(f"all_reduce length mismatch across workers: "
                            f"{sorted({s.shape for s in slots})}")
    acc = slots[0].astype(np.float64 if op == "average" else slots[0].dtype, copy=True)
    f = {"sum": np.add, "average": np.add, "product": np.multiply,
         "min": np.minimum, "max": np.maximum}[op]
    for s in slots[1:]:                   # rank order (collectives.py:198-206)
        f(acc, s, out=acc, casting="unsafe")
    if op == "average":
        acc /= len(slots)
    return acc


def all_reduce(ep: Endpoint, values, op: str = "sum") -> np.ndarray:
    """Elementwise reduction, result on every worker; reduced in rank order
    so the floating-point result is the reference's (collectives.py:199-213)."""
    if op not in REDUCE_OPS:
        raise ProtocolError(f"unsupported reduction {op!r}; choose from {REDUCE_OPS}")
    vec = np.asarray(values)
    if ep.in_process:
        return ep.cluster.rendezvous(ep.rank, f"all_reduce:{op}", vec,
                                     lambda slots: _fold(op, slots)).copy()
    if ep.n == 1:
        return _fold(op, [vec])
    from .nccl import allgather_bytes
    shape = np.asarray(list(vec.shape) + [-1] * (4 - vec.ndim), np.int64)
    if len({tuple(r) for r in allgather_bytes(ep, shape).view(np.int64).reshape(ep.n, 4)
            .tolist()}) > 1:
        raise ProtocolError("all_reduce length mismatch across workers")
    parts = allgather_bytes(ep, np.ascontiguousarray(vec).view(np.uint8).reshape(-1))
    return _fold(op, [p.view(vec.dtype).reshape(vec.shape) for p in parts])

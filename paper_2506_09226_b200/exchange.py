"""Hash partitioning and the NVLink exchanges (shuffle / broadcast).

Drop-in for ``shufflecast.exchange`` (`/root/reference/pkg/src/shufflecast/
exchange.py`):

* ``hash_keys`` (35-49): the reference's Fibonacci hash, computed by the
  ``scx_hash_keys`` kernel with identical u64 wraparound;
* ``hash_partition`` (59-70): ``scx_partition`` = warp-aggregated histogram,
  exclusive scan, stable shared-memory-ranked scatter of every column --
  parts are contiguous in bucket order and keep input order, exactly like
  the reference's stable argsort + take;
* ``size_exchange`` (73-97): an N-int64 all-to-all of outgoing row counts;
* ``shuffle_table`` (131-174): partition once, one size exchange, then one
  all-to-all-v per column (NCCL grouped send/recv = the paper's Alg. 1)
  straight from the partitioned send buffer into a contiguous receive
  buffer ordered by source rank (exchange.py:161-166);
* ``broadcast_table`` (195-285): every rank gets the rank-ordered
  concatenation (Alg. 2: N per-root broadcasts, or N-1 sends per root with
  ``use_p2p``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .cluster import Endpoint, ProtocolError
from .table import Column, ColumnTable, SchemaError, alloc

_HASHABLE_KINDS = ("int64", "date32", "dict")


def _torch():
    import torch
    return torch


def _stream():
    return L.stream_ptr()


@dataclass
class ExchangeStats:
    """Per-worker exchange instrumentation (exchange.py:100-111)."""

    messages: list[int] = field(default_factory=list)
    table_bytes: int = 0


def _key_cols(table: ColumnTable, key_columns: list[str]) -> list[Column]:
    if not key_columns:
        raise SchemaError("at least one key column is required")
    cols = []
    for name in key_columns:
        c = table.column(name)
        if c.kind not in _HASHABLE_KINDS:
            raise SchemaError(f"column {name!r} of kind {c.kind} is not hashable; "
                              f"keys must be one of {_HASHABLE_KINDS}")
        cols.append(c)
    return cols


def hash_keys(table: ColumnTable, key_columns: list[str]):
    """u64 Fibonacci hash per row, on the device (exchange.py:35-49)."""
    table = table.materialize()
    cols = _key_cols(table, key_columns)
    n = table.row_count
    out = alloc(n, np.uint64)
    arr = (L.Column_ * len(cols))(*[c.scx() for c in cols])
    L.call("scx_hash_keys", arr, len(cols), n, C.c_void_p(out.data_ptr() if n else 0), _stream())
    return out


def partition_device(table: ColumnTable, key_columns: list[str], n_parts: int):
    """Partitioned copy of every column + per-part row counts (host ints)."""
    table = table.materialize()
    if n_parts < 1:
        raise ValueError("n_parts must be >= 1")
    cols = _key_cols(table, key_columns)
    n = table.row_count
    names = table.column_names
    outs = {nm: alloc(n, table.column(nm).np_dtype) for nm in names}
    counts = alloc(n_parts, np.uint64)
    ws = alloc(max(16, L.load().scx_partition_workspace(n, n_parts)), np.uint8)
    karr = (L.Column_ * len(cols))(*[c.scx() for c in cols])
    in_arr = (L.Column_ * max(1, len(names)))(*[table.column(nm).scx() for nm in names])
    out_arr = (L.Column_ * max(1, len(names)))(
        *[L.Column_(outs[nm].data_ptr(), table.column(nm).scx_dtype, 0) for nm in names])
    L.call("scx_partition", karr, len(cols), in_arr, out_arr, len(names), n, n_parts,
           C.c_void_p(counts.data_ptr()), C.c_void_p(ws.data_ptr()), _stream())
    cnt = [int(x) for x in counts.cpu().numpy()]
    return outs, cnt


def hash_partition(table: ColumnTable, key_columns: list[str], n_parts: int) -> list[ColumnTable]:
    """Split into n_parts by hash mod n_parts, input order kept (exchange.py:59-70)."""
    table = table.materialize()
    outs, cnt = partition_device(table, key_columns, n_parts)
    parts = []
    off = 0
    for c in cnt:
        parts.append(ColumnTable({nm: table.column(nm).like(_aligned_slice(outs[nm], off, c))
                                  for nm in table.column_names}))
        off += c
    return parts


def _aligned_slice(buf, off: int, n: int):
    """Slice [off, off+n) as a 16-byte-aligned buffer (TMA bulk copies need
    aligned column starts): a view when aligned, else a D2D copy."""
    view = buf[off:off + n]
    if view.data_ptr() % 16 == 0:
        return view
    out = alloc(n, np.dtype(str(buf.dtype).replace("torch.", "")))
    if n:
        out.copy_(view)
    return out


# ---------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------

def size_exchange(ep: Endpoint, my_row) -> tuple[np.ndarray, np.ndarray]:
    """N x N size matrix column for this rank + exclusive offsets (exchange.py:73-97)."""
    torch = _torch()
    row = np.asarray(my_row, dtype=np.int64)
    if row.shape != (ep.n,):
        raise ProtocolError(f"size exchange shape mismatch at rank {ep.rank}: "
                            f"{row.shape} for a {ep.n}-worker cluster")
    if ep.n == 1:
        incoming = row.copy()
    else:
        import torch.distributed as dist
        send = torch.from_numpy(row).to(ep.device)
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=ep.group)
        incoming = recv.cpu().numpy()
    offsets = np.zeros(len(incoming), dtype=np.int64)
    np.cumsum(incoming[:-1], out=offsets[1:])
    return incoming, offsets


def alltoallv(ep: Endpoint, send, send_counts, recv_counts):
    """One variable-size all-to-all of a 1-D tensor: parts of `send` in
    destination order -> contiguous output in source-rank order."""
    torch = _torch()
    total = int(sum(recv_counts))
    dt = np.dtype(str(send.dtype).replace("torch.", ""))
    if send.is_cuda:
        out = alloc(total, dt)
    else:
        out = torch.empty(total, dtype=send.dtype)
    if ep.n == 1:
        if total:
            out.copy_(send[:total])
        return out
    import torch.distributed as dist
    dist.all_to_all_single(out, send, [int(x) for x in recv_counts],
                           [int(x) for x in send_counts], group=ep.group)
    return out


def _check_same_schema(ep: Endpoint, table: ColumnTable, label: str):
    sig = tuple((n, c.kind, c.dictionary, str(c.np_dtype), c.scale)
                for n, c in table.columns.items())
    if ep.n == 1:
        return
    import torch.distributed as dist
    sigs = [None] * ep.n
    dist.all_gather_object(sigs, sig, group=ep.group)
    if len(set(sigs)) > 1:
        raise SchemaError(f"{label}: schema mismatch across workers")


def shuffle_table(ep: Endpoint, table, key_columns: list[str],
                  stats: ExchangeStats | None = None) -> ColumnTable:
    """Rows land on rank hash(key) mod N, received in source-rank order
    (exchange.py:131-174)."""
    table = table.materialize()
    n = ep.n
    _check_same_schema(ep, table, "shuffle")
    outs, out_rows = partition_device(table, key_columns, n)
    in_rows, _ = size_exchange(ep, out_rows)
    cols = {}
    for name in table.column_names:
        c = table.column(name)
        recv = alltoallv(ep, outs[name], out_rows, in_rows)
        cols[name] = c.like(recv)
        if stats is not None:
            stats.messages.extend(int(out_rows[d]) * c.itemsize for d in range(n)
                                  if d != ep.rank and out_rows[d] > 0)
            stats.table_bytes += c.nbytes
    if n > 1:
        cols = _merge_ranges(ep, cols)
    return ColumnTable(cols)


def broadcast_table(ep: Endpoint, table, stats: ExchangeStats | None = None,
                    use_p2p: bool = False) -> ColumnTable:
    """Every rank gets the rank-ordered concatenation (exchange.py:195-285)."""
    torch = _torch()
    table = table.materialize()
    n = ep.n
    _check_same_schema(ep, table, "broadcast")
    counts, _ = size_exchange(ep, np.full(n, table.row_count, dtype=np.int64))
    cols = {}
    for name in table.column_names:
        c = table.column(name)
        if n == 1:
            cols[name] = c
        else:
            import torch.distributed as dist
            total = int(counts.sum())
            dt = c.np_dtype
            out = alloc(total, dt) if c.data.is_cuda else torch.empty(total, dtype=c.data.dtype)
            offs = np.concatenate([[0], np.cumsum(counts)])
            if use_p2p:
                ops = []
                for peer in range(n):
                    if peer == ep.rank:
                        continue
                    ops.append(dist.P2POp(dist.isend, c.data, peer, group=ep.group))
                    ops.append(dist.P2POp(dist.irecv, out[offs[peer]:offs[peer + 1]], peer,
                                          group=ep.group))
                if ops:
                    for r in dist.batch_isend_irecv(ops):
                        r.wait()
                out[offs[ep.rank]:offs[ep.rank + 1]].copy_(c.data)
            else:
                for root in range(n):
                    seg = out[offs[root]:offs[root + 1]]
                    if root == ep.rank:
                        seg.copy_(c.data)
                    if counts[root]:
                        dist.broadcast(seg, src=root, group=ep.group)
            cols[name] = Column(c.kind, out, c.scale, c.dictionary, c.lo, c.hi)
        if stats is not None:
            if c.nbytes > 0:
                copies = (n - 1) if use_p2p else (1 if n > 1 else 0)
                stats.messages.extend([c.nbytes] * copies)
            stats.table_bytes += c.nbytes
    if n > 1:
        cols = _merge_ranges(ep, cols)
    return ColumnTable(cols)


def _merge_ranges(ep: Endpoint, cols: dict[str, Column]) -> dict[str, Column]:
    """Receivers adopt the union of every rank's [lo, hi] metadata."""
    import torch.distributed as dist
    mine = {n: (c.lo, c.hi) for n, c in cols.items()}
    allr = [None] * ep.n
    dist.all_gather_object(allr, mine, group=ep.group)
    out = {}
    for n, c in cols.items():
        ranges = [r[n] for r in allr if r[n][1] >= r[n][0]]
        lo = min((a for a, _ in ranges), default=0)
        hi = max((b for _, b in ranges), default=-1)
        out[n] = Column(c.kind, c.data, c.scale, c.dictionary, lo, hi)
    return out


def all_gather_tensor(ep: Endpoint, t):
    """Stack every rank's same-shape tensor: [n, *t.shape]."""
    torch = _torch()
    if ep.n == 1:
        return t.unsqueeze(0)
    import torch.distributed as dist
    # flat output: gloo requires it, NCCL accepts it
    out = torch.empty(ep.n * t.numel(), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, t.contiguous().reshape(-1), group=ep.group)
    return out.view(ep.n, *t.shape)

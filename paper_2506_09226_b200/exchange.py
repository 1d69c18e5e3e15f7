"""Hash partitioning and the exchanges (shuffle / broadcast).

Drop-in for ``shufflecast.exchange`` (`/root/reference/pkg/src/shufflecast/
exchange.py`):

* ``hash_keys`` (35-49): the reference's Fibonacci hash, ``scx_hash_keys``
  with identical u64 wraparound;
* ``hash_partition`` (52-70): ``scx_part_hist`` (warp-private histograms per
  2048-row tile + part-major scan) then ``scx_part_scatter`` (TMA-staged
  column tiles permuted into partition order in shared memory, written out
  as contiguous part runs) -- parts keep input order, exactly the
  reference's stable argsort + take;
* ``size_exchange`` (73-97): the N x N matrix of outgoing row counts;
* ``shuffle_table`` (131-174): rows land on worker hash(key) mod N, in
  source-rank order, then source order (exchange.py:161-166).
  - In-process workers (virtual ranks on one GPU, cluster.py): the
    partition kernel IS the send -- ``scx_part_scatter`` writes every row
    straight into its receiver's buffer at the receiver-side offset of this
    source (no send buffer, no copy).  The same destination-pointer kernel
    targets a peer GPU's HBM when the receive buffers are peer-mapped.
  - One process per GPU: partition into a local send buffer, then one
    all-to-all-v per column: ``scx_alltoallv`` = one NCCL group of
    send/recv behind the C-ABI (the paper's Alg. 1; csrc/comm.cu).
* ``broadcast_table`` (177-285): every worker gets the rank-ordered
  concatenation; differing dictionaries are reconciled first (union in
  rank order, codes remapped on the device, exchange.py:177-192,217-251).

Exchange metadata (schema check, per-column value ranges, the size matrix)
travels in ONE collective per exchange: a rendezvous in-process, a single
int64 all-gather across processes (no pickled objects).  Across NCCL
processes every data-plane transfer goes through libscx's NCCL entry points
(nccl.py); torch.distributed only bootstraps the job (and runs the gloo
CPU protocol tests).
"""

from __future__ import annotations

import ctypes as C
import hashlib
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .cluster import Endpoint, ProtocolError
from .nccl import allgather_bytes, comm_of
from .table import Column, ColumnTable, SchemaError, alloc, narrow_dtype, torch_dtype

_HASHABLE_KINDS = ("int64", "date32", "dict")
_MAX_META_COLS = 64


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


# ---------------------------------------------------------------------------
# partition kernels
# ---------------------------------------------------------------------------

class _Partitioner:
    """Pass 1 (counts) now, pass 2 (scatter to any destinations) later --
    between them the caller learns the sizes and places the receive buffers."""

    def __init__(self, table: ColumnTable, key_columns: list[str], n_parts: int,
                 fetch: bool = True):
        if n_parts < 1:
            raise ValueError("n_parts must be >= 1")
        if n_parts > 64:
            raise SchemaError(f"hash partitioning supports at most 64 parts, got {n_parts}")
        self.table = table.materialize()
        self.n_parts = n_parts
        self.names = self.table.column_names
        self.n = self.table.row_count
        keys = _key_cols(self.table, key_columns)
        self.karr = (L.Column_ * len(keys))(*[c.scx() for c in keys])
        self.n_keys = len(keys)
        self.ws = alloc(max(16, L.load().scx_part_workspace(self.n, n_parts)), np.uint8)
        self._cnt = alloc(n_parts, np.uint64)
        L.call("scx_part_hist", self.karr, self.n_keys, self.n, n_parts,
               C.c_void_p(self.ws.data_ptr()), C.c_void_p(self._cnt.data_ptr()), _stream())
        self.counts = None
        if fetch:
            self.fetch_counts()

    def fetch_counts(self) -> np.ndarray:
        """Per-part row totals to the host (waits for pass 1)."""
        if self.counts is None:
            self.counts = self._cnt.cpu().numpy().astype(np.int64)
        return self.counts

    def scatter(self, dst_addr: np.ndarray) -> None:
        """dst_addr[c, p]: device byte address of column c's part-p run."""
        cols = [self.table.column(nm) for nm in self.names]
        if not cols or self.n == 0:
            return
        arr = (L.Column_ * len(cols))(*[c.scx() for c in cols])
        dst = _torch().from_numpy(np.ascontiguousarray(dst_addr, dtype=np.uint64).reshape(-1)
                                  .view(np.int64)).to(cols[0].data.device)
        L.call("scx_part_scatter", self.karr, self.n_keys, arr, len(cols), self.n, self.n_parts,
               C.c_void_p(dst.data_ptr()), C.c_void_p(self.ws.data_ptr()), _stream())
        self._keep = dst     # the launch reads it asynchronously

    def local(self, cols: dict[str, Column]) -> list:
        """Every column partitioned into one local buffer, parts in bucket
        order (the send buffer of an all-to-all-v)."""
        bufs = [_alloc_like(cols[nm], self.n) for nm in self.names]
        base = np.concatenate([[0], np.cumsum(self.counts)[:-1]])
        self.scatter(np.array([[bufs[c].data_ptr() + int(base[d]) * cols[nm].itemsize
                                for d in range(self.n_parts)] for c, nm in enumerate(self.names)],
                              np.uint64))
        return bufs


def _alloc_like(c: Column, n: int, np_dtype=None):
    """n rows of c's dtype on c's device (CPU tensors in the gloo tests)."""
    dt = np_dtype or c.np_dtype
    if c.data.is_cuda:
        return alloc(n, dt)
    return _torch().empty(n, dtype=torch_dtype(np.dtype(dt)))


def partition_device(table: ColumnTable, key_columns: list[str], n_parts: int):
    """Partitioned copy of every column in one contiguous buffer per column
    (parts in bucket order) + per-part row counts (host ints)."""
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
    """Split into n_parts by hash mod n_parts, input order kept (exchange.py:59-70).
    Every part's columns are their own (aligned) buffers: the scatter writes
    each part run straight into its buffer."""
    P = _Partitioner(table, key_columns, n_parts)
    bufs = [[alloc(int(P.counts[p]), P.table.column(nm).np_dtype) for p in range(n_parts)]
            for nm in P.names]
    P.scatter(np.array([[b.data_ptr() for b in row] for row in bufs], dtype=np.uint64)
              .reshape(len(P.names), n_parts))
    return [ColumnTable({nm: P.table.column(nm).like(bufs[c][p]) for c, nm in enumerate(P.names)})
            for p in range(n_parts)]


# ---------------------------------------------------------------------------
# exchange metadata: one collective per exchange
# ---------------------------------------------------------------------------

def _schema(table: ColumnTable) -> tuple:
    return tuple((nm, c.kind) for nm, c in table.columns.items())


def _schema_hash(sig: tuple) -> int:
    return int.from_bytes(hashlib.blake2b(repr(sig).encode(), digest_size=8).digest(), "little") >> 1


def _col_meta(c: Column) -> tuple:
    return (int(c.scale), int(c.lo), int(c.hi), int(np.dtype(c.np_dtype).kind == "u"),
            int(c.scx_dtype))


def _exchange_meta(ep: Endpoint, table: ColumnTable, label: str, row=None, dicts: bool = False):
    """All workers' (schema, per-column (scale, lo, hi, unsigned), size row
    [, dictionaries]) in rank order; SchemaError when the schemas differ."""
    sig = _schema(table)
    metas = [_col_meta(table.column(nm)) for nm in table.column_names]
    row = np.zeros(ep.n, np.int64) if row is None else np.asarray(row, np.int64)
    dd = {nm: c.dictionary for nm, c in table.columns.items() if c.kind == "dict"} if dicts else None
    if ep.n == 1:
        slots = [(sig, metas, row, dd)]
    elif ep.in_process:
        slots = ep.cluster.rendezvous(ep.rank, label, (sig, metas, row, dd), lambda s: list(s))
    else:
        slots = _dist_meta(ep, sig, metas, row, table, dicts)
    if len({s[0] for s in slots}) > 1:
        raise SchemaError(f"{label}: schema mismatch across workers")
    return slots


def _dist_meta(ep: Endpoint, sig, metas, row, table, dicts):
    """One int64 all-gather: [schema hash, ncols, size row (N), 5 per column,
    dictionary hashes]; dictionaries themselves travel only if they differ."""
    torch = _torch()
    import torch.distributed as dist
    if len(metas) > _MAX_META_COLS:
        raise SchemaError(f"exchange of more than {_MAX_META_COLS} columns")
    names = table.column_names
    width = 2 + ep.n + 5 * _MAX_META_COLS + _MAX_META_COLS
    v = np.zeros(width, np.int64)
    v[0], v[1] = _schema_hash(sig), len(metas)
    v[2:2 + ep.n] = row
    m = np.asarray(metas, np.int64).reshape(-1)
    v[2 + ep.n:2 + ep.n + len(m)] = m
    dh = 2 + ep.n + 5 * _MAX_META_COLS
    for i, nm in enumerate(names):
        d = table.column(nm).dictionary
        if d is not None:
            v[dh + i] = _schema_hash(d)
    allv = allgather_bytes(ep, v).view(np.int64).reshape(ep.n, width)
    if len({int(r[0]) for r in allv}) > 1:
        raise SchemaError("exchange: schema mismatch across workers")
    slots = []
    for r in allv:
        k = int(r[1])
        mm = [tuple(int(x) for x in r[2 + ep.n + 5 * i:2 + ep.n + 5 * i + 5]) for i in range(k)]
        slots.append((sig, mm, r[2:2 + ep.n].copy(), None))
    if dicts and any(len({int(r[dh + i]) for r in allv}) > 1 for i in range(len(names))):
        mine = {nm: c.dictionary for nm, c in table.columns.items() if c.kind == "dict"}
        every = [None] * ep.n
        dist.all_gather_object(every, mine, group=ep.group)   # rare: dictionaries differ
        slots = [(s[0], s[1], s[2], every[i]) for i, s in enumerate(slots)]
    elif dicts:
        mine = {nm: c.dictionary for nm, c in table.columns.items() if c.kind == "dict"}
        slots = [(s[0], s[1], s[2], mine) for s in slots]
    return slots


def _unified(table: ColumnTable, slots) -> dict[str, Column]:
    """Every worker's columns brought to one physical layout: the largest
    decimal scale and a dtype wide enough for the union of all workers'
    ranges (cast on the device only where this worker's differs)."""
    out = {}
    for i, nm in enumerate(table.column_names):
        c = table.column(nm)
        ms = [s[1][i] for s in slots]
        scale = max(m[0] for m in ms)
        if any(m[0] < 0 for m in ms) and scale >= 0:
            raise SchemaError(f"column {nm!r}: raw float64 and fixed-point parts do not mix")
        mult = [10 ** (scale - m[0]) if scale >= 0 else 1 for m in ms]
        rng = [(m[1] * k, m[2] * k) for m, k in zip(ms, mult) if m[2] >= m[1]]
        lo = min((a for a, _ in rng), default=0)
        hi = max((b for _, b in rng), default=-1)
        if scale < 0 or len({(m[0], m[4]) for m in ms}) == 1:
            # every worker already stores it alike (the normal case): no cast
            out[nm] = Column(c.kind, c.data, c.scale, c.dictionary, lo, hi)
            continue
        dt = narrow_dtype(min(lo, 0) if hi < lo else lo, max(hi, 0),
                          unsigned=all(m[3] for m in ms))
        data = c.data
        if np.dtype(c.np_dtype) != dt or scale != c.scale:
            data = data.to(torch_dtype(dt))
            if scale != c.scale:
                data = data * (10 ** (scale - c.scale))
        out[nm] = Column(c.kind, data, scale, c.dictionary, lo, hi)
    return out


def _reconcile_dicts(ep: Endpoint, cols: dict[str, Column], slots) -> dict[str, Column]:
    """Union of differing dictionaries in rank order, first seen wins; this
    worker's codes go through its remap (exchange.py:177-192, 217-251)."""
    torch = _torch()
    out = dict(cols)
    for nm, c in cols.items():
        if c.kind != "dict":
            continue
        dicts = [s[3][nm] for s in slots]
        if len(set(dicts)) == 1:
            continue
        union, index, remaps = [], {}, []
        for d in dicts:
            rm = np.empty(len(d), np.int32)
            for i, sv in enumerate(d):
                code = index.get(sv)
                if code is None:
                    code = index[sv] = len(union)
                    union.append(sv)
                rm[i] = code
            remaps.append(rm)
        dt = narrow_dtype(0, max(len(union) - 1, 0))
        n = c.row_count
        new = alloc(n, dt)
        lut = torch.from_numpy(remaps[ep.rank]).to(c.data.device)
        bad = torch.zeros(1, dtype=torch.int32, device=c.data.device)
        L.call("scx_remap_codes", c.scx(), n, C.c_void_p(lut.data_ptr()), len(remaps[ep.rank]),
               L.Column_(new.data_ptr(), Column(c.kind, new, 0, union).scx_dtype, 0),
               C.c_void_p(bad.data_ptr()), _stream())
        if n and int(bad.item()):
            raise SchemaError(f"column {nm!r}: code outside its dictionary")
        out[nm] = Column("dict", new, 0, tuple(union), 0, len(union) - 1)
    return out


def size_exchange(ep: Endpoint, my_row) -> tuple[np.ndarray, np.ndarray]:
    """This worker's column of the N x N size matrix (row r = what worker r
    sends) + exclusive offsets (exchange.py:73-97)."""
    row = np.asarray(my_row, dtype=np.int64)
    if row.shape != (ep.n,):
        raise ProtocolError(f"size exchange shape mismatch at rank {ep.rank}: "
                            f"{row.shape} for a {ep.n}-worker cluster")
    if ep.n == 1:
        incoming = row.copy()
    elif ep.in_process:
        M = ep.cluster.rendezvous(ep.rank, "size_exchange", row, lambda s: np.stack(s))
        incoming = M[:, ep.rank].copy()
    else:
        incoming = allgather_bytes(ep, row).view(np.int64).reshape(ep.n, ep.n)[:, ep.rank].copy()
    offsets = np.zeros(len(incoming), dtype=np.int64)
    np.cumsum(incoming[:-1], out=offsets[1:])
    return incoming, offsets


def alltoallv(ep: Endpoint, send, send_counts, recv_counts):
    """One variable-size all-to-all of a 1-D tensor (process-per-GPU jobs):
    parts of `send` in destination order -> output in source-rank order."""
    torch = _torch()
    total = int(sum(recv_counts))
    dt = np.dtype(str(send.dtype).replace("torch.", ""))
    out = alloc(total, dt) if send.is_cuda else torch.empty(total, dtype=send.dtype)
    if ep.n == 1:
        if total:
            out.copy_(send[:total])
        return out
    c = comm_of(ep)
    if c is not None:                 # NCCL through the C-ABI: one group of send/recv
        so = np.concatenate([[0], np.cumsum(send_counts)[:-1]])
        ro = np.concatenate([[0], np.cumsum(recv_counts)[:-1]])
        c.alltoallv(send, send_counts, so, out, recv_counts, ro, send.element_size())
        return out
    import torch.distributed as dist  # gloo (CPU protocol tests)
    dist.all_to_all_single(out, send, [int(x) for x in recv_counts],
                           [int(x) for x in send_counts], group=ep.group)
    return out


# ---------------------------------------------------------------------------
# shuffle
# ---------------------------------------------------------------------------

def shuffle_table(ep: Endpoint, table, key_columns: list[str],
                  stats: ExchangeStats | None = None) -> ColumnTable:
    """Rows land on worker hash(key) mod N, received in source-rank order,
    source order within a source (exchange.py:131-174)."""
    table = table.materialize()
    n = ep.n
    if n == 1:
        _key_cols(table, key_columns)
        out = table
    else:
        P = _Partitioner(table, key_columns, n)
        slots = _exchange_meta(ep, table, "shuffle", P.counts)
        cols = _unified(table, slots)
        if any(cols[nm].data is not table.column(nm).data for nm in cols):
            P = _Partitioner(ColumnTable(cols), key_columns, n)   # re-typed columns
        M = np.stack([s[2] for s in slots])          # M[s, d]: rows s sends to d
        if ep.in_process:
            out = _shuffle_direct(ep, P, cols, M)
        else:
            out = _shuffle_alltoall(ep, P, cols, M)
    if stats is not None:
        counts = P.counts if n > 1 else np.asarray([table.row_count])
        for nm in table.column_names:
            c = table.column(nm)
            stats.messages.extend(int(counts[d]) * c.itemsize for d in range(n)
                                  if d != ep.rank and counts[d] > 0)
            stats.table_bytes += c.nbytes
    return out


def _shuffle_direct(ep: Endpoint, P: _Partitioner, cols: dict[str, Column], M) -> ColumnTable:
    """In-process: allocate this worker's receive buffers, publish their
    addresses, and let every source's scatter kernel write into them."""
    names = P.names
    total = int(M[:, ep.rank].sum())
    recv = [alloc(total, cols[nm].np_dtype) for nm in names]
    addrs = ep.cluster.rendezvous(ep.rank, "shuffle:buffers",
                                  [b.data_ptr() for b in recv], lambda s: list(s))
    # column c of receiver d: this source's rows start after sources < rank
    before = M[:ep.rank, :].sum(axis=0)              # per destination
    dst = np.zeros((len(names), ep.n), np.uint64)
    for c, nm in enumerate(names):
        w = cols[nm].itemsize
        for d in range(ep.n):
            dst[c, d] = addrs[d][c] + int(before[d]) * w
    P.scatter(dst)
    # every source's scatter is enqueued (one shared stream) before anyone
    # reads its receive buffers or frees a source table
    ep.cluster.rendezvous(ep.rank, "shuffle:done", None, lambda s: None)
    return ColumnTable({nm: cols[nm].like(recv[c]) for c, nm in enumerate(names)})


def _shuffle_alltoall(ep: Endpoint, P: _Partitioner, cols: dict[str, Column], M) -> ColumnTable:
    names = P.names
    local = P.local(cols)
    out = {}
    for c, nm in enumerate(names):
        out[nm] = cols[nm].like(alltoallv(ep, local[c], M[ep.rank, :], M[:, ep.rank]))
    return ColumnTable(out)


# ---------------------------------------------------------------------------
# broadcast
# ---------------------------------------------------------------------------

def broadcast_table(ep: Endpoint, table, stats: ExchangeStats | None = None,
                    use_p2p: bool = False) -> ColumnTable:
    """Every worker gets the rank-ordered concatenation of all workers'
    tables (exchange.py:195-285)."""
    table = table.materialize()
    n = ep.n
    names = table.column_names
    if n == 1:
        cols = dict(table.columns)
        counts = np.asarray([table.row_count])
    else:
        slots = _exchange_meta(ep, table, "broadcast",
                               np.full(n, table.row_count, np.int64), dicts=True)
        counts = np.asarray([int(s[2][0]) for s in slots])
        cols = _reconcile_dicts(ep, _unified(table, slots), slots)
        offs = np.concatenate([[0], np.cumsum(counts)])
        total = int(offs[-1])
        outs = {nm: _alloc_like(cols[nm], total) for nm in names}
        if ep.in_process:
            peers = ep.cluster.rendezvous(ep.rank, "broadcast:data",
                                          {nm: cols[nm].data for nm in names}, lambda s: list(s))
            for nm in names:
                for r in range(n):
                    if counts[r]:
                        outs[nm][offs[r]:offs[r + 1]].copy_(peers[r][nm])
            ep.cluster.rendezvous(ep.rank, "broadcast:done", None, lambda s: None)
        elif comm_of(ep) is not None:
            c = comm_of(ep)
            for nm in names:
                src = cols[nm].data.contiguous()
                w = cols[nm].itemsize
                outs[nm][offs[ep.rank]:offs[ep.rank + 1]].copy_(src)
                if use_p2p:   # N-1 sends of this rank's rows + N-1 receives, one group
                    sc = [0 if d == ep.rank else int(counts[ep.rank]) for d in range(n)]
                    rc = [0 if r == ep.rank else int(counts[r]) for r in range(n)]
                    c.alltoallv(src, sc, [0] * n, outs[nm], rc, offs[:-1], w)
                else:         # the N root broadcasts of the column in ONE group (Alg. 2)
                    c.bcast_group([outs[nm][offs[r]:offs[r + 1]] if counts[r] else None
                                   for r in range(n)], [int(counts[r]) * w for r in range(n)])
        else:
            import torch.distributed as dist
            for nm in names:
                src = cols[nm].data.contiguous()
                outs[nm][offs[ep.rank]:offs[ep.rank + 1]].copy_(src)
                if use_p2p:
                    ops = []
                    for peer in range(n):
                        if peer == ep.rank:
                            continue
                        if counts[ep.rank]:
                            ops.append(dist.P2POp(dist.isend, src, peer, group=ep.group))
                        if counts[peer]:
                            ops.append(dist.P2POp(dist.irecv, outs[nm][offs[peer]:offs[peer + 1]],
                                                  peer, group=ep.group))
                    if ops:
                        for w in dist.batch_isend_irecv(ops):
                            w.wait()
                else:
                    for root in range(n):      # N root broadcasts per column (Alg. 2)
                        if counts[root]:
                            dist.broadcast(outs[nm][offs[root]:offs[root + 1]], src=root,
                                           group=ep.group)
        cols = {nm: cols[nm].like(outs[nm]) for nm in names}
    if stats is not None:
        for nm in names:
            c = table.column(nm)
            if c.nbytes > 0:
                copies = (n - 1) if use_p2p else (1 if n > 1 else 0)
                stats.messages.extend([c.nbytes] * copies)
            stats.table_bytes += c.nbytes
    return ColumnTable(cols)


def all_gather_tensor(ep: Endpoint, t):
    """Stack every worker's same-shape tensor: [n, *t.shape]."""
    torch = _torch()
    if ep.n == 1:
        return t.unsqueeze(0)
    if ep.in_process:
        parts = ep.cluster.rendezvous(ep.rank, "all_gather_tensor", t, lambda s: list(s))
        if len({tuple(p.shape) for p in parts}) > 1:
            raise ProtocolError("all_gather_tensor: shape mismatch across workers")
        out = torch.stack(parts)
        ep.cluster.rendezvous(ep.rank, "all_gather_tensor:done", None, lambda s: None)
        return out
    c = comm_of(ep)
    if c is not None:
        return c.allgather(t.contiguous().reshape(-1)).view(ep.n, *t.shape)
    import torch.distributed as dist
    # flat output: gloo requires it
    out = torch.empty(ep.n * t.numel(), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, t.contiguous().reshape(-1), group=ep.group)
    return out.view(ep.n, *t.shape)

"""SPMD executor over HBM-resident partitions: context, plans, reports.

Drop-in for ``shufflecast.engine`` (`/root/reference/pkg/src/shufflecast/
engine.py`): the exchange-plan registry (41-133), ``RunReport`` (144-179),
``result_digest`` (182-197), the driver-facing context protocol
(``LocalContext``/``WorkerContext``, 221-365), ``run_query`` (382-460) and
``reference_run`` (463-469).

Workers: one process per GPU (torchrun, NCCL exchanges), or -- the
reference's own ``MODE_IN_PROCESS`` -- N worker threads in one process,
each a virtual rank whose partition lives in the same GPU's HBM
(``run_query(qid, variant, cluster, dataset)``, cluster.py).  Tables live in
HBM and relational operators are fused kernels either way.  Timing follows
the reference's barrier method (engine.py:318-340): every exchange is
bracketed by a barrier (device-drained across processes), compute is the
remainder.
"""

from __future__ import annotations

import hashlib
import json
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import exchange as X
from . import relops as R
from .cluster import Cluster, Endpoint, barrier, create_cluster, run_workers
from .data import (DEFAULT_PARTITION_KEYS, Dataset, PARTITION_SCHEMES, DataError,
                   PartitionedDataset)
from .table import Column, ColumnTable, alloc, concat_tables


class PlanError(ValueError):
    """Unsupported query/variant or a plan-vs-partitioning mismatch (engine.py:37)."""


@dataclass(frozen=True)
class ExchangePlan:
    """Declarative plan shape (engine.py:41-72)."""

    query_id: str
    variant: str
    steps: tuple[str, ...]
    expected_exchanges: tuple[int, int]
    requires_co_partition: tuple[tuple[str, str], ...] = ()

    def validate(self) -> None:
        if self.steps.count("final_gather") != 1 or self.steps[-1] != "final_gather":
            raise PlanError(f"{self.query_id}/{self.variant}: need exactly one final_gather, last")
        for step in self.steps:
            if step.startswith("local_hash_join:"):
                prep = step.split(":", 1)[1]
                if prep not in ("co_partitioned", "shuffle", "broadcast"):
                    raise PlanError(f"{self.query_id}: join without a valid alignment: {prep}")
                if prep == "co_partitioned" and not self.requires_co_partition:
                    raise PlanError(f"{self.query_id}/{self.variant}: co-partitioned join must "
                                    "state its partitioning requirement")


EXCHANGE_PLANS: dict[tuple[str, str], ExchangePlan] = {}

_CO_LO = (("lineitem", "l_orderkey"), ("orders", "o_orderkey"))


def _register(qid, variant, steps, expected, co=()):
    p = ExchangePlan(qid, variant, tuple(steps), expected, tuple(co))
    p.validate()
    EXCHANGE_PLANS[(qid, variant)] = p


# engine.py:83-133 (same shapes and Table-4 counts)
_register("Q1", "default", ["scan:lineitem", "filter", "group_aggregate", "final_gather"], (0, 0))
_register("Q3", "default", ["scan:customer", "filter", "broadcast:customer", "scan:orders",
                            "filter", "local_hash_join:broadcast", "scan:lineitem", "filter",
                            "local_hash_join:co_partitioned", "group_aggregate", "final_gather"],
          (0, 1), _CO_LO)
_register("Q6", "default", ["scan:lineitem", "filter", "group_aggregate", "final_gather"], (0, 0))
_register("Q12", "default", ["scan:lineitem", "filter", "scan:orders",
                             "local_hash_join:co_partitioned", "group_aggregate", "final_gather"],
          (0, 0), _CO_LO)
_register("Q12", "pa", ["scan:lineitem", "filter", "shuffle:l_orderkey", "scan:orders",
                        "shuffle:o_orderkey", "local_hash_join:shuffle", "group_aggregate",
                        "final_gather"], (2, 0))
_register("Q12", "pb", ["scan:lineitem", "filter", "broadcast:lineitem", "scan:orders",
                        "local_hash_join:broadcast", "group_aggregate", "final_gather"], (0, 1))
_register("Q14", "default", ["scan:lineitem", "filter", "shuffle:l_partkey", "scan:part",
                             "local_hash_join:shuffle", "group_aggregate", "final_gather"],
          (1, 0), (("part", "p_partkey"),))
_register("Q19", "default", ["scan:part", "filter", "broadcast:part", "scan:lineitem", "filter",
                             "local_hash_join:broadcast", "filter", "group_aggregate",
                             "final_gather"], (0, 1))


# The 16 queries the reference lacks (queries.py q2..q22).  Counts are what
# these plans execute; nation / region are replicated on every rank
# (data.REPLICATED_TABLES), so like the paper's Table 4
# they cost no exchange.  13 of 16 equal Table 4; Q11, Q13 and Q18 differ
# (DESIGN.md §4 says why per query).
_CO_PS = (("partsupp", "ps_partkey"), ("part", "p_partkey"))
_CO_C = (("customer", "c_custkey"),)
_CO_S = (("supplier", "s_suppkey"),)
for _qid, _steps, _counts, _co in [
    ("Q2", ["broadcast:supplier", "local_hash_join:broadcast", "local_hash_join:co_partitioned"],
     (0, 1), _CO_PS),
    ("Q4", ["local_hash_join:co_partitioned"], (0, 0), _CO_LO),
    ("Q5", ["broadcast:customer", "broadcast:supplier", "local_hash_join:co_partitioned"], (0, 2),
     _CO_LO),
    ("Q7", ["broadcast:supplier", "broadcast:customer", "local_hash_join:co_partitioned"], (0, 2),
     _CO_LO),
    ("Q8", ["broadcast:customer", "broadcast:part", "broadcast:supplier",
            "local_hash_join:co_partitioned"], (0, 3), _CO_LO),
    ("Q9", ["broadcast:part", "broadcast:supplier", "local_hash_join:co_partitioned",
            "shuffle:l_partkey", "local_hash_join:shuffle"], (1, 2), _CO_LO + _CO_PS),
    ("Q10", ["local_hash_join:co_partitioned", "shuffle:o_custkey", "local_hash_join:shuffle"],
     (1, 0), _CO_LO + _CO_C),
    ("Q11", ["broadcast:supplier", "local_hash_join:broadcast"], (0, 1), ()),
    ("Q13", ["shuffle:o_custkey", "local_hash_join:shuffle"], (1, 0), _CO_C),
    ("Q15", ["shuffle:l_suppkey", "local_hash_join:shuffle"], (1, 0), _CO_S),
    ("Q16", ["broadcast:supplier", "local_hash_join:co_partitioned", "shuffle:p_brand"], (1, 1),
     _CO_PS),
    ("Q17", ["broadcast:part", "local_hash_join:broadcast", "shuffle:l_partkey"], (1, 1), ()),
    ("Q18", ["local_hash_join:co_partitioned"], (0, 0), _CO_LO),
    ("Q20", ["shuffle:l_partkey", "local_hash_join:shuffle", "broadcast:partsupp"], (1, 1),
     _CO_PS),
    ("Q21", ["broadcast:supplier", "local_hash_join:co_partitioned"], (0, 1), _CO_LO),
    ("Q22", ["shuffle:o_custkey", "local_hash_join:shuffle"], (1, 0), _CO_C),
]:
    _register(_qid, "default", ["scan"] + _steps + ["group_aggregate", "final_gather"], _counts,
              _co)


def get_plan(qid: str, variant: str) -> ExchangePlan:
    plan = EXCHANGE_PLANS.get((qid, variant))
    if plan is None:
        known = sorted({q for q, _ in EXCHANGE_PLANS})
        raise PlanError(f"no plan for query {qid!r} variant {variant!r}; queries: {known}")
    return plan


@dataclass
class RunReport:
    """Per-query instrumentation (engine.py:144-179), device-timed."""

    query_id: str
    variant: str
    mode: str
    compute_s: float
    shuffle_s: float
    broadcast_s: float
    shuffle_msgs: list[int]
    broadcast_msgs: list[int]
    peak_bytes: list[int]
    result_digest: str
    exchange_counts: tuple[int, int]
    shuffle_bytes: int = 0
    broadcast_bytes: int = 0

    @property
    def total_s(self) -> float:
        return self.compute_s + self.shuffle_s + self.broadcast_s

    def to_json(self) -> str:
        return json.dumps({
            "compute_s": self.compute_s, "shuffle_s": self.shuffle_s,
            "broadcast_s": self.broadcast_s, "shuffle_msgs": self.shuffle_msgs,
            "broadcast_msgs": self.broadcast_msgs, "peak_bytes": self.peak_bytes,
            "result_digest": self.result_digest, "exchange_counts": list(self.exchange_counts),
        }, indent=2)


def result_digest(table) -> str:
    """Order-insensitive sha256 of result rows, floats at 9 significant digits
    (engine.py:182-197).  Not N-stable for float queries."""
    if table is None:
        return "empty"
    return hashlib.sha256("\n".join(digest_lines(table)).encode()).hexdigest()


def digest_lines(table) -> list[str]:
    """The lines result_digest hashes: the header, then the sorted rows."""
    table = table.materialize()
    decoded = [table.column(n).decoded() for n in table.column_names]
    kinds = [table.column(n).kind for n in table.column_names]
    lines = []
    for i in range(table.row_count):
        lines.append("|".join(f"{col[i]:.9e}" if k == "float64" else str(col[i])
                              for col, k in zip(decoded, kinds)))
    lines.sort()
    return [",".join(table.column_names)] + lines


# ---------------------------------------------------------------------------
# the context protocol used by query drivers
# ---------------------------------------------------------------------------

class DeviceContext:
    """One rank's view: its HBM partition, fused relops, NCCL exchanges.

    With ``ep.n == 1`` exchanges are the identity, which makes this the
    single-context execution (``LocalContext``, engine.py:221-258) as well.
    """

    def __init__(self, ep: Endpoint, tables: dict[str, ColumnTable], variant: str = "default",
                 scheme: str = "default_keys", p2p_broadcast: bool = False,
                 timed: bool = True, ready: dict | None = None):
        self.ep = ep
        self.tables = tables
        # table name -> CUDA event of its (asynchronous) upload: the first
        # access makes this stream wait for it (upload_tables_async)
        self.ready = ready
        self._waited: set = set()
        self.variant = variant
        self.scheme = scheme
        self.p2p_broadcast = p2p_broadcast
        self.timed = timed
        self.shuffle_s = 0.0
        self.broadcast_s = 0.0
        self.shuffle_msgs: list[int] = []
        self.broadcast_msgs: list[int] = []
        self.shuffle_bytes = 0
        self.broadcast_bytes = 0
        self.n_shuffles = 0
        self.n_broadcasts = 0

    @property
    def is_root(self) -> bool:
        return self.ep.rank == 0

    def table(self, name: str) -> ColumnTable:
        # the query's stream waits for the table's upload events once per
        # context (the dict is shared by concurrent queries: never consumed)
        if self.ready is not None and name in self.ready and name not in self._waited \
                and not getattr(self.tables.get(name), "column_ready", False):
            import torch
            evs = self.ready[name]
            for ev in (evs if isinstance(evs, (list, tuple)) else [evs]):
                torch.cuda.current_stream().wait_event(ev)
            self._waited.add(name)
        return self.tables[name]

    def filter(self, t, mask):
        return R.filter_table(t, mask)

    def join(self, left, right, on, how="inner"):
        return R.local_hash_join(left, right, on, how)

    def group(self, t, keys, aggs, sort: bool = True, having: tuple | None = None):
        """group_aggregate; ``sort=False`` (an extension) skips the key-order
        sort for intermediates that feed a join or a re-aggregation, and
        ``having=(name, lo, hi)`` keeps groups with lo <= name <= hi (rank-local:
        the groups must be complete on this rank)."""
        return R.group_aggregate(t, keys, aggs, sort=sort, having=having)

    def add_column(self, t, name, col):
        return R.as_view(t).with_column(name, col)

    def require_co_partitioned(self, *tables) -> None:
        if self.ep.n > 1 and self.scheme != "default_keys":
            raise PlanError(f"plan needs co-partitioned {tables}, but data is partitioned "
                            f"as {self.scheme!r}")

    def _bracket(self):
        if self.timed:
            barrier(self.ep)
        return time.perf_counter()

    def shuffle(self, t, keys):
        t0 = self._bracket()
        stats = X.ExchangeStats()
        out = X.shuffle_table(self.ep, t, keys, stats) if self.ep.n > 1 else t
        self.shuffle_s += self._bracket() - t0
        self.shuffle_msgs.extend(stats.messages)
        self.shuffle_bytes += stats.table_bytes
        self.n_shuffles += 1
        return out

    def broadcast(self, t):
        t0 = self._bracket()
        stats = X.ExchangeStats()
        out = (X.broadcast_table(self.ep, t, stats, use_p2p=self.p2p_broadcast)
               if self.ep.n > 1 else t)
        self.broadcast_s += self._bracket() - t0
        self.broadcast_msgs.extend(stats.messages)
        self.broadcast_bytes += stats.table_bytes
        self.n_broadcasts += 1
        return out

    def global_group(self, t, keys, aggs):
        """Group + exact cross-rank final aggregation; result on the root.

        The reference does this with a float64 ``all_reduce_sum`` of the
        numpy grid (queries.py:51-54, 116); here the per-rank partials are
        exact 128-bit integers and are summed exactly (all-gather + exact
        fold), so the result is rank-count independent.
        """
        g = R.group_aggregate(t, keys, aggs, cross=self)
        return g if self.is_root else None

    def global_group_all(self, t, keys, aggs):
        """global_group with the (dense, small-domain) result on every rank."""
        g = R.group_aggregate(t, keys, aggs, cross=self)
        if g is None:
            raise PlanError("global_group_all needs a dense (small key domain) aggregate")
        return g

    def all_reduce_sum(self, vec) -> np.ndarray:
        """float64 sum over workers, folded in rank order (engine.py:342-343,
        collectives.py:198-206)."""
        from .collectives import all_reduce
        return all_reduce(self.ep, np.asarray(vec, dtype=np.float64), "sum")

    def gather(self, t):
        """Partials to rank 0, rank order (engine.py:345-365)."""
        t = t.materialize()
        if self.ep.n == 1:
            return t
        if self.ep.in_process:
            parts = self.ep.cluster.rendezvous(self.ep.rank, "gather", t, lambda s: list(s))
            full = concat_tables(parts) if self.is_root else None
            # the root's concatenation copies are enqueued before any worker
            # drops its partial (one shared stream)
            self.ep.cluster.rendezvous(self.ep.rank, "gather:done", None, lambda s: None)
            return full
        names = t.column_names
        counts, _ = X.size_exchange(self.ep, np.full(self.ep.n, t.row_count, dtype=np.int64))
        from .nccl import comm_of
        c = comm_of(self.ep)
        if c is not None:             # NCCL through the C-ABI (scx_gather_to0)
            parts_cols = [dict() for _ in range(self.ep.n)]
            for name in names:
                ref = t.column(name)
                src = ref.data.contiguous()
                if self.is_root:
                    bufs = [R.alloc(int(counts[r]), ref.np_dtype) for r in range(self.ep.n)]
                    c.gather_to0(src, src.numel() * src.element_size(), bufs,
                                 [int(counts[r]) * ref.itemsize for r in range(self.ep.n)])
                    for r in range(self.ep.n):
                        parts_cols[r][name] = t.column(name) if r == 0 else ref.like(bufs[r])
                else:
                    c.gather_to0(src, src.numel() * src.element_size())
            if not self.is_root:
                return None
            return concat_tables([t] + [ColumnTable(pc) for pc in parts_cols[1:]])
        import torch.distributed as dist
        parts = [t] if self.is_root else []
        if self.is_root:
            for src in range(1, self.ep.n):
                cols = {}
                for name in names:
                    ref = t.column(name)
                    buf = R.alloc(int(counts[src]), ref.np_dtype, ref.data.device)
                    if counts[src]:
                        dist.recv(buf, src=src)
                    cols[name] = ref.like(buf)
                parts.append(ColumnTable(cols))
            return concat_tables(parts)
        for name in names:
            if t.row_count:
                dist.send(t.column(name).data.contiguous(), dst=0)
        return None


# ---------------------------------------------------------------------------
# data placement
# ---------------------------------------------------------------------------

def reserve_device_pool(nbytes: int) -> int:
    """Grow the caching allocator's pool by one segment of `nbytes` up front
    (allocate + free): later intermediates are carved from it instead of
    cudaMalloc'ing new multi-GB segments mid-query (a 25-30 ms stall seen
    once in a timed pass).  Returns the bytes reserved (0 if it did not fit)."""
    import torch
    free, _ = torch.cuda.mem_get_info()
    nbytes = min(int(nbytes), max(0, free - (8 << 30)))
    if nbytes <= 0:
        return 0
    blk = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    del blk
    return nbytes


_COPY_STREAMS: dict = {}


def upload_tables_async(host: dict, order=None, stream=None):
    """Upload pinned host columns in `order` on a copy stream (their unpack
    kernels on a second, high-priority stream) without blocking the compute
    stream.

    ``host``: {table: {column: (HostColumn, pinned torch tensor or
    codec.PinnedPacked)}} (codec.pin_tables).  ``order``: table names (each
    table's columns in host order) or ``(table, column)`` pairs -- first use
    first; whatever it leaves out follows in host order.  Every column gets
    the CUDA event of its own copy (``Column.set_ready``): the first stream
    that reads a column waits for that event only, so a query starts as soon
    as the columns it touches have crossed PCIe while the rest are still in
    flight (H2D overlapped with the queries that can already run).  Returns
    (device tables, {table: [its column events]}); ``DeviceContext(ready=...)``
    takes the dict (tables marked ``column_ready`` need no table-level wait).
    Single-rank tables only.
    """
    import torch
    from .codec import FKDIFF, FKIDX, PinnedPacked, scratch_bytes, upload_packed
    # SCX_UPLOAD_STREAMS=1 (default): one copy stream lands the columns
    # strictly in `order` at full PCIe rate, their unpack kernels run on a
    # separate high-priority stream (the next copy never waits for an unpack,
    # and an unpack is scheduled ahead of the queries' pending CTAs).  =2: two
    # copy streams, columns alternating, each unpacked on its copy stream
    # (columns then land interleaved, out of `order`).  Kept per device.
    global _COPY_STREAMS
    dev = torch.cuda.current_device()
    if dev not in _COPY_STREAMS:
        _COPY_STREAMS[dev] = [torch.cuda.Stream(priority=-1) for _ in range(3)]
    two = os.environ.get("SCX_UPLOAD_STREAMS", "1") == "2"
    streams = [stream or _COPY_STREAMS[dev][0]] + ([_COPY_STREAMS[dev][1]] if two else [])
    unpack_stream = None if two else _COPY_STREAMS[dev][2]
    main = torch.cuda.current_stream()
    for cs in streams + ([unpack_stream] if unpack_stream is not None else []):
        cs.wait_stream(main)       # buffers below are allocated on `main`
    # one scratch arena for every packed column's words: the same size each
    # pass, so the caching allocator hands back the same block (per-column
    # scratch allocations cudaMalloc'ed / freed inside timed passes)
    total = sum(scratch_bytes(src) for cols in host.values() for _, src in cols.values()
                if isinstance(src, PinnedPacked))
    arena = alloc(max(total, 256), np.uint8)
    for cs in streams + ([unpack_stream] if unpack_stream is not None else []):
        arena.record_stream(cs)
    # the column sequence: explicit pairs / tables first, then the rest
    seq = []
    for item in (order or list(host)):
        if isinstance(item, tuple):
            if item[0] in host and item[1] in host[item[0]]:
                seq.append(item)
        elif item in host:
            seq.extend((item, c) for c in host[item])
    seen = set(seq)
    seq += [(t, c) for t in host for c in host[t] if (t, c) not in seen]
    cols = {t: {} for t in host}
    stream_of = {}
    events = {t: [] for t in host}
    aoff = 0
    k = 0

    def put(tname, cname):
        nonlocal aoff, k
        if cname in cols[tname]:
            return
        hc, pinned = host[tname][cname]
        pc = pinned.col if isinstance(pinned, PinnedPacked) else None
        fkd = pc is not None and pc.encoding in (FKDIFF, FKIDX)
        # a column-relative (DIFF) column is unpacked against its reference:
        # the reference goes first, and the diff on the reference's copy stream
        ref = pc.ref if pc is not None and not fkd else None
        if ref is not None:
            put(tname, ref)
            cs = stream_of[(tname, ref)]
        else:
            if fkd:
                # key-relative: the foreign key and the parent column first
                put(tname, pc.fk)
                put(pc.ref_table, pc.ref)
            cs = streams[k % len(streams)]
            k += 1
        stream_of[(tname, cname)] = cs
        if isinstance(pinned, PinnedPacked):
            # packed words cross PCIe, scx_unpack rebuilds the column
            nb = scratch_bytes(pinned)
            if fkd:       # the unpack reads columns that may have landed on another stream
                us = unpack_stream or cs
                for dep in (cols[tname][pc.fk], cols[pc.ref_table][pc.ref]):
                    us.wait_event(dep._ready[0])
            buf = upload_packed(pc, pinned.words, pinned.bases, cs,
                                arena[aoff:aoff + nb],
                                cols[pc.ref_table][pc.ref]._data if fkd else
                                (cols[tname][ref]._data if ref is not None else None),
                                unpack_stream=unpack_stream,
                                fk_col=cols[tname][pc.fk]._data if fkd else None)
            aoff += nb
            done_on = unpack_stream or cs
        else:
            buf = alloc(hc.row_count, hc.values.dtype)
            with torch.cuda.stream(cs):
                buf.copy_(pinned, non_blocking=True)
            done_on = cs
        col = Column(hc.kind, buf, hc.scale, hc.dictionary, hc.lo, hc.hi,
                     hc.dense and hc.row_count == hc.hi - hc.lo + 1)
        if hc.sorted:
            col.sorted = True
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(done_on)
        col.set_ready(ev)
        events[tname].append(ev)
        cols[tname][cname] = col

    for tname, cname in seq:
        put(tname, cname)
    tables = {}
    for tname in host:
        t = ColumnTable({c: cols[tname][c] for c in host[tname]})   # host column order
        t.column_ready = True
        tables[tname] = t
    return tables, events


def load_tables(ds: Dataset, ep: Endpoint | None = None, scheme: str = "default_keys",
                names=None) -> dict[str, ColumnTable]:
    """Upload this rank's partition of a host dataset into HBM.

    At N > 1 each rank selects its own rows on the host -- ``default_keys``:
    the reference's hash of the table's partition key mod N, input order
    kept (data.py:284-302, bit-identical to the device partition kernel);
    other schemes: host row ranges -- and uploads only those (1/N of every
    table crosses PCIe per rank, not the whole table).
    """
    from .data import worker_rows
    ep = ep or Endpoint(0, 1, "nccl")
    if scheme not in PARTITION_SCHEMES:
        raise DataError(f"unknown partitioning scheme {scheme!r}; choose from {PARTITION_SCHEMES}")
    out = {}
    for name, ht in ds.tables.items():
        if names is not None and name not in names:
            continue
        if ep.n == 1:
            out[name] = ht.to_device()
        else:
            rows = worker_rows(name, ht, scheme, ep.n)[ep.rank]
            out[name] = ht.to_device() if len(rows) == ht.row_count else ht.take(rows).to_device()
    return out


def partition_tables(ds, n: int, scheme: str = "default_keys", names=None) -> list[dict]:
    """Per-worker device tables for an in-process cluster of n virtual ranks
    on this GPU.  A host ``Dataset`` is uploaded once and split on the
    device by the partition kernel (``default_keys``, data.py:284-302
    semantics) or by host row ranges (other schemes); a host
    ``PartitionedDataset`` uploads each worker's share."""
    from .data import REPLICATED_TABLES, partition_rows
    if isinstance(ds, PartitionedDataset):
        if ds.n_workers != n:
            raise PlanError(f"cluster has {n} endpoints but dataset is partitioned for "
                            f"{ds.n_workers}")
        return [{t: ht.to_device() for t, ht in w.items() if names is None or t in names}
                for w in ds.workers]
    if scheme not in PARTITION_SCHEMES:
        raise DataError(f"unknown partitioning scheme {scheme!r}; choose from {PARTITION_SCHEMES}")
    out: list[dict] = [{} for _ in range(n)]
    for name, ht in ds.tables.items():
        if names is not None and name not in names:
            continue
        if name in REPLICATED_TABLES:
            dev = ht.to_device() if not isinstance(ht, ColumnTable) else ht
            parts = [dev] * n
        elif scheme == "default_keys":
            dev = ht.to_device() if not isinstance(ht, ColumnTable) else ht
            parts = X.hash_partition(dev, [DEFAULT_PARTITION_KEYS[name]], n) if n > 1 else [dev]
        else:
            parts = [ht.take(r).to_device() for r in partition_rows(ht, scheme, None, n)]
        for r in range(n):
            out[r][name] = parts[r]
    return out


@dataclass
class _WorkerOutcome:
    result: object
    total_s: float
    shuffle_s: float
    broadcast_s: float
    shuffle_msgs: list
    broadcast_msgs: list
    shuffle_bytes: int
    broadcast_bytes: int
    peak: int
    counts: tuple


def _run_worker(ep: Endpoint, fn, tables, variant, scheme, p2p_broadcast) -> _WorkerOutcome:
    import torch
    ctx = DeviceContext(ep, tables, variant, scheme, p2p_broadcast)
    barrier(ep)
    t0 = time.perf_counter()
    result = fn(ctx)
    if result is not None:
        result = result.materialize()
    barrier(ep)
    if ep.in_process:
        torch.cuda.synchronize()
    total = time.perf_counter() - t0
    return _WorkerOutcome(result, total, ctx.shuffle_s, ctx.broadcast_s, ctx.shuffle_msgs,
                          ctx.broadcast_msgs, ctx.shuffle_bytes, ctx.broadcast_bytes,
                          int(torch.cuda.max_memory_allocated()),
                          (ctx.n_shuffles, ctx.n_broadcasts))


def run_query(qid: str, variant: str = "default", cluster=None, dataset=None,
              p2p_broadcast: bool = False, *, scheme: str | None = None, tables=None):
    """Execute one query; (result on the root | None, RunReport) (engine.py:382-460).

    ``cluster``: an in-process ``Cluster`` (reference call shape:
    ``run_query(qid, variant, cluster, partitioned_dataset)``; every worker
    thread runs the plan on its virtual rank, the root's result is
    returned), or this process's ``Endpoint`` in a process-per-GPU job
    (``dataset`` = this rank's device tables), or None (one GPU, one rank).
    """
    from .queries import PLAN_FUNCTIONS
    import torch
    plan = get_plan(qid, variant)
    dataset = tables if dataset is None else dataset
    if scheme is None:
        scheme = dataset.scheme if isinstance(dataset, PartitionedDataset) else "default_keys"
    n = cluster.n if cluster is not None else 1
    if plan.requires_co_partition and scheme != "default_keys" and n > 1:
        needs = ", ".join(f"{t} on {k}" for t, k in plan.requires_co_partition)
        raise PlanError(f"{qid}/{variant} requires co-partitioned inputs ({needs}); "
                        f"got scheme {scheme!r}")
    fn = PLAN_FUNCTIONS[qid]
    torch.cuda.reset_peak_memory_stats()
    if isinstance(cluster, Cluster):
        if isinstance(dataset, (list, tuple)):
            per = list(dataset)
            if len(per) != n:
                raise PlanError(f"cluster has {n} endpoints but dataset is partitioned for "
                                f"{len(per)}")
        else:
            per = partition_tables(dataset, n, scheme)
        outcomes = run_workers(cluster, lambda ep: _run_worker(ep, fn, per[ep.rank], variant,
                                                               scheme, p2p_broadcast))
        mode = cluster.mode
    else:
        ep = cluster or Endpoint(0, 1, "nccl")
        if isinstance(dataset, Dataset):
            dataset = load_tables(dataset, ep, scheme)
        outcomes = [_run_worker(ep, fn, dataset, variant, scheme, p2p_broadcast)]
        mode = ep.backend
    root = outcomes[0]
    if any(o.counts != root.counts for o in outcomes):
        raise PlanError(f"{qid}/{variant}: workers disagree on exchange counts")
    if root.counts != plan.expected_exchanges:
        raise PlanError(f"{qid}/{variant}: plan declares exchanges {plan.expected_exchanges}, "
                        f"run produced {root.counts}")
    result = root.result
    report = RunReport(
        query_id=qid, variant=variant, mode=mode,
        compute_s=root.total_s - root.shuffle_s - root.broadcast_s, shuffle_s=root.shuffle_s,
        broadcast_s=root.broadcast_s,
        shuffle_msgs=[m for o in outcomes for m in o.shuffle_msgs],
        broadcast_msgs=[m for o in outcomes for m in o.broadcast_msgs],
        peak_bytes=[o.peak for o in outcomes],
        result_digest=result_digest(result) if result is not None else "empty",
        exchange_counts=root.counts, shuffle_bytes=sum(o.shuffle_bytes for o in outcomes),
        broadcast_bytes=sum(o.broadcast_bytes for o in outcomes))
    return result, report


def q12_variants(cluster, dataset: Dataset) -> dict[str, RunReport]:
    """Q12 under its three plans -- default (co-partitioned), Pa (shuffle
    both sides), Pb (broadcast) -- whose results must agree
    (engine.py:472-490).  The reference compares virtual times on a
    simulated cluster; here the reports carry measured times (in-process
    ``Cluster``, this process's ``Endpoint``, or None for one GPU)."""
    if isinstance(cluster, Cluster):
        by_key = partition_tables(dataset, cluster.n, "default_keys")
        by_range = partition_tables(dataset, cluster.n, "unpartitioned")
    else:
        ep = cluster or Endpoint(0, 1, "nccl")
        by_key = load_tables(dataset, ep, "default_keys")
        by_range = load_tables(dataset, ep, "unpartitioned")
    reports = {}
    _, reports["default"] = run_query("Q12", "default", cluster, by_key, scheme="default_keys")
    _, reports["pa"] = run_query("Q12", "pa", cluster, by_range, scheme="unpartitioned")
    _, reports["pb"] = run_query("Q12", "pb", cluster, by_range, scheme="unpartitioned")
    digests = {r.result_digest for r in reports.values()}
    if len(digests) != 1:
        raise PlanError(f"Q12 variants disagree: {digests}")
    return reports


def reference_run(qid: str, tables, variant: str = "default") -> ColumnTable:
    """Single-context execution over full device tables (engine.py:463-469)."""
    from .queries import PLAN_FUNCTIONS
    if qid not in PLAN_FUNCTIONS:
        from .queries import SUPPORTED_QUERIES
        raise PlanError(f"unsupported query {qid!r}; supported: {SUPPORTED_QUERIES}")
    if isinstance(tables, Dataset):
        tables = load_tables(tables)
    ctx = DeviceContext(Endpoint(0, 1, "nccl"), tables, variant, timed=False)
    res = PLAN_FUNCTIONS[qid](ctx)
    return res.materialize() if res is not None else None

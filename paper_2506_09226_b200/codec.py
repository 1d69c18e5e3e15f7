"""Bit-packed host columns for the host -> HBM load path (csrc/codec.cu).

The cold path -- a dataset in host memory becoming HBM-resident tables
(the reference's ``partition_dataset`` hand-off, data.py:284-302; the
paper's cold run) -- is bound by PCIe, ~48 GB/s against
~6.5 TB/s of HBM.  Columns are already narrowed losslessly at generation
(table.py); for the copy they are packed further:

* FOR   -- frame of reference: ``value - lo`` in ``k = bits(hi - lo)`` bits
           (dates 12 bits, quantity 6, flags 1-3, keys 20-28, prices 24);
* DELTA -- a non-decreasing column (l_orderkey) packs its deltas per 2048-row
           block (1 bit per row at uniform SF100) plus one int64 base per block;
* IOTA  -- a surrogate key column (lo, lo+1, ...) sends nothing;
* DIFF  -- a date against another date of the same row (l_shipdate against
           l_receiptdate: 5 bits);
* FKDIFF-- a date against its parent row's date through a foreign key into a
           dense key (l_receiptdate - o_orderdate[l_orderkey - 1]: 8 bits
           instead of 12; l_commitdate: 6), chosen only where it is narrower;
* FKIDX -- a column that is one of its parent group's values, as its index in
           the group (l_suppkey = the j-th partsupp supplier of l_partkey:
           2 bits instead of 20), where the parent is grouped by a dense key
           with a fixed fan-out;
* RAW   -- anything that would not shrink (raw float64, k >= the narrowed width).

``scx_pack_host`` (threaded C++) packs; ``scx_unpack`` rebuilds the narrowed
column on the device on the copy stream, right behind its words.  At SF100
the 21.7 GB of narrowed columns cross PCIe as ~10 GB.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import os

import numpy as np

from . import _lib as L
from .table import NP_TO_SCX, HostColumn

RAW = -1
DIFF = 3                 # column-relative: value = ref[i] + lo + field (scx_unpack_diff)
FKDIFF = 4               # key-relative: value = parent[fk[i] - fk_lo] + lo + field
# (child table, foreign key, parent table, dense parent key): the key-relative
# candidates the packer tries (TPC-H's lineitem -> orders, data.py schema)
FOREIGN_KEYS = (("lineitem", "l_orderkey", "orders", "o_orderkey"),)
FKIDX = 5                # key-indexed: value = parent[(fk[i] - fk_lo) * fanout + field]
# (child, group key, member, parent, parent group key, parent member): the
# composite foreign keys the packer tries (lineitem (partkey, suppkey) ->
# partsupp, TPC-H's PARTSUPP relation)
COMPOSITE_KEYS = (("lineitem", "l_partkey", "l_suppkey", "partsupp", "ps_partkey", "ps_suppkey"),)
_CHUNK = 1 << 24


@dataclass
class PackedColumn:
    """A HostColumn in its transfer encoding (``meta`` keeps the logical
    description; its ``values`` are only needed by RAW)."""

    meta: HostColumn
    n: int
    encoding: int
    k: int = 0
    lo: int = 0
    words: np.ndarray | None = None      # u32
    bases: np.ndarray | None = None      # i64, DELTA only
    ref: str | None = None               # DIFF: the reference column of the same table
    fk: str | None = None                # FKDIFF: foreign-key column of this table
    fk_lo: int = 0                       # FKDIFF: parent row = fk - fk_lo
    ref_table: str | None = None         # FKDIFF / FKIDX: parent table (ref = its column)
    fanout: int = 1                      # FKIDX: parent rows per key

    @property
    def dtype(self) -> np.dtype:
        return self.meta.values.dtype

    @property
    def nbytes(self) -> int:
        """Bytes that cross PCIe for this column."""
        if self.encoding == RAW:
            return int(self.meta.values.nbytes)
        b = 0 if self.words is None else int(self.words.nbytes)
        return b + (0 if self.bases is None else int(self.bases.nbytes))


def _bits(span: int) -> int:
    return int(span).bit_length() if span > 0 else 0


def _delta_bits(v: np.ndarray, block: int) -> int | None:
    """Bits of the largest in-block delta of a non-decreasing column (None if
    a delta is negative: the column is not sorted after all)."""
    mx = 0
    for s in range(0, len(v), _CHUNK):
        c = v[s:min(len(v), s + _CHUNK + 1)].astype(np.int64)
        d = np.diff(c)
        if d.size == 0:
            continue
        # block-start rows carry field 0: their deltas are not encoded
        starts = np.arange(s + 1, s + 1 + d.size)
        d = np.where(starts % block == 0, 0, d)
        if d.min() < 0:
            return None
        mx = max(mx, int(d.max()))
    return _bits(mx)


def pack_column(hc: HostColumn, threads: int = 0) -> PackedColumn:
    v = np.ascontiguousarray(hc.values)
    n = len(v)
    if v.dtype.kind not in "iu" or v.dtype not in NP_TO_SCX:
        return PackedColumn(hc, n, RAW)
    if hc.dense and n and hc.hi - hc.lo + 1 == n:
        return PackedColumn(hc, n, L.PACK_IOTA, 0, hc.lo)
    lib = L.load()
    k_for = _bits(hc.hi - hc.lo) if n and hc.hi >= hc.lo else 0
    enc, k = L.PACK_FOR, k_for
    block = int(lib.scx_pack_delta_block())
    if hc.sorted and n:
        kd = _delta_bits(v, block)
        if kd is not None and kd < k_for:
            enc, k = L.PACK_DELTA, kd
    if k > 32 or k >= 8 * v.dtype.itemsize:
        return PackedColumn(hc, n, RAW)
    words = np.empty(int(lib.scx_pack_words(n, k)), dtype=np.uint32)
    bases = np.empty(max(1, (n + block - 1) // block), dtype=np.int64) \
        if enc == L.PACK_DELTA else None
    L.call("scx_pack_host", v.ctypes.data_as(C.c_void_p), NP_TO_SCX[v.dtype], n, hc.lo, k,
           1 if enc == L.PACK_DELTA else 0, words.ctypes.data_as(C.c_void_p),
           bases.ctypes.data_as(C.c_void_p) if bases is not None else None, threads)
    return PackedColumn(hc, n, enc, k, hc.lo, words, bases)


def _pack_diff(hc: HostColumn, ref: HostColumn, name: str, threads: int) -> PackedColumn | None:
    """value - ref[i] in FOR bits, or None when that is not narrower."""
    v = np.asarray(hc.values)
    n = len(v)
    lo = hi = None
    for s0 in range(0, n, _CHUNK):       # chunked min / max of the difference
        d = v[s0:s0 + _CHUNK].astype(np.int64) - np.asarray(ref.values[s0:s0 + _CHUNK]).astype(np.int64)
        lo = int(d.min()) if lo is None else min(lo, int(d.min()))
        hi = int(d.max()) if hi is None else max(hi, int(d.max()))
    k = _bits(hi - lo)
    k_for = _bits(hc.hi - hc.lo) if hc.hi >= hc.lo else 0
    if k > 32 or k + 2 > k_for:
        return None
    lib = L.load()
    words = np.empty(int(lib.scx_pack_words(n, k)), dtype=np.uint32)
    d = (v.astype(np.int64) - np.asarray(ref.values).astype(np.int64))
    L.call("scx_pack_host", d.ctypes.data_as(C.c_void_p), L.SCX_I64, n, lo, k, 0,
           words.ctypes.data_as(C.c_void_p), None, threads)
    return PackedColumn(hc, n, DIFF, k, lo, words, None, name)


def pack_table(ht, threads: int = 0) -> dict[str, PackedColumn]:
    """Every column in its cheapest transfer encoding; a date column may be
    stored against another date of the same table (l_receiptdate against
    l_shipdate: 5 bits; l_commitdate: 8 instead of 12) when that saves > 2
    bits per row.  References are never themselves column-relative."""
    out = {c: pack_column(hc, threads) for c, hc in ht.columns.items()}
    if len(ht.columns) and next(iter(ht.columns.values())).row_count == 0:
        return out
    dates = [c for c, hc in ht.columns.items() if hc.kind == "date32" and out[c].encoding != RAW]
    refs = set()
    for c in dates:
        if c in refs:                     # another column is stored against it
            continue
        best = None
        for r in dates:
            if r == c or out[r].encoding == DIFF:
                continue
            pc = _pack_diff(ht.columns[c], ht.columns[r], r, threads)
            if pc is not None and (best is None or pc.k < best.k):
                best = pc
        if best is not None and best.k + 2 <= out[c].k:
            out[c] = best
            refs.add(best.ref)
    return out


def _pack_fkdiff(hc: HostColumn, fk: HostColumn, parent: HostColumn, fk_lo: int, ref: str,
                 ref_table: str, fk_name: str, threads: int) -> PackedColumn | None:
    """value - parent[fk[i] - fk_lo] in FOR bits (None when out of range)."""
    v = np.asarray(hc.values)
    n = len(v)
    pv = np.asarray(parent.values)
    lo = hi = None
    for s0 in range(0, n, _CHUNK):
        idx = np.asarray(fk.values[s0:s0 + _CHUNK]).astype(np.int64) - fk_lo
        if idx.size and (idx.min() < 0 or idx.max() >= len(pv)):
            return None
        d = v[s0:s0 + _CHUNK].astype(np.int64) - pv[idx].astype(np.int64)
        if d.size:
            lo = int(d.min()) if lo is None else min(lo, int(d.min()))
            hi = int(d.max()) if hi is None else max(hi, int(d.max()))
    if lo is None:
        return None
    k = _bits(hi - lo)
    if k > 32:
        return None
    lib = L.load()
    words = np.empty(int(lib.scx_pack_words(n, k)), dtype=np.uint32)
    d = v.astype(np.int64) - pv[np.asarray(fk.values).astype(np.int64) - fk_lo].astype(np.int64)
    L.call("scx_pack_host", d.ctypes.data_as(C.c_void_p), L.SCX_I64, n, lo, k, 0,
           words.ctypes.data_as(C.c_void_p), None, threads)
    return PackedColumn(hc, n, FKDIFF, k, lo, words, None, ref, fk_name, fk_lo, ref_table)


def _pack_fkidx(hc: HostColumn, fk: HostColumn, pkey: HostColumn, pval: HostColumn,
                ref: str, ref_table: str, fk_name: str, threads: int) -> PackedColumn | None:
    """Index of each value within its parent group (None when the parent is
    not grouped by a dense key with a fixed fan-out, or a value is not among
    its group's)."""
    pk = np.asarray(pkey.values)
    npar = len(pk)
    if npar == 0 or pkey.hi < pkey.lo:
        return None
    nkeys = pkey.hi - pkey.lo + 1
    if npar % nkeys:
        return None
    fan = npar // nkeys
    for s0 in range(0, npar, _CHUNK):           # grouped: key = lo + row // fanout
        r = np.arange(s0, min(npar, s0 + _CHUNK), dtype=np.int64)
        if not np.array_equal(pk[s0:s0 + _CHUNK].astype(np.int64), pkey.lo + r // fan):
            return None
    pv = np.asarray(pval.values)
    v = np.asarray(hc.values)
    n = len(v)
    idx = np.empty(n, dtype=np.int64)
    for s0 in range(0, n, _CHUNK):
        f = np.asarray(fk.values[s0:s0 + _CHUNK]).astype(np.int64) - pkey.lo
        if f.size and (f.min() < 0 or f.max() >= nkeys):
            return None
        base = f * fan
        want = v[s0:s0 + _CHUNK]
        j = np.full(len(f), -1, dtype=np.int64)
        for g in range(fan - 1, -1, -1):        # first match wins
            j[pv[base + g] == want] = g
        if (j < 0).any():
            return None
        idx[s0:s0 + len(f)] = j
    k = _bits(fan - 1)
    lib = L.load()
    words = np.empty(int(lib.scx_pack_words(n, k)), dtype=np.uint32)
    L.call("scx_pack_host", idx.ctypes.data_as(C.c_void_p), L.SCX_I64, n, 0, k, 0,
           words.ctypes.data_as(C.c_void_p), None, threads)
    return PackedColumn(hc, n, FKIDX, k, 0, words, None, ref, fk_name, pkey.lo, ref_table, fan)


def pack_tables(tables: dict, threads: int = 0) -> dict[str, dict[str, PackedColumn]]:
    """pack_table for every table, then each child date column of a
    FOREIGN_KEYS pair stored against a parent date (FKDIFF) where that is at
    least 2 bits narrower than its own encoding.  A column another column is
    stored against (a DIFF reference) may itself become key-relative: it is
    rebuilt first on the device."""
    out = {t: pack_table(ht, threads) for t, ht in tables.items()}
    for child, fk, parent, pk in FOREIGN_KEYS:
        if child not in tables or parent not in tables:
            continue
        ct, pt = tables[child], tables[parent]
        if fk not in ct.columns or pk not in pt.columns or ct.columns[fk].row_count == 0:
            continue
        pkc = pt.columns[pk]
        if not (pkc.dense and pkc.row_count == pkc.hi - pkc.lo + 1):
            continue                       # parent row = key - lo needs a dense key
        pdates = [c for c, hc in pt.columns.items() if hc.kind == "date32"]
        for c, hc in ct.columns.items():
            if hc.kind != "date32" or out[child][c].encoding == RAW:
                continue
            best = None
            for r in pdates:
                pc = _pack_fkdiff(hc, ct.columns[fk], pt.columns[r], pkc.lo, r, parent, fk,
                                  threads)
                if pc is not None and (best is None or pc.k < best.k):
                    best = pc
            if best is not None and best.k + 2 <= out[child][c].k:
                out[child][c] = best
    for child, fk, member, parent, pkey, pmember in COMPOSITE_KEYS:
        if child not in tables or parent not in tables:
            continue
        ct, pt = tables[child], tables[parent]
        if not ({fk, member} <= set(ct.columns) and {pkey, pmember} <= set(pt.columns)):
            continue
        if ct.columns[member].row_count == 0 or out[child][member].encoding == RAW:
            continue
        pc = _pack_fkidx(ct.columns[member], ct.columns[fk], pt.columns[pkey],
                         pt.columns[pmember], pmember, parent, fk, threads)
        if pc is not None and pc.k + 2 <= out[child][member].k:
            out[child][member] = pc
    return out


def unpack_host(pc: PackedColumn, ref_values: np.ndarray | None = None,
                fk_values: np.ndarray | None = None) -> np.ndarray:
    """numpy restatement of scx_unpack / scx_unpack_diff / scx_unpack_fkdiff
    (test infrastructure)."""
    if pc.encoding == RAW:
        return np.asarray(pc.meta.values)
    if pc.encoding == FKIDX:
        f = unpack_host(PackedColumn(pc.meta, pc.n, L.PACK_FOR, pc.k, 0, pc.words)).astype(np.int64) \
            if pc.k else np.zeros(pc.n, dtype=np.int64)
        row = (np.asarray(fk_values).astype(np.int64) - pc.fk_lo) * pc.fanout + f
        return np.asarray(ref_values)[row].astype(pc.dtype)
    if pc.encoding == FKDIFF:
        f = unpack_host(PackedColumn(pc.meta, pc.n, L.PACK_FOR, pc.k, 0, pc.words)).astype(np.int64) \
            if pc.k else np.zeros(pc.n, dtype=np.int64)
        par = np.asarray(ref_values).astype(np.int64)[np.asarray(fk_values).astype(np.int64) - pc.fk_lo]
        return (par + pc.lo + f).astype(pc.dtype)
    if pc.encoding == DIFF:
        f = unpack_host(PackedColumn(pc.meta, pc.n, L.PACK_FOR, pc.k, 0, pc.words)).astype(np.int64) \
            if pc.k else np.zeros(pc.n, dtype=np.int64)
        return (np.asarray(ref_values).astype(np.int64) + pc.lo + f).astype(pc.dtype)
    n, k = pc.n, pc.k
    if pc.encoding == L.PACK_IOTA:
        return (pc.lo + np.arange(n, dtype=np.int64)).astype(pc.dtype)
    if k == 0:
        f = np.zeros(n, dtype=np.int64)
    else:
        bit = np.arange(n, dtype=np.int64) * k
        w = pc.words.astype(np.uint64)
        two = w[bit >> 5] | (w[(bit >> 5) + 1] << np.uint64(32))
        f = ((two >> (bit & 31).astype(np.uint64)) & np.uint64((1 << k) - 1)).astype(np.int64)
    if pc.encoding == L.PACK_FOR:
        return (pc.lo + f).astype(pc.dtype)
    block = int(L.load().scx_pack_delta_block())
    out = np.empty(n, dtype=np.int64)
    for b in range(0, n, block):
        out[b:b + block] = pc.bases[b // block] + np.cumsum(f[b:b + block])
    return out.astype(pc.dtype)


def scratch_bytes(pp: "PinnedPacked") -> int:
    """Device scratch (256-B aligned words + bases) of one packed column."""
    n = 0
    if pp.words is not None:
        n += (pp.words.numel() * 4 + 255) // 256 * 256
    if pp.bases is not None:
        n += (pp.bases.numel() * 8 + 255) // 256 * 256
    return n


_H2D_CHUNK = int(os.environ.get("SCX_H2D_CHUNK_MB", "64")) * (1 << 20) // 4


def upload_packed(pc: PackedColumn, src_words, src_bases, stream, scratch=None, ref_col=None,
                  unpack_stream=None, fk_col=None):
    """Device column buffer of ``pc``: H2D of the pinned words (+ bases) on
    ``stream``, then scx_unpack on the same stream.  ``scratch``: a uint8
    device view of >= scratch_bytes() (the caller carves one arena per upload
    so repeated uploads reuse one allocation); without it the words get their
    own allocation, fenced to ``stream`` (record_stream)."""
    import torch
    from .table import alloc
    buf = alloc(pc.n, pc.dtype)
    dw = db = None
    off = 0
    if src_words is not None and pc.words is not None:
        nw = src_words.numel()
        if scratch is not None:
            dw = scratch[off:off + nw * 4].view(torch.int32)
            off += (nw * 4 + 255) // 256 * 256
        else:
            dw = alloc(nw, np.int32)
    if src_bases is not None:
        nb = src_bases.numel()
        db = scratch[off:off + nb * 8].view(torch.int64) if scratch is not None \
            else alloc(nb, np.int64)
    with torch.cuda.stream(stream):
        if dw is not None:
            # H2D in pieces of _H2D_CHUNK words: the copy engines interleave the
            # other copy stream's pieces and the queries' D2H result reads with
            # them instead of queueing behind one multi-GB transfer
            for a in range(0, nw, _H2D_CHUNK or max(nw, 1)):
                dw[a:a + (_H2D_CHUNK or nw)].copy_(src_words[a:a + (_H2D_CHUNK or nw)],
                                                   non_blocking=True)
            if scratch is None:
                dw.record_stream(stream)
        if db is not None:
            db.copy_(src_bases, non_blocking=True)
            if scratch is None:
                db.record_stream(stream)
    us = stream
    if unpack_stream is not None:
        # the unpack on its own stream, behind this column's copy: the copy
        # stream goes on with the next column's words
        ev = torch.cuda.Event()
        ev.record(stream)
        unpack_stream.wait_event(ev)
        us = unpack_stream
        if scratch is None:
            for t in (dw, db):
                if t is not None:
                    t.record_stream(us)
    with torch.cuda.stream(us):
        if pc.encoding == FKIDX:
            L.call("scx_unpack_fkidx", C.c_void_p(dw.data_ptr() if dw is not None else 0), pc.n,
                   pc.k, L.Column_(fk_col.data_ptr(), _scx_of(fk_col), 0), pc.fk_lo, pc.fanout,
                   L.Column_(ref_col.data_ptr(), _scx_of(ref_col), 0), ref_col.numel(),
                   L.Column_(buf.data_ptr(), NP_TO_SCX[pc.dtype], 0), L.stream_ptr(us))
        elif pc.encoding == FKDIFF:
            L.call("scx_unpack_fkdiff", C.c_void_p(dw.data_ptr() if dw is not None else 0), pc.n,
                   pc.k, pc.lo, L.Column_(fk_col.data_ptr(), _scx_of(fk_col), 0), pc.fk_lo,
                   L.Column_(ref_col.data_ptr(), _scx_of(ref_col), 0), ref_col.numel(),
                   L.Column_(buf.data_ptr(), NP_TO_SCX[pc.dtype], 0), L.stream_ptr(us))
        elif pc.encoding == DIFF:
            L.call("scx_unpack_diff", C.c_void_p(dw.data_ptr() if dw is not None else 0), pc.n,
                   pc.k, pc.lo, L.Column_(ref_col.data_ptr(), _scx_of(ref_col), 0),
                   L.Column_(buf.data_ptr(), NP_TO_SCX[pc.dtype], 0), L.stream_ptr(us))
        else:
            L.call("scx_unpack", C.c_void_p(dw.data_ptr() if dw is not None else 0), pc.n, pc.k,
                   pc.lo, pc.encoding, C.c_void_p(db.data_ptr() if db is not None else 0),
                   L.Column_(buf.data_ptr(), NP_TO_SCX[pc.dtype], 0), L.stream_ptr(us))
    return buf


def _scx_of(t) -> int:
    """SCX dtype of a torch device tensor."""
    return NP_TO_SCX[np.dtype(str(t.dtype).replace("torch.", ""))]


@dataclass
class PinnedPacked:
    """A packed column with its words / bases in pinned host memory."""

    col: PackedColumn
    words: object = None       # torch uint32 (int32 view) pinned tensor
    bases: object = None       # torch int64 pinned tensor

    @property
    def nbytes(self) -> int:
        return self.col.nbytes


def _pin(a: np.ndarray):
    import torch
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a if a.flags.writeable else a.copy()).pin_memory()


def pin_tables(tables: dict, packed: bool = True, threads: int = 0) -> dict:
    """{table: {column: (HostColumn, source)}} for engine.upload_tables_async:
    the source is a pinned raw tensor, or a PinnedPacked (packed=True) whose
    words cross PCIe and are unpacked on the device."""
    out = {}
    packs = pack_tables(tables, threads) if packed else {}
    for t, ht in tables.items():
        cols = {}
        pt = packs[t] if packed else {}
        for c, hc in ht.columns.items():
            pc = pt[c] if packed else PackedColumn(hc, hc.row_count, RAW)
            if pc.encoding == RAW:
                cols[c] = (hc, _pin(hc.values))
            else:
                cols[c] = (hc, PinnedPacked(pc, _pin(pc.words) if pc.words is not None else None,
                                            _pin(pc.bases) if pc.bases is not None else None))
        out[t] = cols
    return out


def h2d_bytes(host: dict) -> int:
    """Bytes a pin_tables() result moves over PCIe."""
    tot = 0
    for cols in host.values():
        for _, src in cols.values():
            tot += src.nbytes if isinstance(src, PinnedPacked) else src.numel() * src.element_size()
    return tot

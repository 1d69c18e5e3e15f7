"""Local relational operators on HBM-resident tables, compiled to libscx.

Drop-in for ``shufflecast.relops`` (`/root/reference/pkg/src/shufflecast/
relops.py`): ``filter_table`` (20), ``local_hash_join`` (59), and
``group_aggregate`` (97), plus the ``ColumnTable.take/sort_by/head`` bodies
(`table.py:171-214`).  Semantics follow the reference exactly:

* filter keeps input order; inner join returns left order, left columns then
  right columns, duplicate names raise ``SchemaError``; semi/anti return left
  rows in left order (relops.py:73-94);
* group output is sorted by the group keys, dict keys by *string*
  (relops.py:160, table.py:198-214); sum of int -> int64, sum/avg of float ->
  float64, count -> int64, min/max keep the kind; a no-key aggregate of an
  empty input is one row (relops.py:124-158).

Execution is *lazy*: ``filter``/``select``/``join``/``add_column`` on a base
table return a ``TableView`` that records a predicate, probe stages and
computed measures.  The view runs as ONE fused scan-kernel launch when it is
aggregated (``group_aggregate``), materialised (stable compaction), or used
as a join build side -- so Q1/Q6/Q14/Q19 read each touched column exactly
once (late materialisation), and no numpy touches a row.
"""

from __future__ import annotations

import collections
import ctypes as C
import os
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from . import _lib as L
from .expr import (INT64_MAX, INT64_MIN, Atom, ColRef, DerivedKey, IntMeasure, Poly, Pred,
                   as_poly, decimal_exponent, integerise)
from .table import Column, ColumnTable, HostColumn, SchemaError, alloc, to_host

AGG_OPS = ("sum", "count", "min", "max", "avg")
_KEY_KINDS = ("int64", "date32", "dict")
_GROUP_MAT = os.environ.get("SCX_GROUP_MAT", "1") != "0"
_SORTED_RANK = os.environ.get("SCX_SORTED_RANK", "1") != "0"
# stream aggregation over a sorted key (scx_sorted_group_agg) measured on
# B200 for Q18: 7.7 ms (warp segmented scan: shuffle-bound) vs 4.4 ms for the
# direct table + HAVING compaction, so it is opt-in (SCX_STREAM_AGG=1)
_STREAM_AGG = os.environ.get("SCX_STREAM_AGG", "0") == "1"
# measured on B200 (SF100, kernel ms): Q8 3.5 -> 5.4, Q3 6.1 -> 7.1, Q17 3.9 -> 4.1
# with the coarse level on, so it is opt-in (SCX_COARSE=1)
_COARSE_BITMAPS = os.environ.get("SCX_COARSE", "0") == "1"
_COARSE_MIN_ROWS = 1 << 22       # big scans only: each CTA stages the coarse bits once
_COARSE_BITS = 1 << 18           # 32 KB of shared memory per kernel
_DIRECT_MAX_SPAN = 1 << 28       # direct lookup tables up to 1 GB of u32 rows
_DENSE_SMEM_BYTES = 48 * 1024     # per-CTA shared-memory group table (keeps 4 CTAs/SM)
_OPCODE = {"sum": L.AGG_SUM, "count": L.AGG_COUNT, "min": L.AGG_MIN, "max": L.AGG_MAX}


def _torch():
    import torch
    return torch


def _stream():
    return L.stream_ptr()


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def _bits(span: int) -> int:
    """bits to hold values 0..span"""
    return int(span).bit_length() if span > 0 else 0


def _device():
    return _torch().device("cuda", _torch().cuda.current_device())


def fill_i64(t, value: int, n: int | None = None, stride: int = 1, offset: int = 0):
    n = t.numel() if n is None else n
    ptr = C.c_void_p(t.data_ptr() + 8 * offset)
    L.call("scx_fill_i64", ptr, n, stride, value, _stream())


def _new_i64(n: int, value: int = 0):
    t = alloc(max(n, 1), np.int64)[:n] if n else alloc(0, np.int64)
    if n:
        fill_i64(t, value)
    return t


def _to_host(t) -> np.ndarray:
    return to_host(t)


# ---------------------------------------------------------------------------
# join build side
# ---------------------------------------------------------------------------

@dataclass
class KeyPacking:
    lo: list[int]
    bits: list[int]
    shift: list[int]

    @property
    def total_bits(self) -> int:
        return sum(self.bits)

    def spec(self, slots: list[int]) -> L.KeySpec:
        ks = L.KeySpec()
        ks.n = len(slots)
        for i, s in enumerate(slots):
            ks.slot[i] = s
            ks.shift[i] = self.shift[i]
            ks.bits[i] = self.bits[i]
            ks.lo[i] = self.lo[i]
        return ks


def key_packing(cols: list[Column]) -> KeyPacking:
    lo = [c.lo if c.hi >= c.lo else 0 for c in cols]
    bits = [_bits(c.hi - c.lo) if c.hi >= c.lo else 0 for c in cols]
    shift = []
    acc = 0
    for b in reversed(bits):
        shift.append(acc)
        acc += b
    shift.reverse()
    if acc > 64:
        raise SchemaError(f"packed key needs {acc} bits (> 64)")
    return KeyPacking(lo, bits, shift)


class Lookup:
    """Device lookup table over a materialised build table's key columns.

    Direct-addressed array when the packed key range is dense (TPC-H primary
    keys), else open addressing with linear probing at load factor <= 0.5.
    """

    def __init__(self, table: ColumnTable, keys: list[str]):
        self.table = table
        self.keys = list(keys)
        cols = [table.column(k) for k in keys]
        self.packing = key_packing(cols)
        n = table.row_count
        span = 1 << self.packing.total_bits if len(keys) > 1 else (
            (cols[0].hi - cols[0].lo + 1) if cols[0].hi >= cols[0].lo else 1)
        self.lk = L.Lookup()
        self._keys = None
        self._unique = None
        if len(cols) == 1 and cols[0].dense and cols[0].row_count == n and n == span:
            # surrogate key column (row i holds lo + i): the packed key is
            # the build row -- no table to build, nothing to read but payload
            self.lk.kind = L.HT_IDENTITY
            self.lk.cap = n
            self.lk.vals = 0
            self.lk.keys = 0
            self._unique = True
            return
        if (span <= max(4 * n, 1 << 16) or span <= _DIRECT_MAX_SPAN) and span <= (1 << 31):
            # a direct table costs span x 4 B of fill (<= 1 GB, ~0.15 ms) but
            # each probe is ONE random sector instead of key + row sectors of
            # open addressing -- the probes dominate (Q7: 171M probes)
            self.lk.kind = L.HT_DIRECT
            self.lk.cap = span
            self._vals = alloc(span, np.uint32)
            self.lk.vals = self._vals.data_ptr()
            self.lk.keys = 0
        else:
            cap = 1024
            while cap < 2 * n:
                cap *= 2
            self.lk.kind = L.HT_HASH
            self.lk.cap = cap
            # 16-byte {key, row} slots: a probe reads both in one sector
            self._keys = alloc(2 * cap, np.uint64)
            self._vals = None
            self.lk.keys = self._keys.data_ptr()
            self.lk.vals = 0
        if self.keys and set(self.keys) == set(getattr(table, "unique_keys", ())):
            self._unique = True            # group-by output keyed on these columns
        self._flags = alloc(4, np.uint32)
        L.call("scx_lookup_clear", C.byref(self.lk), _stream())
        fill_i64(self._flags.view(_torch().int64), 0)
        colarr = (L.Column_ * len(cols))(*[c.scx() for c in cols])
        spec = self.packing.spec(list(range(len(cols))))
        L.call("scx_lookup_build", C.byref(self.lk), colarr, len(cols), C.byref(spec), n,
               _ptr(self._flags), _stream())

    @property
    def unique(self) -> bool:
        if self._unique is None:
            f = _to_host(self._flags)
            self._unique = int(f[1]) == 0
        return self._unique


_BITMAP_MAX_BITS = 1 << 30       # 128 MB of bitmap words


def _key_span(packing: KeyPacking, cols: list[Column]) -> int:
    if len(cols) > 1:
        return 1 << packing.total_bits
    c = cols[0]
    return (c.hi - c.lo + 1) if c.hi >= c.lo else 1


class BitmapLookup:
    """Membership table for semi / anti joins: one bit per packed key.

    At TPC-H key densities the bitmap is 32x smaller than a direct row-index
    table (150M orderkeys: 19 MB, L2-resident) and is built either from a
    materialised table or -- without materialising anything -- by a fused
    scan of the build-side view (SCX_SINK_BITMAP).
    """

    unique = False
    table = None

    def coarse(self, shift: int):
        """Coarse level (bit j = any of fine bits [j << shift, (j+1) << shift)),
        built once per shift (scx_bitmap_coarsen)."""
        if not hasattr(self, "_coarse"):
            self._coarse = {}
        if shift not in self._coarse:
            cbits = ((self.lk.cap - 1) >> shift) + 1 if self.lk.cap else 1
            buf = alloc((cbits + 31) // 32 + 1, np.uint32)
            L.call("scx_bitmap_coarsen", _ptr(self._bits), self.lk.cap, shift, _ptr(buf), _stream())
            self._coarse[shift] = buf
        return self._coarse[shift]

    def __init__(self, source, keys: list[str], cols: list[Column], packing: KeyPacking,
                 span: int):
        self.keys = list(keys)
        self.packing = packing
        self.lk = L.Lookup()
        self.lk.kind = L.HT_BITMAP
        self.lk.cap = span
        self._bits = alloc((span + 31) // 32, np.uint32)
        self.lk.vals = self._bits.data_ptr()
        self.lk.keys = 0
        # build-side row estimate (a tiling hint only, see _first_stage_survival)
        if isinstance(source, TableView):
            f = _pred_survival(source.pre, source.meta) if not source.pre.is_true else 1.0
            self.rows_est = source.base.row_count * f
        else:
            self.rows_est = source.row_count
        L.call("scx_lookup_clear", C.byref(self.lk), _stream())
        if isinstance(source, TableView) and (source.probes or not source.pre.is_true
                                              or not source.post.is_true):
            b = _Builder(source, set(keys))
            S = b.P.sink
            S.kind = L.SINK_BITMAP
            S.gkey = packing.spec([b.slot[k] for k in keys])
            S.gkeys = self._bits.data_ptr()
            S.gcap = span
            b.run()
        else:
            t = source.materialize() if isinstance(source, TableView) else source
            flags = alloc(4, np.uint32)
            fill_i64(flags.view(_torch().int64), 0)
            colarr = (L.Column_ * len(keys))(*[t.column(k).scx() for k in keys])
            spec = packing.spec(list(range(len(keys))))
            L.call("scx_lookup_build", C.byref(self.lk), colarr, len(keys), C.byref(spec),
                   t.row_count, _ptr(flags), _stream())


# ---------------------------------------------------------------------------
# lazy views
# ---------------------------------------------------------------------------

@dataclass
class ProbeStage:
    lookup: Lookup
    probe_keys: list[str]       # names in the view (probe side)
    kind: int                   # JOIN_*
    payload: list[str] = field(default_factory=list)   # right column names exposed
    after: Pred = field(default_factory=Pred.true)      # filter right after this probe


class TableView:
    """A base table seen through predicate / probe / computed-column stages."""

    def __init__(self, base: ColumnTable):
        self.base = base
        self.meta: dict[str, Column] = dict(base.columns)
        self.origin: dict[str, tuple] = {n: ("base", n) for n in base.column_names}
        self.visible: list[str] = list(base.column_names)
        self.pre: Pred = Pred.true()
        self.probes: list[ProbeStage] = []
        self.post: Pred = Pred.true()
        self.computed: dict[str, Poly] = {}
        self.derived: dict[str, DerivedKey] = {}

    def _copy(self) -> "TableView":
        v = TableView.__new__(TableView)
        v.base = self.base
        v.meta = dict(self.meta)
        v.origin = dict(self.origin)
        v.visible = list(self.visible)
        v.pre = self.pre
        v.probes = list(self.probes)
        v.post = self.post
        v.computed = dict(self.computed)
        v.derived = dict(self.derived)
        return v

    # ---- ColumnTable-like surface ----
    @property
    def column_names(self) -> list[str]:
        return list(self.visible)

    def __contains__(self, name: str) -> bool:
        return name in self.visible

    def __getitem__(self, name: str):
        if name in self.computed:
            return self.computed[name]
        if name not in self.meta:
            raise SchemaError(f"unknown column {name!r}; have {self.visible}")
        return ColRef(name, self.meta[name])

    def schema(self) -> dict[str, str]:
        out = {}
        for n in self.visible:
            if n in self.computed:
                out[n] = "int64" if self.computed[n].integral else "float64"
            else:
                out[n] = self.meta[n].kind
        return out

    def isin(self, name: str, values):
        from .expr import isin
        return isin(self[name], values)

    def select(self, names: list[str]) -> "TableView":
        for n in names:
            if n not in self.meta and n not in self.computed:
                raise SchemaError(f"unknown column {n!r}; have {self.visible}")
        v = self._copy()
        v.visible = list(names)
        return v

    def column(self, name: str) -> Column:
        return self.materialize().column(name)

    @property
    def row_count(self) -> int:
        return count_rows(self)

    def with_column(self, name: str, col) -> "TableView":
        v = self._copy()
        if isinstance(col, DerivedKey):
            if col.src not in v.meta:
                raise SchemaError(f"unknown column {col.src!r} for derived key {name!r}")
            v.derived[name] = col
            v.meta[name] = derived_meta(_narrowed(v, col.src), col)
            v.origin[name] = ("derived", col.src)
        elif isinstance(col, (Poly, ColRef)):
            v.computed[name] = as_poly(col)
        elif isinstance(col, Column):
            if self.probes or not self.pre.is_true:
                raise SchemaError("add a materialised Column only to an unfiltered table")
            v.base = self.base.with_column(name, col)
            v.meta[name] = col
            v.origin[name] = ("base", name)
        else:
            raise SchemaError(f"cannot add column of type {type(col).__name__}")
        if name not in v.visible:
            v.visible.append(name)
        return v

    def filter(self, pred) -> "ColumnTable":
        return filter_table(self, pred).materialize()

    def materialize(self) -> ColumnTable:
        return _materialize(self)

    def sort_by(self, names, descending=None) -> ColumnTable:
        return sort_table(self.materialize(), names, descending or set())

    def head(self, n: int) -> ColumnTable:
        return self.materialize().head(n)

    def top(self, names, descending, n: int) -> ColumnTable:
        return sort_table(self.materialize(), names, descending or set(), limit=n)

    def __repr__(self) -> str:
        return (f"TableView(base_rows={self.base.row_count}, visible={self.visible}, "
                f"probes={len(self.probes)})")


def _civil_year(days: int) -> int:
    import datetime
    return (datetime.date(1970, 1, 1) + datetime.timedelta(days=int(days))).year


def _pred_range(pred: Pred, col: str):
    """[lo, hi] that `pred` (DNF) implies for an integer column, or None."""
    if pred.is_true:
        return None
    lo_all, hi_all = None, None
    for clause in pred.clauses:
        lo, hi = INT64_MIN, INT64_MAX
        for a in clause:
            if a.op == "range" and a.col == col and a.col2 is None and not a.negate:
                lo, hi = max(lo, a.lo), min(hi, a.hi)
        if lo == INT64_MIN and hi == INT64_MAX:
            return None            # this clause does not restrict the column
        lo_all = lo if lo_all is None else min(lo_all, lo)
        hi_all = hi if hi_all is None else max(hi_all, hi)
    return (lo_all, hi_all) if lo_all is not None else None


def _narrowed(v: "TableView", name: str) -> Column:
    """Column metadata of `name` with its proven range intersected with the
    ranges the view's predicates imply (Q7's l_shipdate in 1995-1996 gives a
    2-year l_year key domain instead of the column's 7)."""
    import copy
    c = v.meta[name]
    if c.kind not in ("int64", "date32") or v.origin.get(name, ("",))[0] != "base":
        return c
    lo, hi = c.lo, c.hi
    for pred in (v.pre, v.post):
        r = _pred_range(pred, name)
        if r is not None:
            lo, hi = max(lo, r[0]), min(hi, r[1])
    if (lo, hi) == (c.lo, c.hi):
        return c
    c = copy.copy(c)
    c.lo, c.hi = lo, hi
    return c


def derived_meta(src: Column, dk: DerivedKey) -> Column:
    """Metadata (kind, proven range, physical dtype) of a derived group key."""
    from .table import narrow_dtype
    if src.hi < src.lo:
        lo, hi = 0, -1
    elif dk.xform == "year":
        lo, hi = _civil_year(src.lo), _civil_year(src.hi)
    else:
        lo, hi = src.lo, src.hi
    lo, hi = lo + dk.offset, hi + dk.offset
    dt = narrow_dtype(min(lo, 0), max(hi, 0))
    return Column("int64", alloc(0, dt), 0, None, lo, hi)


_XFORM = {"none": L.XFORM_NONE, "year": L.XFORM_YEAR}


def as_view(t) -> TableView:
    if isinstance(t, TableView):
        return t
    if isinstance(t, ColumnTable):
        return TableView(t)
    raise SchemaError(f"expected a table, got {type(t).__name__}")


def _check_pred_columns(v: TableView, pred: Pred, allow_payload: bool):
    for n in pred.columns:
        if n in v.computed:
            raise SchemaError(f"predicate on computed column {n!r} is not supported")
        if n not in v.meta:
            raise SchemaError(f"unknown column {n!r} in predicate")
        if not allow_payload and v.origin[n][0] != "base":
            raise SchemaError("internal: pre-predicate on payload column")


def filter_table(table, predicate) -> TableView:
    """Keep rows where the predicate holds (relops.py:20-22); lazy."""
    v = as_view(table)
    if isinstance(predicate, Pred):
        pred = predicate
    else:
        # a host boolean mask (reference-style numpy filter): upload it as a
        # u8 column and filter on it in the same kernel
        if v.probes or not v.pre.is_true:
            v = TableView(v.materialize())
        mask = np.asarray(predicate)
        if mask.dtype != np.bool_ or len(mask) != v.base.row_count:
            raise SchemaError("filter mask must be boolean and row-aligned")
        mcol = Column.from_numpy("int64", mask.astype(np.int64))
        name = f"__mask{len(v.meta)}"
        v = v._copy()
        v.base = v.base.with_column(name, mcol)
        v.meta[name] = mcol
        v.origin[name] = ("base", name)
        pred = Pred.atom(Atom("range", name, 1, 1))
    v = v._copy()
    _check_pred_columns(v, pred, allow_payload=True)
    _place_pred(v, pred)
    return v


def _place_pred(v: TableView, pred: Pred) -> None:
    """Attach a filter (in place on a copied view) at the earliest stage where
    its columns exist: base-column atoms before any probe (pre-predicate),
    atoms on a join's payload right after that probe -- so a selective
    condition drops rows before the later (random-access) probes."""
    if pred.is_true:
        return

    def stage(cols) -> int:
        return max((v.origin[c][1] if v.origin[c][0] == "payload" else -1 for c in cols),
                   default=-1)

    if len(pred.clauses) == 1:
        groups: dict[int, list] = {}
        for a in pred.clauses[0]:
            groups.setdefault(stage(a.columns), []).append(a)
        parts = [(s, Pred([tuple(atoms)])) for s, atoms in groups.items()]
    else:
        parts = [(stage(pred.columns), pred)]
    for s, p in parts:
        if s < 0:
            v.pre = v.pre & p
        else:
            st = v.probes[s]
            v.probes[s] = ProbeStage(st.lookup, st.probe_keys, st.kind, st.payload, st.after & p)


def local_hash_join(left, right, on: list[tuple[str, str]], how: str = "inner"):
    """Equi-join (relops.py:59-94): probe stage appended to the left view."""
    if how not in ("inner", "semi", "anti", "left"):
        raise SchemaError(f"unknown join type {how!r}")
    if not on:
        raise SchemaError("join requires at least one key pair")
    lv = as_view(left)
    if how == "inner" and isinstance(right, TableView) and len(on) == 1:
        pushed = _pushdown_join(lv, right, on[0], how)
        if pushed is not None:
            return pushed
    if how in ("semi", "anti"):
        rmeta = right.meta if isinstance(right, TableView) else right.columns
        rt = right
    else:
        rt = right.materialize() if isinstance(right, TableView) else right
        rmeta = rt.columns
    for lname, rname in on:
        lc = lv[lname]
        if not isinstance(lc, ColRef):
            raise SchemaError(f"join key {lname!r} must be a column")
        if rname not in rmeta:
            raise SchemaError(f"unknown column {rname!r}")
        rc = rmeta[rname]
        if lc.col.kind != rc.kind:
            raise SchemaError(f"join key type mismatch: {lname} is {lc.col.kind}, "
                              f"{rname} is {rc.kind}")
        if lc.col.kind not in _KEY_KINDS:
            raise SchemaError(f"column {lname!r} of kind {lc.col.kind} cannot be a key")
        if lc.col.kind == "dict" and lc.col.dictionary != rc.dictionary:
            raise SchemaError(f"join keys {lname}/{rname} have different dictionaries")
    if how in ("inner", "left"):
        overlap = set(lv.visible) & set(rt.column_names)
        if overlap:
            raise SchemaError(f"inner join would duplicate columns: {sorted(overlap)}")
    if len(lv.probes) >= L.MAX_PROBES:
        LIMIT_FALLBACKS["probe_stages_materialized"] += 1
        lv = TableView(lv.materialize())
    rkeys = [r for _, r in on]
    lookup = None
    if how in ("semi", "anti"):
        kc = [rmeta[r] for r in rkeys]
        packing = key_packing(kc)
        span = _key_span(packing, kc)
        if span <= _BITMAP_MAX_BITS:
            lookup = BitmapLookup(rt, rkeys, kc, packing, span)
        else:
            rt = rt.materialize() if isinstance(rt, TableView) else rt
    if lookup is None:
        lookup = Lookup(rt, rkeys)
    if how == "inner" and not lookup.unique:
        # duplicate build keys: the fused probe returns one row per probe,
        # so the pairs are expanded by a dedicated count -> scan -> write
        return _expand_join(lv.materialize(), rt, on)
    if how == "left" and not lookup.unique:
        raise SchemaError("left join with duplicate build-side keys is not supported "
                          "(build keys must be unique)")
    v = lv._copy()
    kind = {"inner": L.JOIN_INNER, "semi": L.JOIN_SEMI, "anti": L.JOIN_ANTI,
            "left": L.JOIN_LEFT}[how]
    stage = ProbeStage(lookup, [lname for lname, _ in on], kind)
    if how in ("inner", "left"):
        pidx = len(v.probes)
        for n in rt.column_names:
            stage.payload.append(n)
            c = rt.column(n)
            if how == "left":
                # unmatched rows read 0 (SQL NULL for count / sum payloads)
                if c.kind == "dict":
                    raise SchemaError(f"left join cannot carry dict payload {n!r}")
                c = Column(c.kind, c.data, c.scale, None, min(c.lo, 0), max(c.hi, 0))
            v.meta[n] = c
            v.origin[n] = ("payload", pidx, n)
            v.visible.append(n)
    v.probes.append(stage)
    return v


def _expand_join(lt: ColumnTable, rt: ColumnTable, on: list[tuple[str, str]]) -> ColumnTable:
    """Inner join with duplicate right keys, in the reference's output order
    (relops.py:81-93): left row order, each left row's matches in right row
    order, left columns then right columns.

    Both sides' keys are packed over the union of their value ranges; the
    right keys are radix-sorted stably with their row ids, each left key
    finds its run by binary search (scx_join_match), and one thread per
    output pair writes (left row, right row) (scx_join_expand); the columns
    are then gathered."""
    n, m = lt.row_count, rt.row_count
    lcols = [lt.column(a) for a, _ in on]
    rcols = [rt.column(b) for _, b in on]
    if n == 0 or m == 0:
        idx = alloc(0, np.uint32)
        return ColumnTable({**take_table(lt, idx).columns, **take_table(rt, idx).columns})
    spec = []
    for lc, rc in zip(lcols, rcols):
        l0, l1 = _col_range(lc)
        r0, r1 = _col_range(rc)
        lo, hi = min(l0, r0), max(l1, r1)
        spec.append((lo, _bits(hi - lo)))
    total_bits = sum(b for _, b in spec)
    if total_bits > 64:
        raise SchemaError(f"packed join key needs {total_bits} bits (> 64)")
    shifts, acc = [], 0
    for _, b in reversed(spec):
        shifts.append(acc)
        acc += b
    shifts.reverse()

    def pack(cols, rows):
        key = alloc(rows, np.uint64)
        for i, (c, (lo, b), sh) in enumerate(zip(cols, spec, shifts)):
            L.call("scx_encode_sort_key", c.scx(), None, rows, lo, b, 0, sh, None, _ptr(key),
                   1 if i else 0, _stream())
        return key

    rkey = pack(rcols, m)
    lkey = pack(lcols, n)
    rsorted, rperm = sort_pairs(rkey, None, max(1, total_bits))
    ws = alloc(L.load().scx_join_workspace(n), np.uint8)
    tot = alloc(1, np.uint64)
    L.call("scx_join_match", _ptr(lkey), n, _ptr(rsorted), m, _ptr(ws), _ptr(tot), _stream())
    total = int(_to_host(tot)[0])
    out_l, out_r = alloc(total, np.uint32), alloc(total, np.uint32)
    L.call("scx_join_expand", _ptr(ws), n, _ptr(rperm), total, _ptr(out_l), _ptr(out_r),
           _stream())
    return ColumnTable({**take_table(lt, out_l).columns, **take_table(rt, out_r).columns})


def _pushdown_join(lv: TableView, rv: TableView, on: tuple[str, str], how: str):
    """Join against a *view* of a table keyed by a dense surrogate key without
    materialising the view: the probe reads the base table directly (identity
    lookup, row = key - lo) and the view's own predicates and probes are
    replayed on the gathered payload in the same scan.  E.g. Q3's
    ``lineitem JOIN filter(orders) SEMI customer`` becomes one pipeline:
    lineitem -> orders[row] (o_orderdate, o_custkey, ...) -> customer bitmap
    -> o_orderdate < d.  Returns None when the shape does not fit (the caller
    then materialises the right side as before)."""
    lname, rname = on
    if rv.origin.get(rname, ("x",))[0] != "base":
        return None
    rbase = rv.base
    kc = rbase.column(rname)
    if not (kc.dense and kc.row_count == rbase.row_count and kc.hi - kc.lo + 1 == kc.row_count):
        return None
    if any(n in rv.computed or n in rv.derived for n in rv.visible):
        return None
    lc = lv[lname]
    if not isinstance(lc, ColRef) or lc.col.kind != kc.kind or kc.kind not in _KEY_KINDS:
        return None
    if how == "inner":
        overlap = set(lv.visible) & set(rv.visible)
        if overlap:
            raise SchemaError(f"inner join would duplicate columns: {sorted(overlap)}")
    # right-side columns the replayed plan reads from the base table
    need = {n for n in (rv.visible if how == "inner" else []) if rv.origin[n][0] == "base"}
    need |= {n for n in rv.pre.columns | rv.post.columns if rv.origin[n][0] == "base"}
    for st in rv.probes:
        need |= {k for k in set(st.probe_keys) | st.after.columns if rv.origin[k][0] == "base"}
    need = sorted(need)
    added = set(need) | {n for st in rv.probes for n in st.payload}
    if (len(need) > L.MAX_PAYLOAD or len(lv.probes) + 1 + len(rv.probes) > L.MAX_PROBES
            or added & set(lv.meta) or len(lv.meta) + len(added) > L.MAX_SLOTS):
        if not added & set(lv.meta):
            LIMIT_FALLBACKS["pushdown_join_over_limits"] += 1
        return None
    lookup = Lookup(rbase.select([rname] + [n for n in need if n != rname]), [rname])
    if lookup.lk.kind != L.HT_IDENTITY:
        return None
    v = lv._copy()
    p0 = ProbeStage(lookup, [lname], L.JOIN_INNER, [], rv.pre)
    pidx = len(v.probes)
    for n in need:
        p0.payload.append(n)
        v.meta[n] = rbase.column(n)
        v.origin[n] = ("payload", pidx, n)
    v.probes.append(p0)
    for st in rv.probes:
        idx = len(v.probes)
        v.probes.append(ProbeStage(st.lookup, list(st.probe_keys), st.kind, list(st.payload),
                                   st.after))
        for n in st.payload:
            v.meta[n] = rv.meta[n]
            v.origin[n] = ("payload", idx, n)
    last = v.probes[-1]
    v.probes[-1] = ProbeStage(last.lookup, last.probe_keys, last.kind, last.payload,
                              last.after & rv.post)
    if how == "inner":
        v.visible += [n for n in rv.visible if n not in v.visible]
    return v


# ---------------------------------------------------------------------------
# pipeline construction
# ---------------------------------------------------------------------------

# Plans that hit a descriptor hard limit (scx.h SCX_MAX_PROBES / _PAYLOAD /
# _SLOTS) take a slower shape -- an extra materialisation, or a join that is
# not pushed into the probe scan.  Each such decision is counted here so the
# bench and tests can report it instead of it happening silently.
LIMIT_FALLBACKS: collections.Counter = collections.Counter()

# Per-launch timing for the bench's dominant-kernel roofline: while
# LAUNCH_LOG is a list, every fused-scan launch appends its (start, end) CUDA
# events and LAUNCH_BYTES its algorithmic bytes (rows x narrowed width of the
# base columns it scans).
LAUNCH_LOG: list | None = None
LAUNCH_BYTES: list = []
_DT_BYTES = {L.SCX_I8: 1, L.SCX_U8: 1, L.SCX_I16: 2, L.SCX_U16: 2, L.SCX_I32: 4, L.SCX_U32: 4,
             L.SCX_I64: 8, L.SCX_F64: 8}

# Optional byte trace for roofline accounting: when set to a set(), every
# pipeline adds (device address, bytes) of each base column it scans, so
# the union is the query's distinct HBM bytes read (bench.py).
TRACE: set | None = None


_GATHER_PF_MIN_ROWS = 1 << 20


def _atom_survival(a, meta) -> float:
    c = meta.get(a.col)
    if a.op == "set" and c is not None and c.dictionary:
        f = len(a.codes) / max(1, len(c.dictionary))
    elif a.op == "range" and c is not None and c.hi > c.lo:
        lo, hi = max(a.lo, c.lo), min(a.hi, c.hi)
        f = max(0.0, (hi - lo + 1) / (c.hi - c.lo + 1))
    else:
        f = 0.5
    return 1.0 - f if a.negate else f


def _pred_survival(pred: Pred, meta) -> float:
    """Uniform-independence guess; the range atoms of one column in a clause
    are intersected first (lo <= d AND d < hi is one interval)."""
    tot = 0.0
    for clause in pred.clauses:
        f = 1.0
        ranges = {}
        for a in clause:
            if a.op == "range" and not a.negate:
                lo, hi = ranges.get(a.col, (INT64_MIN, INT64_MAX))
                ranges[a.col] = (max(lo, a.lo), min(hi, a.hi))
            else:
                f *= _atom_survival(a, meta)
        for col, (lo, hi) in ranges.items():
            f *= _atom_survival(Atom("range", col, lo, hi), meta)
        tot += f
    return min(1.0, tot)


def _first_stage_survival(v: "TableView"):
    """Guess of the fraction of rows passing the first filtering stage (the
    pre-predicate, else probe 0 with its after-filter), None if unknown."""
    if not v.pre.is_true:
        return _pred_survival(v.pre, v.meta)
    if not v.probes:
        return None
    st = v.probes[0]
    lk = st.lookup
    f = 1.0
    if lk.lk.kind == L.HT_BITMAP or (lk.lk.kind == L.HT_DIRECT and st.kind != L.JOIN_LEFT):
        t = getattr(lk, "table", None)
        rows = t.row_count if t is not None else getattr(lk, "rows_est", None)
        if rows is not None and lk.lk.cap:
            f = min(1.0, rows / lk.lk.cap)
            if st.kind == L.JOIN_ANTI:
                f = 1.0 - f
        else:
            return None
    if not st.after.is_true:
        f *= _pred_survival(st.after, v.meta)
    return f


def _probe_key_sorted(c: Column) -> bool:
    """Non-decreasing probe key, known without a device check: generated in
    order (l_orderkey, surrogate keys), kept by increasing row selections and
    the stable compaction (_materialize), or verified earlier on the device."""
    return bool(c.sorted)


class _Builder:
    """Assigns operand slots and serialises a TableView into scx_pipeline."""

    def __init__(self, v: TableView, extra: set[str]):
        self.v = v
        self.P = L.Pipeline()
        P = self.P
        P.n_rows = v.base.row_count
        names = set(extra)
        names |= v.pre.columns | v.post.columns
        for st in v.probes:
            names |= st.after.columns
        for st in v.probes:
            names |= set(st.probe_keys)
        base = [n for n in v.base.column_names if n in names and v.origin[n][0] == "base"]
        payload = [n for n in names if v.origin.get(n, ("x",))[0] == "payload"]
        payload.sort(key=lambda n: (v.origin[n][1], v.probes[v.origin[n][1]].payload.index(n)))
        if len(base) > L.MAX_BASE:
            raise SchemaError(f"pipeline touches {len(base)} base columns (> {L.MAX_BASE})")
        if len(base) + len(payload) > L.MAX_SLOTS:
            raise SchemaError("pipeline needs too many operand slots")
        self.slot: dict[str, int] = {}
        for i, n in enumerate(base):
            c = v.meta[n]
            if TRACE is not None:
                TRACE.add((c.data.data_ptr(), c.nbytes))
            P.base[i] = c.scx()
            P.slot_dtype[i] = c.scx_dtype
            self.slot[n] = i
        P.n_base = len(base)
        for j, n in enumerate(payload):
            s = len(base) + j
            self.slot[n] = s
            P.slot_dtype[s] = v.meta[n].scx_dtype
        P.n_slots = len(base) + len(payload)
        self.n_atoms = 0
        self.n_polys = 0
        self.poly_index: dict[str, int] = {}
        self.n_words = 0
        self.n_lut = 0
        self._keep = []   # tensors that must outlive the launch
        # probes
        P.n_probes = len(v.probes)
        n_coarse = sum(1 for st in v.probes if st.lookup.lk.kind == L.HT_BITMAP)
        for i, st in enumerate(v.probes):
            pb = P.probe[i]
            pb.kind = st.kind
            pb.key = st.lookup.packing.spec([self.slot[k] for k in st.probe_keys])
            pb.table = st.lookup.lk
            if (st.lookup.lk.kind == L.HT_BITMAP
                    and (_COARSE_BITMAPS or os.environ.get("SCX_COARSE") == "1")
                    and P.n_rows >= _COARSE_MIN_ROWS):
                # shared-memory coarse level: <= 32 KB of coarse bits shared by
                # this kernel's bitmap probes
                budget = (_COARSE_BITS // n_coarse)
                shift = 0
                while ((st.lookup.lk.cap - 1) >> shift) + 1 > budget:
                    shift += 1
                cb = st.lookup.coarse(shift)
                pb.table.keys = cb.data_ptr()
                pb.table._pad = shift + 1
            if (st.lookup.lk.kind in (L.HT_IDENTITY, L.HT_DIRECT) and len(st.probe_keys) == 1
                    and P.n_rows >= _GATHER_PF_MIN_ROWS
                    and v.origin.get(st.probe_keys[0], ("x",))[0] == "base"
                    and _probe_key_sorted(v.meta[st.probe_keys[0]])):
                # monotone probe sweep: the kernel prefetches the next tile's
                # build range into L2 (jit.cu emit_gather_prefetch)
                pb.table._pad = 1
            used = [n for n in st.payload if n in self.slot]
            if len(used) > L.MAX_PAYLOAD:
                raise SchemaError("too many payload columns from one join")
            pb.n_payload = len(used)
            for j, n in enumerate(used):
                pb.payload[j] = st.lookup.table.column(n).scx()
                pb.payload_slot[j] = self.slot[n]
        self._pred(P.pre, v.pre)
        for i, st in enumerate(v.probes):
            self._pred(P.probe[i].after, st.after)
        self._pred(P.post, v.post)
        # hint for the kernel generator (scx_pipeline._pad): estimated percent
        # of rows surviving the first filtering stage (uniform-range guess;
        # 0 = unknown).  Very selective first stages get bigger chunk tiles.
        est = _first_stage_survival(v)
        P._pad = 0 if est is None else max(1, min(100, int(round(est * 100))))

    # ---- atoms ----
    def _atom(self, a: Atom, clause: int) -> int:
        if self.n_atoms >= L.MAX_ATOMS:
            raise SchemaError("predicate too large (atoms)")
        i = self.n_atoms
        self.n_atoms += 1
        A = self.P.atoms[i]
        A.clause = clause
        A.negate = 1 if a.negate else 0
        if a.op == "poly":
            k = self.poly_index.get(a.poly_key)      # DNF repeats the same comparison
            if k is None:
                if self.n_polys >= L.MAX_POLYS:
                    raise SchemaError("predicate has too many polynomial comparisons")
                im = integerise(a.poly, self.v.meta)
                if _measure_bound(im, self.v.meta) >= (1 << 62):
                    raise SchemaError("polynomial comparison may overflow 64 bits")
                k = self.n_polys
                self.measure(self.P.polys[k], "sum", im)
                self.poly_index[a.poly_key] = k
                self.n_polys += 1
            A.op = L.ATOM_POLY
            A.slot = k
            A.lo, A.hi = a.lo, a.hi
            return i
        A.slot = self.slot[a.col]
        if a.op == "range":
            A.op = L.ATOM_RANGE
            A.lo, A.hi = a.lo, a.hi
        elif a.op == "diff":
            A.op = L.ATOM_DIFF
            A.slot2 = self.slot[a.col2]
            A.lo, A.hi = a.lo, a.hi
        else:
            A.op = L.ATOM_SET
            dsize = len(self.v.meta[a.col].dictionary)
            nw = max(1, (dsize + 31) // 32)
            if self.n_words + nw > L.MAX_SETWORDS:
                raise SchemaError("predicate too large (set words)")
            A.set_word = self.n_words
            A.lo = nw
            for code in a.codes:
                self.P.setwords[self.n_words + code // 32] |= (1 << (code % 32))
            self.n_words += nw
        return i

    def _pred(self, dst: L.Pred, pred: Pred):
        dst.first_atom = self.n_atoms
        if pred.is_true:
            dst.n_atoms = 0
            dst.clause_mask = 0
            return
        clauses = pred.clauses
        if not clauses:   # FALSE: one clause with an impossible atom
            any_col = next(iter(self.slot))
            clauses = ((Atom("range", any_col, 1, 0),),)
        for ci, clause in enumerate(clauses):
            for a in clause:
                self._atom(a, ci)
        dst.n_atoms = self.n_atoms - dst.first_atom
        dst.clause_mask = (1 << len(clauses)) - 1

    def lut(self, values: list[int]) -> int:
        off = self.n_lut
        if off + len(values) > L.MAX_LUT:
            raise SchemaError("dictionary rank tables exceed the descriptor LUT")
        for i, x in enumerate(values):
            self.P.lut[off + i] = x
        self.n_lut += len(values)
        return off

    # ---- measures ----
    def measure(self, dst: L.Measure, op: str, im: IntMeasure | None):
        dst.op = _OPCODE[op]
        dst.cond_atom = -1
        if op == "count":
            dst.n_terms = 0
            if im is not None and im.cond is not None:
                dst.cond_atom = self._atom(im.cond, 0)
            return
        if len(im.terms) > 2:
            raise SchemaError("measure has more than 2 product terms")
        dst.n_terms = len(im.terms)
        for ti, (coef, fs) in enumerate(im.terms):
            if len(fs) > 3:
                raise SchemaError("measure term has more than 3 factors")
            T = dst.t[ti]
            T.coef = coef
            T.n_factors = len(fs)
            for fi, (a, b, col) in enumerate(fs):
                T.f[fi].a, T.f[fi].b, T.f[fi].slot = a, b, self.slot[col]
                # narrow flag (scx_factor._pad): a + b*v fits int32 over the
                # column's [lo, hi] -> the kernel's int32 fast path
                c = self.v.meta[col]
                if c.hi >= c.lo:
                    ext = max(abs(a + b * c.lo), abs(a + b * c.hi))
                    narrow = ext < (1 << 31) and abs(a) < (1 << 31) and abs(b) < (1 << 31)
                else:
                    narrow = abs(a) < (1 << 31) and abs(b) < (1 << 31) and b == 0
                T.f[fi]._pad = 1 if narrow else 0
        if im.cond is not None:
            dst.cond_atom = self._atom(im.cond, 0)

    def run(self, timing: list | None = None):
        """Launch; with `timing`, CUDA events bracket exactly this launch."""
        if timing is None and LAUNCH_LOG is not None:
            timing = LAUNCH_LOG
            LAUNCH_BYTES.append(sum(int(self.P.n_rows) * _DT_BYTES.get(int(self.P.base[i].dtype), 8)
                                    for i in range(int(self.P.n_base))))
        if timing is not None:
            torch = _torch()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            L.call("scx_pipeline_run", C.byref(self.P), _stream())
            e1.record()
            timing.append((e0, e1))
            return
        L.call("scx_pipeline_run", C.byref(self.P), _stream())


def _measure_range(im: IntMeasure | None, meta: dict[str, Column]):
    """[lo, hi] of a measure's per-row value from the columns' proven ranges
    (interval arithmetic; count = 1), or None when a range is not proven."""
    if im is None:
        return 1, 1
    lo_t, hi_t = 0, 0
    for coef, fs in im.terms:
        lo, hi = coef, coef
        for a, bb, col in fs:
            c = meta[col]
            if not (c.lo > INT64_MIN and c.hi < INT64_MAX and c.hi >= c.lo) or c.loose:
                return None
            clo, chi = c.lo, c.hi
            x, y = a + bb * clo, a + bb * chi
            cands = (lo * x, lo * y, hi * x, hi * y)
            lo, hi = min(cands), max(cands)
        lo_t, hi_t = lo_t + lo, hi_t + hi
    if im.cond is not None:            # a gated-off row contributes 0
        lo_t, hi_t = min(lo_t, 0), max(hi_t, 0)
    return lo_t, hi_t


_SMS = None


def _num_sms() -> int:
    global _SMS
    if _SMS is None:
        _SMS = int(_torch().cuda.get_device_properties(_torch().cuda.current_device())
                   .multi_processor_count)
    return _SMS


def _pack_budgets(P, measures, meta, n: int) -> None:
    """Dense sinks: mark sum / count measures whose per-thread partial sum is
    provably non-negative and small with their bit budget (measure._pad =
    0x100 | bits), so the kernel can add several of them with ONE 64-bit
    shared-memory update (Q1: qty, discount and count share a word)."""
    # the launch keeps >= 2 CTAs of 256 threads per SM for packed kernels
    # (jit plan_launch), and 148 SMs: rows per thread <= n / (296 * 256) + V
    rows_per_thread = n // (2 * _num_sms() * 256) + 16
    for i, (op, im) in enumerate(measures):
        if op not in ("sum", "count"):
            continue
        r = _measure_range(im, meta)
        if r is None or r[0] < 0:
            continue
        lo, hi = r
        bits = max(1, int(hi * rows_per_thread).bit_length())
        if bits <= 63:
            P.sink.m[i]._pad = 0x100 | bits


def _measure_bound(im: IntMeasure, meta: dict[str, Column], tight: bool = True) -> int:
    """|value| bound of a measure polynomial.  ``tight``: columns whose proven
    range is loose (an aggregate's: rows x per-row range, far wider than its
    values) are measured with a min/max pass, as an unproven column is;
    sort-key packing uses the proven range as is."""
    tot = 0
    for coef, fs in im.terms:
        b = abs(coef)
        for a, bb, col in fs:
            lo, hi = _col_range(meta[col], tight)
            b *= max(abs(a + bb * lo), abs(a + bb * hi), 1)
        tot += b
    return max(tot, 1)


# ---------------------------------------------------------------------------
# materialisation (stable compaction) and counting
# ---------------------------------------------------------------------------

def _materialize(v: TableView) -> ColumnTable:
    cols = [n for n in v.visible]
    comp = [n for n in cols if n in v.computed or n in v.derived]
    if comp:
        raise SchemaError(f"cannot materialise computed columns {comp}; aggregate them instead")
    if not v.probes and v.pre.is_true and v.post.is_true:
        return v.base.select(cols)
    b = _Builder(v, set(cols))
    P = b.P
    n = v.base.row_count
    S = P.sink
    S.kind = L.SINK_COMPACT
    if len(cols) > L.MAX_OUT:
        raise SchemaError("too many output columns")
    outs = {}
    for i, name in enumerate(cols):
        c = v.meta[name]
        buf = alloc(n, c.np_dtype)
        outs[name] = buf
        S.out_slot[i] = b.slot[name]
        S.out[i] = L.Column_(buf.data_ptr(), c.scx_dtype, 0)
    S.n_out = len(cols)
    words = L.load().scx_pipeline_status_words(C.byref(P))
    if words < 0:
        L.check(-1 if words == -1 else int(words), "scx_pipeline_status_words")
    # per-CTA counts + the staging area of the stable compaction: every word
    # the kernel reads is written first, so no clearing is needed
    status = alloc(max(int(words), 2), np.int64)
    count = _new_i64(1, 0)
    S.status = status.data_ptr()
    S.count = count.data_ptr()
    b.run()
    m = int(_to_host(count)[0]) if n else 0
    # probes build on unique keys, so a filtered / joined row set keeps the
    # base table's key property
    out = {}
    for name in cols:
        c = v.meta[name].like(_fit(outs[name], m))
        if v.origin[name][0] == "base" and v.meta[name].sorted:
            c.sorted = True          # the compaction is stable: order is kept
        out[name] = c
    return ColumnTable(out, v.base.unique_keys)


def _fit(buf, m: int):
    """buf[:m], copied into its own allocation when that is much smaller: a
    view would keep the whole capacity-sized buffer alive as long as the
    result (a 150M-slot group table behind a 600-row HAVING result)."""
    if m * 2 >= buf.shape[0] or buf.shape[0] - m < (1 << 16):
        return buf[:m]
    out = alloc(m, np.dtype(str(buf.dtype).replace("torch.", "")))
    if m:
        out.copy_(buf[:m])
    return out


def count_rows(t) -> int:
    if isinstance(t, ColumnTable):
        return t.row_count
    v = t
    if not v.probes and v.pre.is_true and v.post.is_true:
        return v.base.row_count
    b = _Builder(v, set())
    b.P.sink.kind = L.SINK_COUNT
    count = _new_i64(1, 0)
    b.P.sink.count = count.data_ptr()
    b.run()
    return int(_to_host(count)[0])


# ---------------------------------------------------------------------------
# group-by aggregation
# ---------------------------------------------------------------------------

@dataclass
class _Agg:
    out: str
    op: str
    poly: Poly | None
    kind: str               # output logical kind
    m: int = -1             # measure index (sum/min/max/count)
    cnt: int = -1           # count measure index (avg)
    q: int = 1
    scale: int = 0          # source column scale for min/max of decimals
    src: Column | None = None


_LUT_CACHE: dict = {}


def _rank_lut(dictionary) -> list[int]:
    """code -> rank of its string (dict keys sort by string); cached per
    dictionary object (an argsort of the strings per call is host time)."""
    hit = _LUT_CACHE.get(id(dictionary))
    if hit is not None and hit[0] is dictionary:
        return hit[1]
    order = np.argsort(np.asarray(dictionary, dtype=object), kind="stable")
    rank = np.empty(len(dictionary), dtype=np.int64)
    rank[order] = np.arange(len(dictionary))
    lut = [int(x) for x in rank]
    _LUT_CACHE[id(dictionary)] = (dictionary, lut)
    return lut


def _plan_aggs(v: TableView, aggs: dict) -> tuple[list[_Agg], list[tuple[str, IntMeasure | None]]]:
    for out, (op, colname) in aggs.items():
        if op not in AGG_OPS:
            raise SchemaError(f"unknown aggregate {op!r} for {out!r}")
        if op != "count" and colname is None:
            raise SchemaError(f"aggregate {out!r} ({op}) needs a column")
    plan: list[_Agg] = []
    measures: list[tuple[str, IntMeasure | None]] = []
    count_idx = -1

    def add_measure(op, im):
        key = (op, None if im is None else (repr(im.terms), im.q, im.cond))
        for i, (op2, im2) in enumerate(measures):
            if (op2, None if im2 is None else (repr(im2.terms), im2.q, im2.cond)) == key:
                return i
        measures.append((op, im))
        return len(measures) - 1

    def need_count():
        nonlocal count_idx
        if count_idx < 0:
            count_idx = add_measure("count", None)
        return count_idx

    for out, (op, colname) in aggs.items():
        if op == "count":
            plan.append(_Agg(out, op, None, "int64", m=need_count()))
            continue
        expr = v[colname]
        if isinstance(expr, ColRef):
            c = expr.col
            if c.kind == "dict":
                raise SchemaError(f"{op} not supported on dict column {colname!r}")
            poly = expr.poly()
            src = c
        else:
            poly = expr
            src = None
        im = integerise(poly, v.meta)
        if op in ("min", "max"):
            if src is None:
                # min/max of where(cond, col): a single gated column is allowed
                t = poly.terms
                if (len(t) == 1 and t[0].coef == 1 and len(t[0].factors) == 1
                        and t[0].factors[0].a == 0 and t[0].factors[0].b == 1):
                    src = v.meta[t[0].factors[0].col]
                else:
                    raise SchemaError(f"{op} of a computed column is not supported")
            plan.append(_Agg(out, op, poly, src.kind, m=add_measure(op, im), scale=src.scale,
                             src=src))
            continue
        is_float = (src is not None and src.kind == "float64") or (src is None and not poly.integral)
        if op == "sum":
            plan.append(_Agg(out, op, poly, "float64" if is_float else "int64",
                             m=add_measure("sum", im), q=im.q))
        else:  # avg
            plan.append(_Agg(out, op, poly, "float64", m=add_measure("sum", im),
                             cnt=need_count(), q=im.q))
    return plan, measures


def _apply_having(t, having):
    """HAVING lo <= t[name] <= hi as a filter over a group result."""
    if t is None or having is None:
        return t
    name, lo, hi = having
    return filter_table(t, (t[name] >= lo) & (t[name] <= hi)).materialize()


def group_aggregate(table, group_keys: list[str], aggs: dict[str, tuple],
                    cross=None, timing: list | None = None, sort: bool = True,
                    having: tuple | None = None) -> ColumnTable:
    """Aggregate per group (relops.py:97-160), one fused kernel launch.

    ``cross`` (engine.DeviceContext) makes it a global aggregate over all
    ranks: dense partials are all-gathered and summed exactly in 128 bits;
    hash partials are gathered to the root and re-aggregated.

    ``having = (name, lo, hi)`` keeps the groups with lo <= name <= hi (SQL
    HAVING; same result as filtering the output).  For a direct-addressed
    table and an integer sum / count it is folded into the table compaction.
    """
    if having is not None and (cross is not None and cross.ep.n > 1):
        # partial aggregates cannot be filtered before the cross-rank merge
        return _apply_having(group_aggregate(table, group_keys, aggs, cross, timing, sort),
                             having)
    v = as_view(table)
    keys = list(group_keys)
    fd = _dependent_keys(v, keys)
    if fd:
        return _apply_having(_group_with_dependent_keys(v, keys, fd, aggs, cross, timing, sort),
                             having)
    for k in keys:
        if k in v.computed or k not in v.meta:
            raise SchemaError(f"unknown group key {k!r}")
        if v.meta[k].kind not in _KEY_KINDS:
            raise SchemaError(f"column {k!r} of kind {v.meta[k].kind} cannot be a key")
    # derived keys read their source column, transformed in the kernel
    ksrc = [v.derived[k].src if k in v.derived else k for k in keys]
    plan, measures = _plan_aggs(v, aggs)
    # HAVING lo <= sum with lo > 0 over non-negative rows: an empty slot (sum 0)
    # can never qualify, so the sum itself marks live groups -- no count word
    # (Q18: a 150M-slot direct table of one word instead of two)
    having_occ = None
    if keys and having is not None and int(having[1]) > 0 and \
            not any(op == "count" for op, _ in measures):
        a = next((a for a in plan if a.out == having[0]), None)
        if a is not None and a.op == "sum" and a.kind == "int64" and a.q == 1:
            r = _measure_range(measures[a.m][1], v.meta)
            if r is not None and r[0] >= 0:
                having_occ = a.m
    if keys and having_occ is None and not any(op == "count" for op, _ in measures):
        measures.append(("count", None))     # live-group detection
    count_m = (having_occ if having_occ is not None else
               next(i for i, (op, _) in enumerate(measures) if op == "count")) if keys else None
    if len(measures) > L.MAX_MEASURES:
        raise SchemaError("too many aggregate measures")
    names = set(ksrc)
    for _, im in measures:
        if im is not None:
            names |= {f[2] for _, fs in im.terms for f in fs}
            if im.cond is not None:
                names |= set(im.cond.columns)
    b = _Builder(v, names)
    for i, (op, im) in enumerate(measures):
        b.measure(b.P.sink.m[i], op, im)
    b.P.sink.n_measures = len(measures)

    kcols = [v.meta[k] for k in keys]
    cards = []
    for c in kcols:
        cards.append(len(c.dictionary) if c.kind == "dict" else max(1, c.hi - c.lo + 1))
    cells = int(np.prod(cards)) if keys else 1
    dense = (not keys and len(measures) <= 8) or (keys and cells <= 8 and len(measures) <= 6)
    # small key domains (Q5's 25 nations, Q7's nation pairs x years, Q9's
    # nation x year) aggregate in a per-CTA shared-memory table: smem atomics
    # then one global atomic per cell per CTA, instead of every row hitting
    # the same few global accumulators
    n = v.base.row_count
    smem_table = (keys and not dense and cells * len(measures) * 8 <= _DENSE_SMEM_BYTES)
    if smem_table:
        per_cta = n // 148 + 4096
        smem_table = all(_measure_bound(im, v.meta) * per_cta < (1 << 62)
                         for op, im in measures if im is not None and op == "sum")
    dense = dense or smem_table
    # overflow guard: per-thread int64 partials (dense; exact 128-bit across
    # threads); hash groups switch a sum to a 128-bit {lo, hi} accumulator when
    # n rows of its largest value could leave int64
    for i, (op, im) in enumerate(measures):
        if im is not None and op == "sum":
            bound = _measure_bound(im, v.meta)
            if dense and not smem_table:
                if n > 0 and bound * (n // (148 * 256) + 16) >= (1 << 62):
                    raise SchemaError("aggregate may overflow 64-bit partial sums")
            elif not dense and bound * max(n, 1) >= (1 << 62):
                b.P.sink.m[i]._pad = 1
    b.ksrc = ksrc
    if dense:
        return _apply_having(
            _group_dense(v, b, keys, kcols, cards, cells, plan, measures, count_m, cross, timing),
            having)
    dom = int(np.prod([max(1, c.hi - c.lo + 1) if c.kind != "dict" else len(c.dictionary)
                       for c in kcols])) if keys else 1
    if (_GROUP_MAT and n > (1 << 20) and dom > (1 << 22)
            and any(st.kind in (L.JOIN_SEMI, L.JOIN_ANTI) for st in v.probes)):
        # a hash group-by (large key domain: open addressing with CAS) behind
        # a semi / anti join: compact the surviving rows first, so the group
        # kernel's dependent CAS chains run over dense rows instead of idling
        # behind the filter stages (measured at SF100: Q3 8.8 -> 6.5 ms, Q16
        # 6.6 -> 3.8, Q20 8.4 -> 4.1 of kernel time; without a semi join the
        # extra compaction pass costs more than it saves: Q7, Q10, Q13, Q15)
        need = [c for c in v.visible if c in names] + sorted(names - set(v.visible))
        dense_v = as_view(v.select(need).materialize())
        dense_v.computed = dict(v.computed)
        for k, dk in v.derived.items():
            dense_v.derived[k] = dk
            dense_v.meta[k] = v.meta[k]
        dense_v.visible = list(v.visible)
        return group_aggregate(dense_v, group_keys, aggs, cross, timing, sort, having)
    if (_STREAM_AGG and having is not None and not sort and len(keys) == 1
            and keys[0] not in v.derived and v.origin.get(keys[0], ("",))[0] == "base"
            and kcols[0].kind in ("int64", "date32") and not v.probes and v.pre.is_true
            and v.post.is_true and n > (1 << 16) and (cross is None or cross.ep.n == 1)):
        # clustered key + HAVING (Q18: lineitem by l_orderkey, sum > 300):
        # stream aggregation, no group table at all
        r = _stream_group(v, keys[0], kcols[0], plan, measures, having)
        if r is not None:
            return r
    if (_SORTED_RANK and len(keys) == 1 and keys[0] not in v.derived
            and v.origin.get(keys[0], ("",))[0] == "base" and kcols[0].kind in ("int64", "date32")
            and n > (1 << 16) and dom > max(4 * n, 1 << 16)):
        # clustered key (a materialised lineitem subset by l_orderkey): group
        # by the key's dense rank -- a direct table of #distinct-keys slots
        # filled sequentially -- instead of hashing into one sized by rows
        ranked = _sorted_rank(v.base.column(keys[0]), kcols[0].lo)
        if ranked is not None:
            return _apply_having(_group_by_rank(v, keys[0], kcols[0], ranked, aggs, cross, timing),
                                 having)
    hv = None
    if having is not None:
        a = next((a for a in plan if a.out == having[0]), None)
        if a is None:
            raise SchemaError(f"HAVING on unknown aggregate {having[0]!r}")
        if (a.op == "count" or (a.op == "sum" and a.kind == "int64" and a.q == 1)) \
                and not b.P.sink.m[a.m]._pad:
            hv = (a.m, int(having[1]), int(having[2]))
    part = _group_hash(v, b, keys, kcols, plan, measures, count_m, sort, hv)
    if having is not None and not getattr(part, "_having_done", False):
        part = _apply_having(part, having)
    if cross is None or cross.ep.n == 1:
        return part
    full = cross.gather(part)
    return None if full is None else regroup(full, keys, aggs)


def _sorted_rank(col: Column, lo: int):
    """(rank Column u32, keys_by_rank u64 (key - lo), #distinct) when `col`
    is non-decreasing, else None (and the column remembers it)."""
    if col.sorted is False:
        return None
    torch = _torch()
    n = col.row_count
    rank = alloc(n, np.uint32)
    kbr = alloc(n, np.uint64)
    cnt = alloc(2, np.int64)
    ws = alloc(max(2, L.load().scx_sorted_rank_workspace(n) // 8), np.int64)
    L.call("scx_sorted_rank", C.byref(col.scx()), n, lo, _ptr(rank), _ptr(kbr), _ptr(cnt),
           _ptr(ws), _stream())
    g, bad = (int(x) for x in _to_host(cnt))
    col.sorted = bad == 0
    if bad:
        return None
    return Column("int64", rank, 0, None, 0, max(g - 1, 0)), kbr, g


def _group_by_rank(v: TableView, key: str, kcol: Column, ranked, aggs, cross, timing):
    rank_col, kbr, g = ranked
    torch = _torch()
    v2 = v._copy()
    v2.base = v.base.with_column("__rank", rank_col)
    v2.meta["__rank"] = rank_col
    v2.origin["__rank"] = ("base", "__rank")
    part = group_aggregate(v2, ["__rank"], aggs, None, timing, True)
    G = part.row_count
    r = part.column("__rank")
    packed = alloc(G, np.uint64)
    L.call("scx_gather", L.Column_(kbr.data_ptr(), L.SCX_I64, 0), _ptr(r.data), G,
           L.Column_(packed.data_ptr(), L.SCX_I64, 0), _stream())
    data = alloc(G, kcol.np_dtype)
    L.call("scx_unpack_key", _ptr(packed), G, 0, (1 << 64) - 1, kcol.lo,
           L.Column_(data.data_ptr(), kcol.scx_dtype, 0), _stream())
    cols = {key: kcol.like(data)}
    cols[key].sorted = True
    cols.update({name: part.column(name) for name in aggs})
    out = ColumnTable(cols, (key,))
    if cross is None or cross.ep.n == 1:
        return out
    full = cross.gather(out)
    return None if full is None else regroup(full, [key], aggs)


def _dependent_keys(v: TableView, keys: list[str]) -> list[str]:
    """Group keys that are payload of a unique-build inner join whose probe
    keys are all earlier group keys: they are functionally dependent on those
    keys (Q3's o_orderdate / o_shippriority on l_orderkey), so grouping by the
    determinants alone gives the same groups in the same order."""
    out = []
    for st in v.probes:
        if st.kind != L.JOIN_INNER or not set(st.probe_keys) <= set(keys):
            continue
        last = max(keys.index(k) for k in st.probe_keys)
        for i, k in enumerate(keys):
            if (i > last and k in st.payload and k not in st.probe_keys and k not in out
                    and k not in v.derived and v.meta[k].kind != "dict"):
                out.append(k)
    return out


def _group_with_dependent_keys(v, keys, fd, aggs, cross, timing, sort) -> ColumnTable:
    """Group by the determinant keys; each dependent key rides along as a
    MIN aggregate (all rows of a group carry the same value) and is put back
    in its key position."""
    core = [k for k in keys if k not in fd]
    tmp = {f"__fd_{k}": ("min", k) for k in fd}
    for name in aggs:
        if name in tmp:
            raise SchemaError(f"aggregate name {name!r} is reserved")
    g = group_aggregate(v, core, {**tmp, **aggs}, cross, timing, sort)
    if g is None:
        return None
    cols = {k: g.column(f"__fd_{k}") if k in fd else g.column(k) for k in keys}
    cols.update({name: g.column(name) for name in aggs})
    return ColumnTable(cols, tuple(keys))


def regroup(full, keys: list[str], aggs: dict[str, tuple]) -> ColumnTable:
    """Re-aggregate gathered partial aggregates (sum/count add, min/max fold)."""
    re = {}
    for out, (op, _) in aggs.items():
        if op == "avg":
            raise SchemaError("avg partials cannot be re-aggregated; aggregate sum and count")
        re[out] = ("sum" if op in ("sum", "count") else op, out)
    return group_aggregate(full, keys, re)


def _key_xform(v: TableView, k: str) -> int:
    return _XFORM[v.derived[k].xform] if k in v.derived else L.XFORM_NONE


def _key_offset(v: TableView, k: str) -> int:
    return v.derived[k].offset if k in v.derived else 0


def _group_dense(v, b, keys, kcols, cards, cells, plan, measures, count_m, cross=None, timing=None):
    torch = _torch()
    S = b.P.sink
    S.kind = L.SINK_AGG_DENSE
    _pack_budgets(b.P, measures, v.meta, v.base.row_count)
    S.n_cells = cells
    S.gkey.n = len(keys)
    luts = []
    for i, (k, c) in enumerate(zip(keys, kcols)):
        S.gkey.slot[i] = b.slot[b.ksrc[i]]
        S.gkey.xform |= _key_xform(v, k) << (8 * i)
        S.gcard[i] = cards[i]
        if c.kind == "dict":
            S.gkey.lo[i] = 0
            rank = _rank_lut(c.dictionary)
            S.glut[i] = b.lut(rank)
            luts.append(rank)
        else:
            S.gkey.lo[i] = c.lo - _key_offset(v, k)
            S.glut[i] = -1
            luts.append(None)
    M = len(measures)
    # (cells, M, 2) int64 accumulators initialised on the device (a pageable
    # H2D copy here would synchronise the stream)
    pattern = []
    for op, _ in measures:
        pattern += [INT64_MAX if op == "min" else (INT64_MIN if op == "max" else 0), 0]
    acc = alloc(cells * M * 2, np.int64)
    L.call("scx_fill_rows", _ptr(acc), cells, 2 * M, (C.c_int64 * (2 * M))(*pattern), _stream())
    acc = acc.view(cells, M, 2)
    S.acc = acc.data_ptr()
    b.run(timing)
    if GRAPH_CAPTURE is not None and (cross is None or cross.ep.n == 1):
        GRAPH_CAPTURE.append(DenseGraph(b, acc, pattern, cells, M,
                                        (keys, kcols, cards, luts, plan, measures, count_m)))
    if cross is not None and cross.ep.n > 1:
        from .exchange import all_gather_tensor
        parts = all_gather_tensor(cross.ep, acc)
        red = torch.empty_like(acc)
        ops = (C.c_int * M)(*[1 if op == "min" else (2 if op == "max" else 0)
                             for op, _ in measures])
        L.call("scx_dense_reduce", _ptr(parts), cross.ep.n, cells, M, ops, _ptr(red), _stream())
        acc = red
    return finish_dense(_to_host(acc), keys, kcols, cards, luts, plan, measures, count_m)


# CUDA-graph capture of dense final aggregates (bench.py config 1): while set
# to a list, every single-rank dense group-by also records a DenseGraph
GRAPH_CAPTURE: list | None = None


class DenseGraph:
    """A dense aggregation's device work -- accumulator fill, the fused scan
    kernel, D2H of the exact 128-bit cells into pinned memory -- captured once
    as a CUDA graph.  ``replay()`` relaunches it (no host plan building, one
    graph launch instead of per-kernel launches) and finishes the result on
    the host exactly as the eager path does.  The captured descriptor keeps
    its base-column pointers: the tables must stay alive and unchanged."""

    def __init__(self, b: "_Builder", acc, pattern, cells: int, M: int, finish_args):
        torch = _torch()
        self.b, self.acc, self.finish_args = b, acc, finish_args
        self.pattern = (C.c_int64 * (2 * M))(*pattern)
        self.host = torch.empty(acc.shape, dtype=torch.int64, pin_memory=True)
        self.graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(self.graph, stream=side):
            L.call("scx_fill_rows", _ptr(acc), cells, 2 * M, self.pattern, _stream())
            b.run()
            self.host.copy_(acc, non_blocking=True)
        torch.cuda.current_stream().wait_stream(side)

    def launch(self) -> None:
        self.graph.replay()

    def finish(self) -> "ColumnTable":
        _torch().cuda.current_stream().synchronize()
        return finish_dense(self.host.numpy(), *self.finish_args)

    def replay(self) -> "ColumnTable":
        self.launch()
        return self.finish()


def _i128(lohi) -> int:
    lo = int(lohi[0]) & ((1 << 64) - 1)
    return (int(lohi[1]) << 64) + lo


def _lazy_col(kind, values, dictionary=None) -> Column:
    """Host-backed (lazily uploaded) result column of a final aggregation."""
    return Column.from_host_lazy(HostColumn.from_reference(kind, np.asarray(values), dictionary))


def finish_dense(acc: np.ndarray, keys, kcols, cards, luts, plan, measures, count_m) -> ColumnTable:
    """Assemble the (small) dense-aggregate result from exact 128-bit cells.

    This is the final-aggregation step (the reference's all-reduced grid ->
    result table, queries.py:51-69), vectorised over the live cells; values
    that do not fit int64 fall back to Python integers.
    """
    minmax = [op in ("min", "max") for op, _ in measures]
    if keys:
        # counts are non-negative and < 2^63: the low word alone decides liveness
        live = np.flatnonzero(acc[:, count_m, 0] > 0)
    else:
        live = np.zeros(1, dtype=np.int64)
    lo = acc[live, :, 0]
    fits = acc[live, :, 1] == (lo >> 63)          # the 128-bit value is lo itself

    def exact(j):
        """int64 array of measure j over the live cells, or a list of ints."""
        if minmax[j] or bool(fits[:, j].all()):
            return lo[:, j].copy()
        return [_i128(acc[c, j]) for c in live]

    out: dict[str, Column] = {}
    # decode cell -> per-key rank -> value
    for i, (k, c) in enumerate(zip(keys, kcols)):
        stride = int(np.prod(cards[i + 1:])) if i + 1 < len(cards) else 1
        ranks = (live // stride) % cards[i]
        if luts[i] is not None:
            inv = np.empty(len(luts[i]), dtype=np.int64)
            inv[np.asarray(luts[i], dtype=np.int64)] = np.arange(len(luts[i]))
            out[k] = Column.from_host_lazy(HostColumn.from_codes(inv[ranks], c.dictionary))
        else:
            out[k] = Column.from_host_lazy(HostColumn.from_ints(c.kind, (c.lo + ranks).astype(np.int64)))
    for a in plan:
        col = exact(a.m)
        if a.op == "count":
            out[a.out] = Column.from_host_lazy(HostColumn.from_ints("int64", np.asarray(col, dtype=np.int64)))
        elif a.op in ("min", "max"):
            if a.kind == "float64":
                out[a.out] = Column.from_host_lazy(HostColumn.decimal(np.asarray(col, dtype=np.int64),
                                                                      a.scale))
            else:
                out[a.out] = Column.from_host_lazy(HostColumn.from_ints(a.kind, np.asarray(col, dtype=np.int64)))
        elif a.op == "sum":
            if a.kind == "float64":
                k = decimal_exponent(a.q)
                small = isinstance(col, np.ndarray) and bool((np.abs(col) < (1 << 62)).all())
                if k >= 0 and small:
                    # stays an exact fixed-point decimal (value = int / 10^k)
                    out[a.out] = Column.from_host_lazy(HostColumn.decimal(col, k))
                else:
                    arr = np.asarray([float(Fraction(int(x), a.q)) for x in col], dtype=np.float64)
                    out[a.out] = Column.from_host_lazy(HostColumn("float64", arr, -1))
            else:
                if a.q != 1:
                    raise SchemaError("integer sum with fractional coefficients")
                out[a.out] = Column.from_host_lazy(HostColumn.from_ints("int64", np.asarray(col, dtype=np.int64)))
        else:  # avg = sum / max(count, 1), one correctly rounded division
            cnts = exact(a.cnt)
            den_ok = isinstance(cnts, np.ndarray) and bool((cnts < (1 << 40)).all())
            if (isinstance(col, np.ndarray) and bool((np.abs(col) < (1 << 53)).all()) and den_ok
                    and a.q * (1 << 40) < (1 << 53)):
                arr = col.astype(np.float64) / (np.maximum(cnts, 1) * a.q).astype(np.float64)
            else:
                arr = np.asarray([float(Fraction(int(x), a.q * max(int(n), 1)))
                                  for x, n in zip(col, cnts)], dtype=np.float64)
            out[a.out] = Column.from_host_lazy(HostColumn("float64", arr, -1))
    # keys first, then aggregates (relops.py:121,131-158)
    return ColumnTable(out, tuple(keys))


def _agg_bounds(measures, meta, n_in: int) -> dict:
    """Proven [lo, hi] of each aggregated measure over at most n_in input rows
    (per-row interval x row count): a sort / top-k over the result then packs
    its keys without a min/max pass and the host sync that reads it."""
    out = {}
    for j, (op, im) in enumerate(measures):
        if op == "count":
            out[j] = (0, max(0, n_in))
            continue
        if op != "sum":
            continue
        r = _measure_range(im, meta)
        if r is None:
            continue
        lo, hi = min(0, r[0] * n_in), max(0, r[1] * n_in)
        if INT64_MIN < lo and hi < INT64_MAX:
            out[j] = (lo, hi)
    return out


def _agg_columns(out: dict, plan, measure_col, G: int, bounds: dict | None = None) -> None:
    """Result columns of a keyed aggregation from its per-measure int64
    accumulators (measure_col(j) -> tensor of G values), relops.py:131-158.
    ``bounds``: measure index -> proven [lo, hi] (_agg_bounds)."""
    bounds = bounds or {}
    for a in plan:
        if a.op == "count":
            lo, hi = bounds.get(a.m, (0, INT64_MAX))
            out[a.out] = Column("int64", measure_col(a.m), 0, None, lo, hi)
            out[a.out].loose = a.m in bounds
        elif a.op in ("min", "max"):
            s = a.src
            out[a.out] = Column(s.kind, measure_col(a.m), s.scale, None, s.lo, s.hi)
        elif a.op == "sum":
            k = decimal_exponent(a.q)
            lo, hi = bounds.get(a.m, (INT64_MIN, INT64_MAX))
            if a.kind == "float64":
                if k < 0:
                    raise SchemaError("sum with a non-decimal denominator")
                out[a.out] = Column("float64", measure_col(a.m), k, None, lo, hi)
            else:
                out[a.out] = Column("int64", measure_col(a.m), 0, None, lo, hi)
            out[a.out].loose = a.m in bounds
        else:  # avg
            k = decimal_exponent(a.q)
            if k < 0:
                raise SchemaError("avg with a non-decimal denominator")
            s_col, c_col = measure_col(a.m), measure_col(a.cnt)
            dst = alloc(G, np.float64)
            L.call("scx_fixed_to_f64", _ptr(s_col), 1, G, k, _ptr(c_col), 1, _ptr(dst), _stream())
            out[a.out] = Column("float64", dst, -1, None, 0, -1)


def _column_sorted(c: Column) -> bool:
    """Non-decreasing? Checked once on the device and cached on the column."""
    if c.sorted is None:
        bad = alloc(2, np.int64)
        L.call("scx_is_sorted", C.byref(c.scx()), c.row_count, _ptr(bad), _stream())
        c.sorted = int(_to_host(bad)[0]) == 0
    return bool(c.sorted)


def _stream_group(v: TableView, key: str, kcol: Column, plan, measures, having):
    """Group-by with HAVING over an unfiltered table clustered on `key`
    (scx_sorted_group_agg: each group aggregated by the thread holding its
    first row; no table).  None when the shape does not fit."""
    col = v.base.column(key)
    if not _column_sorted(col):
        return None
    vals, ops = [], []
    n = v.base.row_count
    for op, im in measures:
        if im is None:
            vals.append(col.scx())
            ops.append(L.AGG_COUNT)
            continue
        if im.cond is not None or len(im.terms) != 1:
            return None
        coef, fs = im.terms[0]
        if coef != 1 or len(fs) != 1 or fs[0][0] != 0 or fs[0][1] != 1:
            return None
        name = fs[0][2]
        if v.origin.get(name, ("",))[0] != "base":
            return None
        if op == "sum" and _measure_bound(im, v.meta) * max(n, 1) >= (1 << 62):
            return None
        vals.append(v.meta[name].scx())
        ops.append(_OPCODE[op])
    a = next((a for a in plan if a.out == having[0]), None)
    if a is None or not (a.op == "count" or (a.op == "sum" and a.kind == "int64" and a.q == 1)):
        return None
    M = len(measures)
    varr = (L.Column_ * M)(*vals)
    oarr = (C.c_int * M)(*ops)
    stat = alloc(2, np.int64)
    cnt, ovf = stat[:1], stat[1:].view(_torch().uint32)
    cap = 1 << 16
    while True:
        okeys = alloc(cap, np.int64)
        oacc = alloc(cap * M, np.int64)
        L.call("scx_sorted_group_agg", C.byref(col.scx()), varr, oarr, M, n, a.m, int(having[1]),
               int(having[2]), _ptr(okeys), _ptr(oacc), cap, _ptr(cnt), _ptr(ovf), _stream())
        st = _to_host(stat)
        G = int(st[0])
        if not int(st[1]) & 0xFFFFFFFF:
            break
        cap = G + (G & 1)             # keeps every measure slice 16-byte aligned
    out = {key: Column(kcol.kind, okeys[:G], kcol.scale, kcol.dictionary, kcol.lo, kcol.hi)}
    _agg_columns(out, plan, lambda j: oacc[j * cap: j * cap + G], G,
                 _agg_bounds(measures, v.meta, v.base.row_count))
    return ColumnTable(out, (key,))


def _group_hash(v, b, keys, kcols, plan, measures, count_m, sort=True, hv=None) -> ColumnTable:
    torch = _torch()
    S = b.P.sink
    S.kind = L.SINK_AGG_HASH
    # pack group keys (dict keys by string rank so packed order == output order)
    los, bits, luts = [], [], []
    for i, (k, c) in enumerate(zip(keys, kcols)):
        if c.kind == "dict":
            rank = _rank_lut(c.dictionary)
            luts.append(rank)
            los.append(0)
            bits.append(_bits(len(c.dictionary) - 1))
            S.glut[i] = b.lut(rank)
        else:
            luts.append(None)
            los.append(c.lo if c.hi >= c.lo else 0)
            bits.append(_bits(c.hi - c.lo) if c.hi >= c.lo else 0)
            S.glut[i] = -1
    total = sum(bits)
    if total > 64:
        raise SchemaError(f"group key needs {total} bits (> 64)")
    shifts = []
    acc_bits = 0
    for bb in reversed(bits):
        shifts.append(acc_bits)
        acc_bits += bb
    shifts.reverse()
    S.gkey.n = len(keys)
    for i, k in enumerate(keys):
        S.gkey.slot[i] = b.slot[b.ksrc[i]]
        S.gkey.xform |= _key_xform(v, k) << (8 * i)
        S.gkey.lo[i] = los[i] - _key_offset(v, k)
        S.gkey.bits[i] = bits[i]
        S.gkey.shift[i] = shifts[i]
    # capacity: bounded by rows, the key domain, and unique inner-join builds
    n = v.base.row_count
    bound = max(n, 1)
    # packed-key domain: the leading key contributes its value range, the
    # others their full bit width (packed = k0 << shift0 | ...)
    dom = 1
    for i, (c, bb) in enumerate(zip(kcols, bits)):
        if i == 0:
            rng = len(c.dictionary) if c.kind == "dict" else (c.hi - c.lo + 1 if c.hi >= c.lo else 1)
            dom *= max(1, min(rng, 1 << bb))
        else:
            dom *= (1 << bb)
    bound = min(bound, dom)
    for st in v.probes:
        # a unique-build inner join bounds the groups only when every group
        # key is determined by the matched build row
        if st.kind == L.JOIN_INNER and set(keys) <= set(st.probe_keys) | set(st.payload):
            bound = min(bound, max(st.lookup.table.row_count, 1))
    M = len(measures)
    # dense packed-key domain (TPC-H surrogate keys): direct-addressed groups,
    # slot = packed key, no hashing / CAS (sink.n_cells = 1 marks it)
    filtered = bool(v.probes) or not v.pre.is_true or not v.post.is_true
    if filtered and bound > (1 << 20) and (dom > (1 << 24) or dom > 4 * bound):
        # a large, filtered input whose table would be big: one count pass
        # sizes it to the surviving rows (cheaper than filling and compacting
        # a table sized for the unfiltered input)
        bound = min(bound, max(count_rows(v), 1))
    direct = len(keys) >= 1 and dom <= max(4 * bound, 1 << 16) and dom <= (1 << 31)
    wide = [bool(S.m[j]._pad) for j in range(M)]
    # counts / small non-negative sums fit u32 words: a direct table of half
    # the footprint for the random atomics (Q13: 15M customers -> 60 MB, L2)
    narrow = direct and n < (1 << 32) and not any(wide)
    if narrow:
        for op, im in measures:
            if op == "count":
                continue
            r = _measure_range(im, v.meta) if op == "sum" else None
            if r is None or r[0] < 0 or r[1] * max(n, 1) >= (1 << 32):
                narrow = False
                break
    S.n_cells = 2 if narrow else (1 if direct else 0)
    woff = list(np.cumsum([0] + [2 if w else 1 for w in wide])[:-1])
    W = int(sum(2 if w else 1 for w in wide))          # accumulator words per group
    cap = 1024
    while cap < 2 * bound:
        cap *= 2
    if direct:
        cap = int(dom)
    stat = alloc(4, np.int64)          # [u32 flags x 4][count] -> one D2H per attempt
    flags = stat[:2].view(torch.uint32)
    cnt = stat[2:3].view(torch.uint64)
    while True:
        # direct tables need no key array: the slot is the packed key and the
        # group's count word marks it occupied
        gkeys = None if direct else alloc(cap, np.uint64)
        if gkeys is not None:
            fill_i64(gkeys.view(torch.int64), -1)
        if narrow:
            words = (cap * W + 1) // 2
            acc32 = alloc(words, np.int64)
            fill_i64(acc32, 0)
            S.acc = acc32.data_ptr()
        else:
            accb = alloc(cap * W, np.int64)
            pattern = []
            for j, (op, _) in enumerate(measures):
                pattern.append(INT64_MAX if op == "min" else (INT64_MIN if op == "max" else 0))
                if wide[j]:
                    pattern.append(0)
            pat = (C.c_int64 * W)(*pattern)
            L.call("scx_fill_rows", _ptr(accb), cap, W, pat, _stream())
            S.acc = accb.data_ptr()
        fill_i64(stat, 0)
        S.gkeys = 0 if gkeys is None else gkeys.data_ptr()
        S.gcap, S.flags = cap, flags.data_ptr()
        b.run()
        if narrow:
            accb = alloc(cap * W, np.int64)
            L.call("scx_widen_u32", _ptr(acc32), cap * W, _ptr(accb), _stream())
        out_keys = alloc(cap, np.uint64)
        out_acc = alloc(cap * W, np.int64)
        if direct:
            # slot order == packed-key order: ordered compaction, no sort
            ws = alloc(max(2, L.load().scx_direct_agg_workspace(cap) // 8), np.int64)
            if hv is not None:
                # one unordered pass; the survivors are sorted by key below
                L.call("scx_direct_agg_select_having", _ptr(accb), cap, W, int(woff[count_m]),
                       int(woff[hv[0]]), hv[1], hv[2], _ptr(out_keys), _ptr(out_acc), _ptr(cnt),
                       _stream())
            else:
                L.call("scx_direct_agg_compact_counted", _ptr(accb), cap, W, int(woff[count_m]),
                       _ptr(out_keys), _ptr(out_acc), _ptr(cnt), _ptr(ws), _stream())
        else:
            L.call("scx_hash_agg_compact", _ptr(gkeys), _ptr(accb), cap, W, _ptr(out_keys),
                   _ptr(out_acc), _ptr(cnt), _stream())
        st = _to_host(stat)
        if int(st[0]) & 0xFFFFFFFF == 0:
            break
        if direct or cap >= (1 << 34):
            raise SchemaError("group table overflow (group key outside its proven range)")
        cap *= 4   # table overflowed: rerun with a bigger one
    G = int(st[2])
    if direct and hv is not None:
        skeys, perm = sort_pairs(out_keys[:G], None, total) if G > 1 else (out_keys[:G], None)
    elif direct:
        skeys, perm = out_keys[:G], None
    else:
        if sort:
            # sort groups by packed key (== lexicographic key order)
            skeys, perm = sort_pairs(out_keys[:G], None, total)
        else:     # intermediate (e.g. a join build side): order is irrelevant
            skeys, perm = out_keys[:G], None
    out: dict[str, Column] = {}
    for i, (k, c) in enumerate(zip(keys, kcols)):
        mask = (1 << bits[i]) - 1
        if luts[i] is not None:
            ranks = alloc(G, np.uint32)
            L.call("scx_unpack_key", _ptr(skeys), G, shifts[i], mask, 0,
                   L.Column_(ranks.data_ptr(), L.SCX_U32, 0), _stream())
            inv_t = _inv_rank_tensor(c.dictionary, luts[i], c.np_dtype)
            data = alloc(G, c.np_dtype)
            L.call("scx_gather", L.Column_(inv_t.data_ptr(), c.scx_dtype, 0), _ptr(ranks), G,
                   L.Column_(data.data_ptr(), c.scx_dtype, 0), _stream())
        else:
            data = alloc(G, c.np_dtype)
            L.call("scx_unpack_key", _ptr(skeys), G, shifts[i], mask, los[i],
                   L.Column_(data.data_ptr(), c.scx_dtype, 0), _stream())
        out[k] = c.like(data)

    def word_col(w):
        src = out_acc[w * cap: w * cap + G]
        if perm is None:
            if src.data_ptr() % 16 == 0 and (G * 2 >= cap or cap - G < (1 << 16)):
                return src
            dst = alloc(G, np.int64)
            if G:
                dst.copy_(src)
            return dst
        dst = alloc(G, np.int64)
        L.call("scx_gather", L.Column_(src.data_ptr(), L.SCX_I64, 0), _ptr(perm), G,
               L.Column_(dst.data_ptr(), L.SCX_I64, 0), _stream())
        return dst

    def measure_col(j):
        lo = word_col(int(woff[j]))
        if not wide[j]:
            return lo
        hi = word_col(int(woff[j]) + 1)
        out64 = alloc(G, np.int64)
        flag = alloc(4, np.uint32)
        fill_i64(flag.view(torch.int64), 0)
        L.call("scx_i128_narrow", _ptr(lo), _ptr(hi), G, _ptr(out64), _ptr(flag), _stream())
        if int(_to_host(flag)[0]):
            raise SchemaError("aggregate result exceeds the 64-bit output range")
        return out64

    _agg_columns(out, plan, measure_col, G, _agg_bounds(measures, v.meta, v.base.row_count))
    res = ColumnTable(out, tuple(keys))
    res._having_done = direct and hv is not None
    return res


# ---------------------------------------------------------------------------
# sort / take / head
# ---------------------------------------------------------------------------

def sort_pairs(keys, vals, n_bits: int):
    """Stable radix sort of (u64 key, u32 val); vals=None means iota."""
    n = keys.shape[0]
    if vals is None:
        vals = alloc(n, np.uint32)
        L.call("scx_iota", _ptr(vals), n, _stream())
    ko, vo = alloc(n, np.uint64), alloc(n, np.uint32)
    kt, vt = alloc(n, np.uint64), alloc(n, np.uint32)
    ws = alloc(max(16, L.load().scx_sort_workspace(n)), np.uint8)
    L.call("scx_sort_pairs", _ptr(keys), _ptr(vals), _ptr(ko), _ptr(vo), _ptr(kt), _ptr(vt), n,
           n_bits, _ptr(ws), _stream())
    return ko, vo


def _col_range(c: Column, tight: bool = False) -> tuple[int, int]:
    if c.lo > INT64_MIN and c.hi < INT64_MAX and c.hi >= c.lo and not (tight and c.loose):
        return c.lo, c.hi
    if c.row_count == 0:           # no values (e.g. a worker's empty partition)
        return 0, 0
    mm = alloc(2, np.int64)
    L.call("scx_fill_rows", _ptr(mm), 1, 2, (C.c_int64 * 2)(INT64_MAX, INT64_MIN), _stream())
    L.call("scx_minmax", c.scx(), c.row_count, _ptr(mm), _stream())
    lo, hi = (int(x) for x in _to_host(mm))
    if c.scx_dtype != L.SCX_F64 and hi >= lo:
        # columns are immutable: the measured range replaces the proven one,
        # so later guards / sorts over this column need no second pass + sync
        c.lo, c.hi, c.loose = lo, hi, False
    return lo, hi


_RANK_CACHE: dict = {}


def _rank_tensor(dictionary):
    # keyed by identity (dictionaries are shared canonical tuples; hashing a
    # large one per call is not free) -- the entry keeps the tuple alive
    key = (id(dictionary), _torch().cuda.current_device())
    hit = _RANK_CACHE.get(key)
    if hit is None or hit[0] is not dictionary:
        t = _torch().from_numpy(np.asarray(_rank_lut(dictionary), dtype=np.int32)).to(_device())
        hit = _RANK_CACHE[key] = (dictionary, t)
    return hit[1]


_INV_CACHE: dict = {}


def _inv_rank_tensor(dictionary, lut, np_dtype):
    """rank -> dictionary code, on the device, cached per dictionary."""
    key = (id(dictionary), np.dtype(np_dtype).str, _torch().cuda.current_device())
    hit = _INV_CACHE.get(key)
    if hit is None or hit[0] is not dictionary:
        inv = np.empty(len(lut), dtype=np_dtype)
        for code, r in enumerate(lut):
            inv[r] = code
        hit = _INV_CACHE[key] = (dictionary, _torch().from_numpy(inv).to(_device()))
    return hit[1]


_TOPK_SMALL = 2048          # candidates sorted by the single-CTA sort


def sort_table(t, names: list[str], descending: set[str], limit: int | None = None) -> ColumnTable:
    """Stable multi-key sort (table.py:198-214): LSD over packed 64-bit words.

    ``limit=k`` returns only the first k rows (sort_by(...).head(k)): when the
    key fits one 64-bit word, a radix select (scx_range_hist, one 8-bit digit
    per round) finds a threshold below which only a few rows lie; those are
    compacted in row order (scx_select_below) and sorted, not the whole input.
    """
    t = t.materialize() if isinstance(t, TableView) else t
    n = t.row_count
    if limit is not None and limit <= 0:
        return t.head(0)
    if n <= 1 or not names:
        return t if limit is None else t.head(limit)
    def key_specs(tight: bool):
        out = []
        for name in names:
            c = t.column(name)
            desc = 1 if name in descending else 0
            if c.kind == "dict":
                out.append((c, 0, _bits(len(c.dictionary) - 1), desc, _rank_tensor(c.dictionary)))
            elif c.scx_dtype == L.SCX_F64:
                out.append((c, 0, 64, desc, None))
            else:
                lo, hi = _col_range(c, tight)
                out.append((c, lo, _bits(hi - lo), desc, None))
        return out

    # an aggregate's proven range (rows x per-row range) spares a min/max pass
    # + sync for a full sort, but a top-k's radix select narrows one 8-bit
    # digit per round (one sync each) and needs the key in one 64-bit word:
    # measure loose columns there, and whenever the proven key needs > 64 bits
    specs = key_specs(False)
    loose = any(sp[0].loose for sp in specs)
    if loose and (limit is not None or sum(sp[2] for sp in specs) > 64):
        specs = key_specs(True)
    words, cur, used = [], [], 0
    for sp in reversed(specs):            # least significant key first
        if sp[2] == 0:
            continue
        if used + sp[2] > 64:
            words.append(cur)
            cur, used = [], 0
        cur.append((sp, used))
        used += sp[2]
    if cur:
        words.append(cur)
    top_bits = max(sh + sp[2] for sp, sh in words[-1]) if words else 0
    # the select carries an exclusive upper bound hi = 2^nbits through a u64
    # argument, so a 64-bit most significant word (raw f64 key, or keys that
    # pack to exactly 64 bits) takes the full LSD sort instead
    if limit is not None and n > max(_TOPK_SMALL, 4 * limit) and top_bits < 64:
        # radix select on the MOST significant word; rows tied with the k-th
        # one on it are all kept, then the candidates get the full sort
        word = words[-1]
        nbits = top_bits
        key = alloc(n, np.uint64)
        for i, ((c, lo, bits, desc, lut), sh) in enumerate(word):
            L.call("scx_encode_sort_key", c.scx(), None, n, lo, bits, desc, sh,
                   _ptr(lut) if lut is not None else None, _ptr(key), 1 if i else 0, _stream())
        ckeys, crows = _topk_candidates(key, n, nbits, limit)
        if len(words) == 1:
            _, perm = sort_pairs(ckeys, crows, nbits)
            return take_table(t, perm[:limit])
        perm = crows                       # row order: the LSD passes stay stable
        m = crows.shape[0]
        for word in words:
            nbits = max(sh + sp[2] for sp, sh in word)
            key = alloc(m, np.uint64)
            for i, ((c, lo, bits, desc, lut), sh) in enumerate(word):
                L.call("scx_encode_sort_key", c.scx(), _ptr(perm), m, lo, bits, desc, sh,
                       _ptr(lut) if lut is not None else None, _ptr(key), 1 if i else 0,
                       _stream())
            _, perm = sort_pairs(key, perm, nbits)
        return take_table(t, perm[:limit])
    perm = None
    for word in words:
        nbits = max(sh + sp[2] for sp, sh in word)
        key = alloc(n, np.uint64)
        for i, ((c, lo, bits, desc, lut), sh) in enumerate(word):
            L.call("scx_encode_sort_key", c.scx(), _ptr(perm) if perm is not None else None, n,
                   lo, bits, desc, sh, _ptr(lut) if lut is not None else None, _ptr(key),
                   1 if i else 0, _stream())
        _, perm = sort_pairs(key, perm, nbits)
    if perm is None:
        return t if limit is None else t.head(limit)
    out = take_table(t, perm)
    return out if limit is None else out.head(limit)


def _topk_candidates(key, n: int, nbits: int, k: int):
    """(keys, rows) of every row whose key is < T, in row order, for a
    threshold T found by radix select such that the k smallest keys (and all
    rows tied with the k-th) are among them."""
    counts = alloc(256, np.uint32)
    lo, hi = 0, 1 << nbits              # the k-th key lies in [lo, hi)
    below = 0                           # rows with key < lo
    shift = nbits
    while shift > 0:
        shift = max(shift - 8, 0)
        L.call("scx_range_hist", _ptr(key), n, lo, hi, shift, _ptr(counts), _stream())
        h = _to_host(counts).astype(np.int64)
        cum = below + np.cumsum(h)
        d = int(np.searchsorted(cum, k))          # first digit reaching k rows
        below_d = int(cum[d - 1]) if d else below
        lo, hi = lo + (d << shift), lo + ((d + 1) << shift)
        below = below_d
        if below + int(h[d]) <= _TOPK_SMALL:
            break
    # every row with key < hi: the k smallest are among them
    m_cap = n
    ok, oi = alloc(m_cap, np.uint64), alloc(m_cap, np.uint32)
    cnt = alloc(2, np.int64)
    ws = alloc(max(2, L.load().scx_select_below_workspace(n) // 8), np.int64)
    L.call("scx_select_below", _ptr(key), n, hi, _ptr(ok), _ptr(oi), _ptr(cnt), _ptr(ws), _stream())
    m = int(_to_host(cnt)[0])
    return ok[:m], oi[:m]


def take_column(c: Column, idx) -> Column:
    n = idx.shape[0]
    out = alloc(n, c.np_dtype)
    L.call("scx_gather", c.scx(), _ptr(idx), n, L.Column_(out.data_ptr(), c.scx_dtype, 0),
           _stream())
    return c.like(out)


def take_table(t: ColumnTable, idx) -> ColumnTable:
    torch = _torch()
    if isinstance(idx, np.ndarray):
        idx = torch.from_numpy(idx.astype(np.uint32)).to(_device())
    return ColumnTable({n: take_column(c, idx) for n, c in t.columns.items()})

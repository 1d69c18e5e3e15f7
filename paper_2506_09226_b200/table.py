"""Columnar storage: narrowed host columns and HBM-resident device columns.

Mirrors ``shufflecast.table`` (`/root/reference/pkg/src/shufflecast/table.py`)
-- ``Column``, ``ColumnTable``, ``concat_tables``, ``tables_equal``,
``date_to_days``/``days_to_date``, ``SchemaError`` -- with the same logical
column kinds (int64 / float64 / date32 / dict, table.py:25-30) but a
different physical layout:

* integers and dates are stored in the narrowest signed type that holds
  their [lo, hi] range (checked at load, lossless);
* float64 columns that are exact decimals are stored as fixed-point
  integers with a decimal ``scale`` (value = stored / 10**scale); anything
  else stays physical float64 (scale = -1);
* dictionary codes are uint8 (uint16 above 256 entries).

``ColumnTable.__getitem__`` returns a column *expression* (see expr.py), so
query drivers keep the reference's spelling -- ``li["l_shipdate"] <= d`` --
while predicates compile into the fused scan kernel instead of numpy masks.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from datetime import date, timedelta

import numpy as np

from . import _lib

_EPOCH = date(1970, 1, 1)

KINDS = ("int64", "float64", "date32", "dict")
# reference storage dtype per logical kind (table.py:25-30)
REFERENCE_DTYPES = {"int64": np.int64, "float64": np.float64, "date32": np.int32, "dict": np.int32}

NP_TO_SCX = {
    np.dtype(np.int8): _lib.SCX_I8, np.dtype(np.int16): _lib.SCX_I16,
    np.dtype(np.int32): _lib.SCX_I32, np.dtype(np.int64): _lib.SCX_I64,
    np.dtype(np.uint8): _lib.SCX_U8, np.dtype(np.uint16): _lib.SCX_U16,
    np.dtype(np.float64): _lib.SCX_F64, np.dtype(np.uint32): _lib.SCX_U32,
    np.dtype(np.uint64): _lib.SCX_I64,
}
MAX_DECIMAL_SCALE = 4


class SchemaError(ValueError):
    """Column/type mismatches (table.py:33)."""


def date_to_days(iso: str) -> int:
    y, m, d = iso.split("-")
    return (date(int(y), int(m), int(d)) - _EPOCH).days


def days_to_date(days: int) -> str:
    return (_EPOCH + timedelta(days=int(days))).isoformat()


_U_DT = ((np.dtype(np.uint8), 255), (np.dtype(np.uint16), 65535))
_S_DT = ((np.dtype(np.int8), -128, 127), (np.dtype(np.int16), -32768, 32767),
         (np.dtype(np.int32), -(1 << 31), (1 << 31) - 1),
         (np.dtype(np.int64), -(1 << 63), (1 << 63) - 1))


def narrow_dtype(lo: int, hi: int, unsigned: bool = False) -> np.dtype:
    """Narrowest integer dtype holding [lo, hi] (constant bounds: np.iinfo
    per call was measurable host time for small result columns)."""
    if unsigned and lo >= 0:
        for dt, mx in _U_DT:
            if hi <= mx:
                return dt
    for dt, mn, mx in _S_DT:
        if lo >= mn and hi <= mx:
            return dt
    raise SchemaError(f"integer range [{lo}, {hi}] does not fit int64")


def narrow_host(a: np.ndarray, unsigned: bool = False) -> np.ndarray:
    """Lossless cast of an integer array to its narrowest dtype."""
    a = np.asarray(a)
    if a.size == 0:
        return a.astype(np.int8)
    lo, hi = int(a.min()), int(a.max())
    dt = narrow_dtype(lo, hi, unsigned)
    return a if a.dtype == dt else a.astype(dt)


def _range(a: np.ndarray) -> tuple[int, int]:
    if a.size == 0:
        return 0, -1
    return int(a.min()), int(a.max())


def decimal_scale(v: np.ndarray) -> int:
    """Smallest s <= MAX_DECIMAL_SCALE with v == rint(v*10^s)/10^s bit-exactly, else -1."""
    if v.size == 0:
        return 0
    if not np.all(np.isfinite(v)):
        return -1
    for s in range(MAX_DECIMAL_SCALE + 1):
        p = 10.0 ** s
        ints = np.rint(v * p)
        if np.abs(ints).max() >= 2.0 ** 62:
            return -1
        if np.array_equal(ints / p if s else ints, v):
            return s
    return -1


# ---------------------------------------------------------------------------
# host-side narrowed columns (generator / loader output)
# ---------------------------------------------------------------------------

@dataclass
class HostColumn:
    """Narrowed host column: logical kind + physical numpy storage."""

    kind: str
    values: np.ndarray
    scale: int = 0                       # float64: decimal digits; -1 = raw f64
    dictionary: tuple[str, ...] | None = None
    lo: int = 0
    hi: int = -1
    dense: bool = False                  # row i holds lo + i (a surrogate key column)
    sorted: bool = False                 # non-decreasing by construction (l_orderkey)

    @staticmethod
    def from_ints(kind: str, a: np.ndarray) -> "HostColumn":
        v = narrow_host(a)
        lo, hi = _range(v)
        return HostColumn(kind, v, 0, None, lo, hi)

    @staticmethod
    def int_range(start: int, stop: int) -> "HostColumn":
        dt = narrow_dtype(start, max(start, stop - 1))
        return HostColumn("int64", np.arange(start, stop, dtype=dt), 0, None, start, stop - 1,
                          True, True)

    @staticmethod
    def from_codes(codes: np.ndarray, dictionary: tuple[str, ...]) -> "HostColumn":
        dictionary = tuple(dictionary)
        dt = np.uint8 if len(dictionary) <= 256 else np.uint16
        v = np.asarray(codes).astype(dt)
        lo, hi = _range(v)
        if v.size and (lo < 0 or hi >= len(dictionary)):
            raise SchemaError("dictionary codes out of range")
        return HostColumn("dict", v, 0, dictionary, lo, hi)

    @staticmethod
    def decimal(ints: np.ndarray, scale: int) -> "HostColumn":
        v = narrow_host(ints)
        lo, hi = _range(v)
        return HostColumn("float64", v, scale, None, lo, hi)

    @staticmethod
    def from_float(a: np.ndarray) -> "HostColumn":
        a = np.asarray(a, dtype=np.float64)
        s = decimal_scale(a)
        if s < 0:
            return HostColumn("float64", a, -1, None, 0, -1)
        return HostColumn.decimal(np.rint(a * 10.0 ** s).astype(np.int64), s)

    @staticmethod
    def from_reference(kind: str, values: np.ndarray, dictionary=None) -> "HostColumn":
        """Narrow a reference-typed column (Column(kind, values, dictionary))."""
        if kind not in KINDS:
            raise SchemaError(f"unknown column kind {kind!r}")
        if kind == "dict":
            if dictionary is None:
                raise SchemaError("dict column requires a dictionary")
            return HostColumn.from_codes(values, dictionary)
        if dictionary is not None:
            raise SchemaError(f"{kind} column must not carry a dictionary")
        if kind == "float64":
            return HostColumn.from_float(values)
        return HostColumn.from_ints(kind, np.asarray(values).astype(np.int64))

    @property
    def row_count(self) -> int:
        return len(self.values)

    @property
    def nbytes(self) -> int:
        return int(self.values.nbytes)

    def take(self, idx: np.ndarray) -> "HostColumn":
        idx = np.asarray(idx)
        # a sorted column stays sorted under an increasing row selection
        # (partition_rows / row ranges keep input order)
        keep = bool(self.sorted and (idx.dtype == bool or idx.size < 2
                                     or bool(np.all(idx[1:] > idx[:-1]))))
        return HostColumn(self.kind, self.values[idx], self.scale, self.dictionary, self.lo,
                          self.hi, False, keep)

    def to_int64(self) -> np.ndarray:
        return self.values.astype(np.int64)

    def to_reference(self) -> tuple:
        """(kind, values in the reference dtype, dictionary) -- widening copy."""
        if self.kind == "float64":
            if self.scale < 0:
                vals = self.values.astype(np.float64)
            elif self.scale == 0:
                vals = self.values.astype(np.float64)
            else:
                vals = self.values.astype(np.int64) / float(10 ** self.scale)
        else:
            vals = self.values.astype(REFERENCE_DTYPES[self.kind])
        return (self.kind, vals, self.dictionary)


class HostTable:
    """Equal-length named host columns (narrowed)."""

    def __init__(self, columns: dict[str, HostColumn]):
        lengths = {c.row_count for c in columns.values()}
        if len(lengths) > 1:
            raise SchemaError(f"ragged columns: { {n: c.row_count for n, c in columns.items()} }")
        self.columns = dict(columns)
        self.row_count = lengths.pop() if lengths else 0

    @property
    def column_names(self) -> list[str]:
        return list(self.columns)

    @property
    def nbytes(self) -> int:
        return sum(c.nbytes for c in self.columns.values())

    def column(self, name: str) -> HostColumn:
        try:
            return self.columns[name]
        except KeyError:
            raise SchemaError(f"unknown column {name!r}; have {self.column_names}") from None

    def take(self, idx: np.ndarray) -> "HostTable":
        return HostTable({n: c.take(idx) for n, c in self.columns.items()})

    def select(self, names: list[str]) -> "HostTable":
        return HostTable({n: self.column(n) for n in names})

    def to_reference(self) -> dict[str, tuple]:
        return {n: c.to_reference() for n, c in self.columns.items()}

    def to_device(self, device=None) -> "ColumnTable":
        return ColumnTable({n: Column.from_host(c, device) for n, c in self.columns.items()})


# ---------------------------------------------------------------------------
# device columns
# ---------------------------------------------------------------------------

def _torch():
    import torch
    return torch


_TORCH_DTYPE = None
_NP_OF_TORCH: dict = {}


def torch_dtype(np_dtype: np.dtype):
    torch = _torch()
    global _TORCH_DTYPE
    if _TORCH_DTYPE is None:
        _TORCH_DTYPE = {
            np.dtype(np.int8): torch.int8, np.dtype(np.int16): torch.int16,
            np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64,
            np.dtype(np.uint8): torch.uint8, np.dtype(np.uint16): torch.uint16,
            np.dtype(np.float64): torch.float64, np.dtype(np.uint32): torch.uint32,
            np.dtype(np.uint64): torch.uint64,
        }
    return _TORCH_DTYPE[np.dtype(np_dtype)]


def alloc(n: int, np_dtype, device=None):
    """Device buffer of n elements, padded to a 16-byte multiple (TMA bulk
    copies read whole 16-byte granules at the tail)."""
    torch = _torch()
    itemsize = np.dtype(np_dtype).itemsize
    pad = (-(n * itemsize)) % 16 // itemsize + (16 // itemsize if n == 0 else 0)
    buf = torch.empty(n + pad, dtype=torch_dtype(np_dtype), device=device or "cuda")
    return buf[:n] if pad else buf


_MAPPED_OK = os.environ.get("SCX_MAPPED_READS", "1") != "0"
_MAPPED_MAX = 1 << 20


def to_host(t) -> np.ndarray:
    """D2H read of a device tensor into a pinned (cached) host buffer on the
    current stream: up to 1 MB by a kernel storing into the mapped buffer
    (scx_write_mapped, no copy engine), larger reads by an async copy.  A
    pageable ``.cpu()`` copy -- and any copy-engine D2H -- queued behind the
    in-flight H2D transfers of an asynchronous upload
    (engine.upload_tables_async): a query whose columns had landed at 72 ms
    read its result at 106 ms.  SCX_MAPPED_READS=0 keeps the copy path."""
    global _MAPPED_OK
    torch = _torch()
    if t.numel() == 0 or not t.is_cuda:
        return t.cpu().numpy()
    t = t.contiguous()
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    nb = t.numel() * t.element_size()
    done = False
    if _MAPPED_OK and nb <= _MAPPED_MAX:
        # small reads: a kernel stores into the mapped pinned buffer, no copy
        # engine (scx_write_mapped)
        try:
            _lib.call("scx_write_mapped", t.data_ptr(), h.data_ptr(), nb, _lib.stream_ptr())
            done = True
        except _lib.ScxError:
            _MAPPED_OK = False
    if not done:
        h.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return h.numpy()


class Column:
    """Device-resident column (mirror of table.py:46-85).

    ``data`` is a torch tensor on the GPU in the narrowed physical dtype;
    ``kind``/``dictionary`` keep the reference's logical meaning and
    ``scale`` the fixed-point exponent of float64 columns.
    """

    __slots__ = ("kind", "_data", "_host", "scale", "dictionary", "lo", "hi", "dense", "sorted",
                 "loose", "_ready")

    def __init__(self, kind: str, data, scale: int = 0, dictionary=None, lo: int = 0,
                 hi: int = -1, dense: bool = False):
        if data is not None and not hasattr(data, "data_ptr"):
            # the reference's call shape Column(kind, values, dictionary=None)
            # (table.py:46-60): reference-typed host values, narrowed losslessly
            # and uploaded
            if isinstance(scale, (tuple, list)):
                dictionary, scale = scale, 0
            src = Column.from_numpy(kind, data, dictionary)
            for slot in Column.__slots__:
                setattr(self, slot, getattr(src, slot))
            return
        if kind not in KINDS:
            raise SchemaError(f"unknown column kind {kind!r}")
        if kind == "dict" and dictionary is None:
            raise SchemaError("dict column requires a dictionary")
        if kind != "dict" and dictionary is not None:
            raise SchemaError(f"{kind} column must not carry a dictionary")
        self.kind = kind
        self._data = data
        self._host = None      # host copy of a small result column (uploaded lazily)
        self.scale = scale
        self.dictionary = tuple(dictionary) if dictionary is not None else None
        self.lo = lo
        self.hi = hi
        # row i holds lo + i: a join on this column needs no lookup table
        # (row = key - lo), see relops.Lookup
        self.dense = dense
        # non-decreasing in row order: None = not yet checked (relops checks
        # it on the device when a group-by could use dense ranks)
        self.sorted = True if dense else None
        # [lo, hi] proven but loose (an aggregate: rows x per-row range):
        # overflow guards measure the values instead (relops._col_range)
        self.loose = False
        # (CUDA event, waited stream handles) of an asynchronous upload
        # (engine.upload_tables_async): the first access to ``data`` from a
        # stream makes that stream wait for this column's copy -- a query waits
        # for the columns it reads, not for whole tables
        self._ready = None

    def set_ready(self, event) -> None:
        self._ready = (event, set())

    @property
    def data(self):
        """Device tensor (uploaded on first use for host-backed result columns)."""
        if self._ready is not None:
            ev, waited = self._ready
            h = _lib.stream_ptr().value or 0
            if h not in waited:
                _torch().cuda.current_stream().wait_event(ev)
                waited.add(h)
        if self._data is None:
            torch = _torch()
            n = len(self._host)
            buf = alloc(n, self._host.dtype)
            if n:
                buf.copy_(torch.from_numpy(np.ascontiguousarray(self._host)), non_blocking=False)
            self._data = buf
        return self._data

    @data.setter
    def data(self, v):
        self._data = v
        self._host = None

    # ---- construction ----
    @staticmethod
    def from_host_lazy(hc: HostColumn) -> "Column":
        """A small (final-aggregation) result column that stays on the host
        until a kernel needs it: no H2D copy (and no D2H later) for results
        that are only read back."""
        c = Column(hc.kind, None, hc.scale, hc.dictionary, hc.lo, hc.hi,
                   hc.dense and hc.row_count == hc.hi - hc.lo + 1)
        c._host = np.ascontiguousarray(hc.values)
        if hc.sorted:
            c.sorted = True
        return c

    @staticmethod
    def from_host(hc: HostColumn, device=None) -> "Column":
        torch = _torch()
        n = hc.row_count
        buf = alloc(n, hc.values.dtype, device)
        if n:
            v = np.ascontiguousarray(hc.values)
            src = torch.from_numpy(v if v.flags.writeable else v.copy())
            buf.copy_(src, non_blocking=False)
        c = Column(hc.kind, buf, hc.scale, hc.dictionary, hc.lo, hc.hi,
                   hc.dense and n == hc.hi - hc.lo + 1)
        if hc.sorted:
            c.sorted = True
        return c

    @staticmethod
    def from_numpy(kind: str, values, dictionary=None, device=None) -> "Column":
        """Narrow + upload a reference-typed array (Column(kind, values, dictionary))."""
        return Column.from_host(HostColumn.from_reference(kind, np.asarray(values), dictionary),
                                device)

    # ---- properties ----
    @property
    def np_dtype(self) -> np.dtype:
        if self._data is None:
            return self._host.dtype
        td = self._data.dtype
        nd = _NP_OF_TORCH.get(td)
        if nd is None:
            nd = _NP_OF_TORCH[td] = np.dtype(str(td).replace("torch.", ""))
        return nd

    @property
    def scx_dtype(self) -> int:
        return NP_TO_SCX[self.np_dtype]

    @property
    def row_count(self) -> int:
        if self._data is None:
            return len(self._host)
        return int(self._data.shape[0])

    def __len__(self) -> int:
        return self.row_count

    @property
    def nbytes(self) -> int:
        return self.row_count * self.itemsize

    @property
    def itemsize(self) -> int:
        if self._data is None:
            return self._host.dtype.itemsize
        return self._data.element_size()

    @property
    def is_fixed(self) -> bool:
        return self.kind == "float64" and self.scale >= 0

    def scx(self) -> _lib.Column_:
        return _lib.Column_(self.data.data_ptr(), self.scx_dtype, 0)

    def like(self, data, lo=None, hi=None) -> "Column":
        c = Column(self.kind, data, self.scale, self.dictionary,
                   self.lo if lo is None else lo, self.hi if hi is None else hi)
        c.loose = self.loose and lo is None and hi is None
        return c

    # ---- host views (D2H; inspection / result decoding) ----
    def host(self) -> np.ndarray:
        """Physical values on the host."""
        if self._host is not None:
            return self._host
        return to_host(self.data)

    @property
    def values(self) -> np.ndarray:
        """Values in the reference dtype (table.py:25-30), copied to the host."""
        return HostColumn(self.kind, self.host(), self.scale, self.dictionary).to_reference()[1]

    def decoded(self) -> np.ndarray:
        """Strings for dict columns, ISO dates for date32, values otherwise (table.py:79-85)."""
        v = self.values
        if self.kind == "dict":
            return np.asarray(self.dictionary, dtype=object)[v]
        if self.kind == "date32":
            return np.asarray([days_to_date(d) for d in v], dtype=object)
        return v

    def take(self, idx) -> "Column":
        from . import relops
        return relops.take_column(self, idx)

    def __repr__(self) -> str:
        return (f"Column({self.kind}, {self.np_dtype}, rows={self.row_count}, scale={self.scale}, "
                f"range=[{self.lo},{self.hi}])")


class ColumnTable:
    """Immutable named device columns of equal length (table.py:119-217)."""

    def __init__(self, columns: dict[str, Column], unique_keys: tuple = ()):
        lengths = {c.row_count for c in columns.values()}
        if len(lengths) > 1:
            raise SchemaError(f"ragged columns: { {n: c.row_count for n, c in columns.items()} }")
        self._columns = dict(columns)
        self._rows = lengths.pop() if lengths else 0
        # column set known to be a key (group-by output): a join building on
        # it needs no duplicate check (relops.Lookup)
        self.unique_keys = tuple(unique_keys) if set(unique_keys) <= set(columns) else ()

    # ---- reference surface ----
    @property
    def row_count(self) -> int:
        return self._rows

    @property
    def column_names(self) -> list[str]:
        return list(self._columns)

    @property
    def columns(self) -> dict[str, Column]:
        return self._columns

    @property
    def nbytes(self) -> int:
        return sum(c.nbytes for c in self._columns.values())

    def column(self, name: str) -> Column:
        try:
            return self._columns[name]
        except KeyError:
            raise SchemaError(f"unknown column {name!r}; have {self.column_names}") from None

    def __getitem__(self, name: str):
        from .expr import ColRef
        self.column(name)
        return ColRef(name, self.column(name))

    def __contains__(self, name: str) -> bool:
        return name in self._columns

    def schema(self) -> dict[str, str]:
        return {n: c.kind for n, c in self._columns.items()}

    def select(self, names: list[str]) -> "ColumnTable":
        return ColumnTable({n: self.column(n) for n in names}, self.unique_keys)

    def with_column(self, name: str, col: Column) -> "ColumnTable":
        cols = dict(self._columns)
        cols[name] = col
        return ColumnTable(cols, self.unique_keys if name not in self.unique_keys else ())

    def rename(self, mapping: dict[str, str]) -> "ColumnTable":
        return ColumnTable({mapping.get(n, n): c for n, c in self._columns.items()},
                           tuple(mapping.get(k, k) for k in self.unique_keys))

    def take(self, idx) -> "ColumnTable":
        from . import relops
        return relops.take_table(self, idx)

    def filter(self, mask) -> "ColumnTable":
        from . import relops
        return relops.filter_table(self, mask).materialize()

    def head(self, n: int) -> "ColumnTable":
        n = max(0, min(n, self._rows))
        return ColumnTable({k: c.like(c.data[:n]) for k, c in self._columns.items()},
                           self.unique_keys)

    def isin(self, name: str, values: list[str]):
        from .expr import isin
        return isin(self[name], values)

    def sort_by(self, names: list[str], descending: set[str] | None = None) -> "ColumnTable":
        from . import relops
        return relops.sort_table(self, names, descending or set())

    def top(self, names: list[str], descending: set[str] | None, n: int) -> "ColumnTable":
        """sort_by(names, descending).head(n) without sorting the whole table
        (extension; same rows in the same order)."""
        from . import relops
        return relops.sort_table(self, names, descending or set(), limit=n)

    def decode_rows(self) -> list[tuple]:
        cols = [c.decoded() for c in self._columns.values()]
        return [tuple(col[i] for col in cols) for i in range(self._rows)]

    def to_reference(self) -> dict[str, tuple]:
        """{name: (kind, reference-dtype values, dictionary)} on the host."""
        return {n: (c.kind, c.values, c.dictionary) for n, c in self._columns.items()}

    def materialize(self) -> "ColumnTable":
        return self

    def __repr__(self) -> str:
        return f"ColumnTable({self.schema()}, rows={self._rows})"


def concat_tables(tables: list[ColumnTable]) -> ColumnTable:
    """Row-wise concatenation; schemas and dictionaries must agree (table.py:220-239)."""
    torch = _torch()
    tables = [t.materialize() for t in tables]
    if not tables:
        raise SchemaError("cannot concatenate zero tables")
    first = tables[0]
    for t in tables[1:]:
        if t.schema() != first.schema():
            raise SchemaError(f"schema mismatch: {t.schema()} vs {first.schema()}")
    out = {}
    for name, col in first.columns.items():
        parts = [t.column(name) for t in tables]
        if col.kind == "dict" and len({p.dictionary for p in parts}) > 1:
            raise SchemaError(f"column {name!r} has diverging dictionaries")
        if len({p.scale for p in parts}) > 1 or len({p.np_dtype for p in parts}) > 1:
            parts = [unify_physical(p, parts) for p in parts]
        n = sum(p.row_count for p in parts)
        buf = alloc(n, parts[0].np_dtype, col.data.device)
        off = 0
        for p in parts:
            if p.row_count:
                buf[off:off + p.row_count].copy_(p.data)   # D2D memcpy
            off += p.row_count
        lo = min((p.lo for p in parts if p.row_count), default=0)
        hi = max((p.hi for p in parts if p.row_count), default=-1)
        out[name] = Column(col.kind, buf, parts[0].scale, col.dictionary, lo, hi)
    return ColumnTable(out)


def unify_physical(p: Column, parts: list[Column]) -> Column:
    """Bring one part to the widest dtype / largest scale of `parts` (host-side
    metadata decision; the data conversion is a D2D cast)."""
    scale = max(q.scale for q in parts)
    if any(q.scale < 0 for q in parts):
        raise SchemaError("cannot concatenate raw float64 with fixed-point parts")
    # target dtype from the union of the parts' rescaled value ranges: picking
    # by byte width alone would wrap a u8/u32 part cast to i8/i32
    ranges = [(q.lo * 10 ** (scale - q.scale), q.hi * 10 ** (scale - q.scale))
              for q in parts if q.hi >= q.lo]
    lo_all = min((a for a, _ in ranges), default=0)
    hi_all = max((b for _, b in ranges), default=0)
    dt = narrow_dtype(lo_all, hi_all, unsigned=all(np.dtype(q.np_dtype).kind == "u"
                                                   for q in parts))
    data = p.data.to(torch_dtype(dt))
    if scale != p.scale:
        data = data * (10 ** (scale - p.scale))
    mult = 10 ** (scale - p.scale)
    return Column(p.kind, data, scale, p.dictionary, p.lo * mult, p.hi * mult)


def tables_equal(a: ColumnTable, b: ColumnTable) -> bool:
    a, b = a.materialize(), b.materialize()
    if a.schema() != b.schema() or a.row_count != b.row_count:
        return False
    for name, col in a.columns.items():
        other = b.column(name)
        if col.kind == "dict" and col.dictionary != other.dictionary:
            return False
        if not np.array_equal(col.values, other.values):
            return False
    return True


# ---- constructors of the reference's package namespace (__init__.py:86-112)

def int64_col(values) -> Column:
    return Column("int64", np.asarray(values, dtype=np.int64))


def float64_col(values) -> Column:
    return Column("float64", np.asarray(values, dtype=np.float64))


def date32_col(values) -> Column:
    return Column("date32", np.asarray(values, dtype=np.int32))


def dict_col(codes, dictionary) -> Column:
    return Column("dict", np.asarray(codes, dtype=np.int32), tuple(dictionary))


def dict_col_from_strings(strings) -> Column:
    """Encode strings with a first-seen-order dictionary."""
    index: dict[str, int] = {}
    codes = np.empty(len(strings), dtype=np.int32)
    for i, sv in enumerate(strings):
        codes[i] = index.setdefault(sv, len(index))
    return Column("dict", codes, tuple(index))

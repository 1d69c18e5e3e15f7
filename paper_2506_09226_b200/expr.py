"""Predicate and measure expressions for the fused scan kernel.

The reference's query drivers build numpy masks and float64 arrays directly
from columns (`queries.py:39,45-50,110-115,131-135,173-180,209-234`;
``ColumnTable.isin``, `table.py:185-192`; ``_codes_where``,
`queries.py:23-29`).  Here the same spelling builds *expressions*:

* comparisons / ``isin`` / ``codes_where`` / ``&`` / ``|`` / ``~`` build a
  predicate in disjunctive normal form whose atoms are integer range tests
  on the narrowed physical values, dictionary-set bitmap tests, or
  column-difference tests (``cd < rd``).  Float literals against fixed-point
  decimal columns are converted to the exact integer bound that reproduces
  the reference's float64 comparison (``fl(v / 10^s) >= c``), so the row set
  is identical, not approximately equal;
* ``+ - *`` over columns and literals build an exact rational polynomial
  (sum of products of affine factors) that the kernel evaluates in 64-bit
  fixed point; ``where(pred, x, 0)`` gates a measure by one atom.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from fractions import Fraction

from .table import Column, SchemaError

INT64_MIN = -(1 << 63)
INT64_MAX = (1 << 63) - 1


def _frac(c) -> Fraction:
    if isinstance(c, Fraction):
        return c
    if isinstance(c, bool):
        return Fraction(int(c))
    if isinstance(c, int):
        return Fraction(c)
    if isinstance(c, float):
        if not math.isfinite(c):
            raise SchemaError(f"non-finite literal {c!r}")
        return Fraction(repr(c))     # decimal meaning of the literal (0.05 -> 1/20)
    try:
        import numpy as np
        if isinstance(c, np.integer):
            return Fraction(int(c))
        if isinstance(c, np.floating):
            return Fraction(repr(float(c)))
    except ImportError:  # pragma: no cover
        pass
    raise SchemaError(f"unsupported literal {c!r}")


# ---------------------------------------------------------------------------
# predicates
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Atom:
    op: str                      # "range" | "set" | "diff" | "poly"
    col: str
    lo: int = INT64_MIN
    hi: int = INT64_MAX
    col2: str | None = None      # diff: value = col - col2
    codes: frozenset = frozenset()  # set: dictionary codes that pass
    negate: bool = False
    poly: "Poly | None" = field(default=None, compare=False)  # poly: lo <= int form <= hi
    poly_key: str = ""           # identity of `poly` for atom equality / hashing

    def inverted(self) -> "Atom":
        return replace(self, negate=not self.negate)

    @property
    def columns(self) -> tuple[str, ...]:
        if self.op == "poly":
            return tuple(sorted(self.poly.columns))
        return (self.col,) if self.col2 is None else (self.col, self.col2)


class Pred:
    """DNF: OR over clauses, each clause an AND of atoms.  [] clauses = FALSE,
    [()] = TRUE."""

    __slots__ = ("clauses",)

    def __init__(self, clauses):
        self.clauses = tuple(tuple(c) for c in clauses)
        if len(self.clauses) > 32:
            raise SchemaError("predicate has more than 32 DNF clauses")

    @staticmethod
    def true() -> "Pred":
        return Pred([()])

    @staticmethod
    def false() -> "Pred":
        return Pred([])

    @staticmethod
    def atom(a: Atom) -> "Pred":
        return Pred([(a,)])

    @property
    def is_true(self) -> bool:
        return any(len(c) == 0 for c in self.clauses)

    @property
    def columns(self) -> set[str]:
        return {n for c in self.clauses for a in c for n in a.columns}

    def __and__(self, other) -> "Pred":
        other = as_pred(other)
        return Pred([a + b for a in self.clauses for b in other.clauses])

    __rand__ = __and__

    def __or__(self, other) -> "Pred":
        other = as_pred(other)
        if self.is_true or other.is_true:
            return Pred.true()
        return Pred(self.clauses + other.clauses)

    __ror__ = __or__

    def __invert__(self) -> "Pred":
        if not self.clauses:
            return Pred.true()
        if len(self.clauses) == 1:
            (clause,) = self.clauses
            if not clause:
                return Pred.false()
            return Pred([(a.inverted(),) for a in clause])
        if all(len(c) == 1 for c in self.clauses):
            return Pred([tuple(c[0].inverted() for c in self.clauses)])
        raise SchemaError("negation of a multi-clause predicate is not supported")

    def single_atom(self) -> Atom:
        if len(self.clauses) == 1 and len(self.clauses[0]) == 1:
            return self.clauses[0][0]
        raise SchemaError("a measure condition must be a single comparison / set test")

    def __bool__(self):
        raise TypeError("a Pred is evaluated on the GPU; use it in q.filter / where()")

    def __repr__(self) -> str:
        return f"Pred({self.clauses})"


def as_pred(x) -> Pred:
    if isinstance(x, Pred):
        return x
    if isinstance(x, bool):
        return Pred.true() if x else Pred.false()
    raise SchemaError(f"cannot use {type(x).__name__} as a predicate")


# ---------------------------------------------------------------------------
# arithmetic: rational polynomial over columns (logical units)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Factor:
    a: Fraction
    b: Fraction
    col: str          # value = a + b * logical(col)


@dataclass(frozen=True)
class Term:
    coef: Fraction
    factors: tuple[Factor, ...] = ()


def _poly_cmp(left, right, op: str) -> Pred:
    """Exact comparison of two polynomials: (left - right) op 0.  The kernel
    evaluates the integerised difference (a positive multiple of it), so the
    sign -- and therefore the comparison -- is exact."""
    d = as_poly(left) - as_poly(right)
    if d.cond is not None:
        raise SchemaError("cannot compare a conditional measure")
    if not d.columns:
        raise SchemaError("comparison of two constants")
    rng = {">=": (0, INT64_MAX), ">": (1, INT64_MAX), "<": (INT64_MIN, -1),
           "<=": (INT64_MIN, 0), "==": (0, 0), "!=": (0, 0)}[op]
    return Pred.atom(Atom("poly", "", rng[0], rng[1], negate=(op == "!="), poly=d,
                          poly_key=repr(d.terms)))


@dataclass(frozen=True, eq=False)
class Poly:
    terms: tuple[Term, ...]
    cond: Atom | None = None
    integral: bool = True     # all inputs integer-kind and coefficients integral

    @property
    def columns(self) -> set[str]:
        cols = {f.col for t in self.terms for f in t.factors}
        if self.cond is not None:
            cols |= set(self.cond.columns)
        return cols

    def _combine(self, other, sign=1) -> "Poly":
        o = as_poly(other)
        if self.cond is not None or o.cond is not None:
            raise SchemaError("cannot add conditional measures")
        terms = self.terms + tuple(Term(t.coef * sign, t.factors) for t in o.terms)
        return _collapse(Poly(terms, None, self.integral and o.integral))

    def __add__(self, other):
        return self._combine(other)

    __radd__ = __add__

    def __sub__(self, other):
        return self._combine(other, -1)

    def __rsub__(self, other):
        return as_poly(other)._combine(self, -1)

    def __neg__(self):
        return Poly(tuple(Term(-t.coef, t.factors) for t in self.terms), self.cond, self.integral)

    def __mul__(self, other):
        o = as_poly(other)
        if self.cond is not None or o.cond is not None:
            raise SchemaError("cannot multiply conditional measures")
        terms = tuple(Term(a.coef * b.coef, a.factors + b.factors)
                      for a in self.terms for b in o.terms)
        return _collapse(Poly(terms, None, self.integral and o.integral))

    __rmul__ = __mul__

    def sum(self):
        return self

    # comparisons build predicates (SQL-style `qty * 5 * cnt < sum_qty`)
    def __lt__(self, o): return _poly_cmp(self, o, "<")
    def __le__(self, o): return _poly_cmp(self, o, "<=")
    def __gt__(self, o): return _poly_cmp(self, o, ">")
    def __ge__(self, o): return _poly_cmp(self, o, ">=")
    def __eq__(self, o): return _poly_cmp(self, o, "==")
    def __ne__(self, o): return _poly_cmp(self, o, "!=")
    __hash__ = object.__hash__

    def __repr__(self) -> str:
        return f"Poly({self.terms}, cond={self.cond})"


def _collapse(p: Poly) -> Poly:
    """Merge constants; fold `c + k*x` (one column, all terms <= 1 factor)
    into one affine factor so `1 - disc` costs one factor, not two terms."""
    const = sum((t.coef for t in p.terms if not t.factors), Fraction(0))
    lin = [t for t in p.terms if t.factors]
    if all(len(t.factors) == 1 for t in lin) and len({t.factors[0].col for t in lin}) == 1 and lin:
        col = lin[0].factors[0].col
        a = const + sum(t.coef * t.factors[0].a for t in lin)
        b = sum(t.coef * t.factors[0].b for t in lin)
        if b == 0:
            return Poly((Term(a),), p.cond, p.integral)
        if a == 0:
            return Poly((Term(b, (Factor(Fraction(0), Fraction(1), col),)),), p.cond, p.integral)
        return Poly((Term(Fraction(1), (Factor(a, b, col),)),), p.cond, p.integral)
    terms = tuple(lin) + ((Term(const),) if const != 0 or not lin else ())
    return Poly(terms, p.cond, p.integral)


def as_poly(x) -> Poly:
    if isinstance(x, Poly):
        return x
    if isinstance(x, ColRef):
        return x.poly()
    f = _frac(x)
    return Poly((Term(f),), None, f.denominator == 1)


def where(cond, then, otherwise=0) -> Poly:
    """``np.where(cond, x, 0)`` (queries.py:182): measure gated by one atom."""
    if _frac(otherwise) != 0:
        raise SchemaError("where(): only a zero 'otherwise' branch is supported")
    p = as_poly(then)
    if p.cond is not None:
        raise SchemaError("where(): nested conditions are not supported")
    return Poly(p.terms, as_pred(cond).single_atom(), p.integral)


# ---------------------------------------------------------------------------
# column references
# ---------------------------------------------------------------------------

def _float_bound(scale: int, c: float, strict: bool) -> int:
    """min integer v with fl(v / 10^scale) >= c (or > c if strict)."""
    p = 10 ** scale
    div = float(p)

    def f(v):
        return float(v) / div if scale else float(v)

    v = math.floor(c * p) - 2
    while (f(v) > c) if strict else (f(v) >= c):
        v -= 4
    while not ((f(v) > c) if strict else (f(v) >= c)):
        v += 1
    return v


class ColRef:
    """``table["name"]`` -- a column usable in predicates and measures, and
    (via ``values``/``__array__``) as a host array for inspection."""

    __slots__ = ("name", "col")

    def __init__(self, name: str, col: Column):
        self.name = name
        self.col = col

    # ---- host view (compatibility with numpy-style inspection) ----
    @property
    def values(self):
        return self.col.values

    def __array__(self, dtype=None, copy=None):
        v = self.col.values
        return v.astype(dtype) if dtype is not None else v

    def __len__(self):
        return self.col.row_count

    # ---- arithmetic ----
    def poly(self) -> Poly:
        c = self.col
        if c.kind == "dict":
            raise SchemaError(f"arithmetic on dict column {self.name!r}")
        if c.kind == "float64":
            if c.scale < 0:
                raise SchemaError(f"column {self.name!r} is raw float64; only fixed-point "
                                  "decimals are supported in fused measures")
            return Poly((Term(Fraction(1), (Factor(Fraction(0), Fraction(1), self.name),)),),
                        None, False)
        return Poly((Term(Fraction(1), (Factor(Fraction(0), Fraction(1), self.name),)),), None, True)

    def astype(self, dtype):
        """``col.astype(np.float64)`` (queries.py:48): same values, float64 kind."""
        p = self.poly()
        if "float" in str(dtype):
            return Poly(p.terms, None, False)
        return p

    def __add__(self, o): return self.poly() + o
    def __radd__(self, o): return as_poly(o) + self.poly()
    def __sub__(self, o): return self.poly() - o
    def __rsub__(self, o): return as_poly(o) - self.poly()
    def __mul__(self, o): return self.poly() * o
    def __rmul__(self, o): return as_poly(o) * self.poly()
    def __neg__(self): return -self.poly()

    def sum(self):
        return self.poly()

    # ---- comparisons ----
    def _cmp(self, other, op: str) -> Pred:
        if isinstance(other, Poly):
            return _poly_cmp(self.poly(), other, op)
        if isinstance(other, ColRef):
            if (self.col.kind == "float64" and other.col.kind == "float64"
                    and self.col.scale != other.col.scale):
                return _poly_cmp(self.poly(), other.poly(), op)
            return self._cmp_col(other, op)
        c = self.col
        if c.kind == "dict":
            raise SchemaError(f"compare dict column {self.name!r} with isin(), not {op}")
        if c.kind == "float64" and c.scale < 0:
            raise SchemaError(f"predicate on raw float64 column {self.name!r}")
        if c.kind == "float64" and c.scale > 0 and isinstance(other, (Fraction, int)) \
                and not isinstance(other, bool):
            # exact rational literal (e.g. an aggregate read back from the device):
            # compare the fixed-point integer exactly
            x = _frac(other) * (10 ** c.scale)
            fl, ce = math.floor(x), math.ceil(x)
            rng = {">=": (ce, INT64_MAX), ">": (fl + 1, INT64_MAX), "<": (INT64_MIN, ce - 1),
                   "<=": (INT64_MIN, fl), "==": (ce, fl), "!=": (ce, fl)}[op]
        elif c.kind == "float64" and c.scale > 0:
            x = float(other)
            ge = _float_bound(c.scale, x, strict=False)   # first v with f(v) >= x
            gt = _float_bound(c.scale, x, strict=True)    # first v with f(v) >  x
            rng = {">=": (ge, INT64_MAX), ">": (gt, INT64_MAX), "<": (INT64_MIN, ge - 1),
                   "<=": (INT64_MIN, gt - 1), "==": (ge, gt - 1), "!=": (ge, gt - 1)}[op]
        else:
            x = _frac(other)
            fl, ce = math.floor(x), math.ceil(x)
            rng = {">=": (ce, INT64_MAX), ">": (fl + 1, INT64_MAX), "<": (INT64_MIN, ce - 1),
                   "<=": (INT64_MIN, fl), "==": (ce, fl), "!=": (ce, fl)}[op]
        lo, hi = rng
        a = Atom("range", self.name, max(lo, INT64_MIN), min(hi, INT64_MAX), negate=(op == "!="))
        return Pred.atom(a)

    def _cmp_col(self, other: "ColRef", op: str) -> Pred:
        a, b = self.col, other.col
        if a.kind != b.kind or a.kind == "dict" or (a.kind == "float64" and a.scale != b.scale):
            raise SchemaError(f"cannot compare {self.name!r} with {other.name!r}")
        # self op other  <=>  (self - other) op 0
        rng = {">=": (0, INT64_MAX), ">": (1, INT64_MAX), "<": (INT64_MIN, -1),
               "<=": (INT64_MIN, 0), "==": (0, 0), "!=": (0, 0)}[op]
        return Pred.atom(Atom("diff", self.name, rng[0], rng[1], col2=other.name,
                              negate=(op == "!=")))

    def __lt__(self, o): return self._cmp(o, "<")
    def __le__(self, o): return self._cmp(o, "<=")
    def __gt__(self, o): return self._cmp(o, ">")
    def __ge__(self, o): return self._cmp(o, ">=")
    def __eq__(self, o): return self._cmp(o, "==")
    def __ne__(self, o): return self._cmp(o, "!=")
    __hash__ = None

    def __repr__(self) -> str:
        return f"ColRef({self.name!r}, {self.col!r})"


@dataclass(frozen=True)
class DerivedKey:
    """A group-by key computed from one column in the kernel: ``year(date)``
    (SQL ``extract(year from ...)``) and/or a constant offset
    (``c_nationkey + 10`` = the phone country code)."""

    src: str
    xform: str = "none"        # "none" | "year"
    offset: int = 0

    def __add__(self, k):
        return replace(self, offset=self.offset + int(k))


def year(ref: ColRef) -> DerivedKey:
    if ref.col.kind != "date32":
        raise SchemaError(f"year() expects a date32 column, {ref.name} is {ref.col.kind}")
    return DerivedKey(ref.name, "year")


def key_of(ref: ColRef, offset: int = 0) -> DerivedKey:
    if ref.col.kind not in ("int64", "date32"):
        raise SchemaError(f"derived key over {ref.col.kind} column {ref.name!r}")
    return DerivedKey(ref.name, "none", int(offset))


def isin(ref: ColRef, values) -> Pred:
    """Dictionary-set membership (table.py:185-192): codes whose string is in values."""
    if ref.col.kind != "dict":
        raise SchemaError(f"isin expects a dict column, {ref.name} is {ref.col.kind}")
    wanted = set(values)
    codes = frozenset(i for i, s in enumerate(ref.col.dictionary) if s in wanted)
    return Pred.atom(Atom("set", ref.name, codes=codes))


def codes_where(ref: ColRef, fn) -> Pred:
    """Rows whose dictionary string satisfies fn (queries.py:23-29)."""
    if ref.col.kind != "dict":
        raise SchemaError(f"codes_where expects a dict column, {ref.name} is {ref.col.kind}")
    codes = _codes_cached(ref.col.dictionary, fn)
    return Pred.atom(Atom("set", ref.name, codes=codes))


_CODES_CACHE: dict = {}


def _codes_cached(dictionary, fn) -> frozenset:
    """Evaluating a LIKE-style predicate over a dictionary is host time on
    every run of a query; the drivers pass the same lambda code with the same
    captured values each time, so the code set is memoised on (dictionary,
    code object, closure values)."""
    try:
        cells = tuple(c.cell_contents for c in (fn.__closure__ or ()))
        key = (id(dictionary), fn.__code__, cells, fn.__defaults__)
        hash(key)
    except (AttributeError, TypeError, ValueError):
        return frozenset(i for i, s in enumerate(dictionary) if fn(s))
    hit = _CODES_CACHE.get(key)
    if hit is not None and hit[0] is dictionary:
        return hit[1]
    codes = frozenset(i for i, s in enumerate(dictionary) if fn(s))
    _CODES_CACHE[key] = (dictionary, codes)
    return codes


# ---------------------------------------------------------------------------
# integerisation of a measure for the kernel
# ---------------------------------------------------------------------------

@dataclass
class IntMeasure:
    """Kernel form: value * Q = sum_t coef_t * prod_f (a_f + b_f * phys_f)."""

    terms: list = field(default_factory=list)   # [(coef:int, [(a:int, b:int, col)])]
    q: int = 1                                  # denominator: result = acc / q
    cond: Atom | None = None


_INT_CACHE: dict = {}


def integerise(p: Poly, cols: dict[str, Column]) -> IntMeasure:
    """Rewrite a logical-unit polynomial over physical fixed-point integers
    (memoised on the polynomial's structure and its columns' scales: plans
    rebuild the same expressions every run and Fraction arithmetic is slow)."""
    try:
        key = (tuple((t.coef, tuple((f.a, f.b, f.col, cols[f.col].kind == "float64" and
                                     cols[f.col].scale) for f in t.factors)) for t in p.terms),
               p.cond)
        hit = _INT_CACHE.get(key)
    except TypeError:          # unhashable condition: no memo
        key, hit = None, None
    if hit is not None:
        return hit
    res = _integerise(p, cols)
    if key is not None:
        if len(_INT_CACHE) > 4096:
            _INT_CACHE.clear()
        _INT_CACHE[key] = res
    return res


def _integerise(p: Poly, cols: dict[str, Column]) -> IntMeasure:
    raw = []
    for t in p.terms:
        coef = t.coef
        fs = []
        for f in t.factors:
            c = cols[f.col]
            s = c.scale if c.kind == "float64" else 0
            b = f.b / (10 ** s)
            d = math.lcm(f.a.denominator, b.denominator)
            fs.append((int(f.a * d), int(b * d), f.col))
            coef = coef / d
        raw.append((coef, fs))
    q = 1
    for coef, _ in raw:
        q = math.lcm(q, coef.denominator)
    terms = [(int(coef * q), fs) for coef, fs in raw]
    return IntMeasure(terms, q, p.cond)


def decimal_exponent(q: int) -> int:
    """k with q == 10**k, else -1."""
    k = 0
    while q % 10 == 0:
        q //= 10
        k += 1
    return k if q == 1 else -1

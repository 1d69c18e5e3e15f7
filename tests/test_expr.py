"""Host-side predicate/measure compilation (no GPU): the integer bounds must
select exactly the rows the reference's float64 comparisons select."""

import numpy as np
import pytest
import torch

from paper_2506_09226_b200.expr import ColRef, INT64_MAX, INT64_MIN, integerise, isin, where
from paper_2506_09226_b200.table import Column, SchemaError


def col(kind, vals, scale=0, dictionary=None):
    v = np.asarray(vals)
    return Column(kind, torch.from_numpy(v), scale, dictionary, int(v.min()), int(v.max()))


def atom_mask(pred, vals):
    (clause,) = pred.clauses
    (a,) = clause
    m = (vals >= a.lo) & (vals <= a.hi)
    return ~m if a.negate else m


@pytest.mark.parametrize("lit", [0.05, 0.07, 0.06, 0.055, 0.0, 0.1, 0.051, 1.0, -0.01])
@pytest.mark.parametrize("op", ["<", "<=", ">", ">=", "==", "!="])
def test_decimal_literal_bounds_match_float_semantics(lit, op):
    ints = np.arange(-20, 121, dtype=np.int64)
    ref = ints / 100.0                       # the reference stores disc = k/100.0
    c = ColRef("d", col("float64", ints.astype(np.int16), 2))
    pred = {"<": c < lit, "<=": c <= lit, ">": c > lit, ">=": c >= lit,
            "==": c == lit, "!=": c != lit}[op]
    expect = {"<": ref < lit, "<=": ref <= lit, ">": ref > lit, ">=": ref >= lit,
              "==": ref == lit, "!=": ref != lit}[op]
    assert np.array_equal(atom_mask(pred, ints), expect)


def test_int_and_date_bounds():
    vals = np.arange(0, 60)
    c = ColRef("q", col("int64", vals.astype(np.int8)))
    assert np.array_equal(atom_mask(c < 24, vals), vals < 24)
    assert np.array_equal(atom_mask(c <= 23.5, vals), vals <= 23.5)
    assert np.array_equal(atom_mask(c > 23.5, vals), vals > 23.5)
    assert np.array_equal(atom_mask(c == 3.5, vals), vals == 3.5)


def test_dnf_algebra():
    a = ColRef("a", col("int64", np.arange(10)))
    b = ColRef("b", col("int64", np.arange(10)))
    p = ((a < 3) & (b > 4)) | (a == 7)
    assert len(p.clauses) == 2
    q = p & (b < 9)
    assert len(q.clauses) == 2 and all(len(c) in (2, 3) for c in q.clauses)
    n = ~((a < 3) & (b > 4))
    assert len(n.clauses) == 2 and all(x[0].negate for x in n.clauses)
    with pytest.raises(TypeError):
        bool(a < 3)


def test_isin_and_dict_errors():
    d = ("REG AIR", "AIR", "RAIL", "SHIP", "TRUCK", "MAIL", "FOB")
    c = ColRef("m", col("dict", np.arange(7).astype(np.uint8), 0, d))
    p = isin(c, ["MAIL", "SHIP"])
    assert p.clauses[0][0].codes == frozenset({3, 5})
    with pytest.raises(SchemaError):
        c < 3
    with pytest.raises(SchemaError):
        isin(ColRef("x", col("int64", np.arange(3))), ["a"])


def test_measure_integerisation_q1_charge():
    ext = col("float64", np.asarray([90000, 189900], dtype=np.int32), 2)
    dsc = col("float64", np.asarray([0, 10], dtype=np.int8), 2)
    tax = col("float64", np.asarray([0, 8], dtype=np.int8), 2)
    cols = {"e": ext, "d": dsc, "t": tax}
    e, d, t = (ColRef(n, cols[n]) for n in "edt")
    charge = e * (1.0 - d) * (1.0 + t)
    im = integerise(charge, cols)
    assert im.q == 10 ** 6
    assert len(im.terms) == 1 and len(im.terms[0][1]) == 3
    # exact value for ext=1899.00, disc=0.10, tax=0.08
    coef, fs = im.terms[0]
    row = {"e": 189900, "d": 10, "t": 8}
    v = coef
    for a, b, name in fs:
        v *= a + b * row[name]
    assert v == round(1899.00 * 0.9 * 1.08 * 10 ** 6)


def test_where_gates_one_atom():
    d = ("1-URGENT", "2-HIGH", "3-MEDIUM")
    c = ColRef("p", col("dict", np.arange(3).astype(np.uint8), 0, d))
    w = where(isin(c, ["1-URGENT", "2-HIGH"]), 1)
    assert w.cond is not None and w.integral
    w2 = where(~isin(c, ["1-URGENT", "2-HIGH"]), 1)
    assert w2.cond.negate

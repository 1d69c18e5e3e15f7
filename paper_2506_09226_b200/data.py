"""Seeded TPC-H-shaped data, generated straight into the narrowed HBM layout.

Restates the reference generator ``shufflecast.data.generate``
(`/root/reference/pkg/src/shufflecast/data.py:161-268`) value-for-value:
the same ``numpy.random.default_rng(seed)`` stream is consumed by the same
draws in the same order (orders -> lineitem -> customer -> part -> partsupp
-> supplier), so every logical value is identical to
the reference's.  What differs is the *storage*: each draw is narrowed as
soon as it is produced (int64 draws to int8/int16/int32, decimals to
fixed-point integers, dates to int16 days, dictionary codes to uint8), so
SF100 lineitem is ~25 B/row (15 GB) instead of the reference's 76 B/row and
the host never holds the wide copy.  ``Dataset.to_reference()`` widens back
to the reference dtypes for the oracle (tests only).

Also carries ``partition_dataset`` (`data.py:284-302`), whose
``default_keys`` scheme runs on the GPU through the partition kernel
(see ``exchange.hash_partition``) when tables are device resident; the host
variant here only computes row-index lists via the same Fibonacci hash.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

from .table import HostColumn, HostTable, date_to_days, narrow_host

PARTITION_SCHEMES = ("default_keys", "unpartitioned", "round_robin")
# 25-row nation / 5-row region (generator extension, absent from the
# reference): replicated on every worker under every scheme, as the paper's
# Table-4 plan counts assume (Q5 (0,2) = customer +
# supplier broadcasts, no exchange for nation / region)
REPLICATED_TABLES = ("nation", "region")

# data.py:47-56 -- conventional partition key per table
DEFAULT_PARTITION_KEYS = {
    "lineitem": "l_orderkey",
    "orders": "o_orderkey",
    "customer": "c_custkey",
    "part": "p_partkey",
    "partsupp": "ps_partkey",
    "supplier": "s_suppkey",
    "nation": "n_nationkey",
    "region": "r_regionkey",
}

# Canonical dictionaries (data.py:58-82); shared by every table/partition.
RETURN_FLAGS = ("R", "A", "N")
LINE_STATUSES = ("O", "F")
SHIP_INSTRUCTS = ("DELIVER IN PERSON", "COLLECT COD", "NONE", "TAKE BACK RETURN")
SHIP_MODES = ("REG AIR", "AIR", "RAIL", "SHIP", "TRUCK", "MAIL", "FOB")
ORDER_PRIORITIES = ("1-URGENT", "2-HIGH", "3-MEDIUM", "4-NOT SPECIFIED", "5-LOW")
MARKET_SEGMENTS = ("AUTOMOBILE", "BUILDING", "FURNITURE", "MACHINERY", "HOUSEHOLD")
BRANDS = tuple(f"Brand#{a}{b}" for a in range(1, 6) for b in range(1, 6))
TYPES = tuple(" ".join(w) for w in itertools.product(
    ("STANDARD", "SMALL", "MEDIUM", "LARGE", "ECONOMY", "PROMO"),
    ("ANODIZED", "BURNISHED", "PLATED", "POLISHED", "BRUSHED"),
    ("TIN", "NICKEL", "BRASS", "STEEL", "COPPER"),
))
CONTAINERS = tuple(" ".join(w) for w in itertools.product(
    ("SM", "MED", "LG", "JUMBO", "WRAP"),
    ("CASE", "BOX", "BAG", "JAR", "PKG", "PACK", "CAN", "DRUM"),
))
# The reference's nation names are placeholders NATION_00..24 (data.py:80);
# the 22-query extension needs the TPC-H names.  Codes (the stored values)
# are unchanged, so every reference column stays bit-identical.
NATION_NAMES = ("ALGERIA", "ARGENTINA", "BRAZIL", "CANADA", "EGYPT", "ETHIOPIA", "FRANCE",
                "GERMANY", "INDIA", "INDONESIA", "IRAN", "IRAQ", "JAPAN", "JORDAN", "KENYA",
                "MOROCCO", "MOZAMBIQUE", "PERU", "CHINA", "ROMANIA", "SAUDI ARABIA", "VIETNAM",
                "RUSSIA", "UNITED KINGDOM", "UNITED STATES")
REGION_NAMES = ("AFRICA", "AMERICA", "ASIA", "EUROPE", "MIDDLE EAST")

# Logical schema per table (data.py:84-105): (column, reference kind).
SCHEMAS: dict[str, list[tuple[str, str]]] = {
    "lineitem": [
        ("l_orderkey", "int64"), ("l_partkey", "int64"), ("l_quantity", "int64"),
        ("l_extendedprice", "float64"), ("l_discount", "float64"), ("l_tax", "float64"),
        ("l_returnflag", "dict"), ("l_linestatus", "dict"),
        ("l_shipdate", "date32"), ("l_commitdate", "date32"), ("l_receiptdate", "date32"),
        ("l_shipinstruct", "dict"), ("l_shipmode", "dict"), ("l_suppkey", "int64"),
    ],
    "orders": [
        ("o_orderkey", "int64"), ("o_custkey", "int64"), ("o_orderdate", "date32"),
        ("o_orderpriority", "dict"), ("o_shippriority", "int64"), ("o_totalprice", "float64"),
        ("o_orderstatus", "dict"), ("o_comment", "dict"),
    ],
    "customer": [("c_custkey", "int64"), ("c_mktsegment", "dict"), ("c_nationkey", "int64"),
                 ("c_acctbal", "float64")],
    "part": [
        ("p_partkey", "int64"), ("p_brand", "dict"), ("p_type", "dict"),
        ("p_size", "int64"), ("p_container", "dict"), ("p_name", "dict"), ("p_mfgr", "dict"),
    ],
    "partsupp": [("ps_partkey", "int64"), ("ps_suppkey", "int64"), ("ps_supplycost", "float64"),
                 ("ps_availqty", "int64")],
    "supplier": [("s_suppkey", "int64"), ("s_nationkey", "int64"), ("s_acctbal", "float64"),
                 ("s_comment", "dict")],
    "nation": [("n_nationkey", "int64"), ("n_name", "dict"), ("n_regionkey", "int64")],
    "region": [("r_regionkey", "int64"), ("r_name", "dict")],
}

DICTIONARIES: dict[str, tuple[str, ...]] = {
    "l_returnflag": RETURN_FLAGS, "l_linestatus": LINE_STATUSES,
    "l_shipinstruct": SHIP_INSTRUCTS, "l_shipmode": SHIP_MODES,
    "o_orderpriority": ORDER_PRIORITIES, "c_mktsegment": MARKET_SEGMENTS,
    "p_brand": BRANDS, "p_type": TYPES, "p_container": CONTAINERS,
    "n_name": NATION_NAMES, "r_name": REGION_NAMES,
}


_ORDERDATE_LO = date_to_days("1992-01-01")
_ORDERDATE_HI = date_to_days("1998-08-02")
_LINESTATUS_CUTOFF = date_to_days("1995-06-17")


class DataError(ValueError):
    """Bad generator / partitioning arguments (data.py:126)."""


@dataclass
class Dataset:
    """Host-resident narrowed tables plus the knobs that produced them."""

    tables: dict[str, HostTable]
    sf: float | None = None
    skew: float = 0.0
    seed: int | None = None

    def table(self, name: str) -> HostTable:
        return self.tables[name]

    def row_counts(self) -> dict[str, int]:
        return {n: t.row_count for n, t in self.tables.items()}

    def manifest(self) -> dict:
        return {"sf": self.sf, "skew": self.skew, "seed": self.seed,
                "row_counts": self.row_counts()}

    @property
    def nbytes(self) -> int:
        return sum(t.nbytes for t in self.tables.values())

    def to_reference(self) -> dict[str, dict[str, tuple]]:
        """Widen to the reference's dtypes: {table: {col: (kind, values, dict)}}.

        Test/oracle use only -- the product never widens.
        """
        return {n: t.to_reference() for n, t in self.tables.items()}


def _zipf(rng: np.random.Generator, n_items: int, s: float, size: int) -> np.ndarray:
    # Same draw as data.py:154-158 (rank 1 hottest, keys 1..n_items).
    w = np.arange(1, n_items + 1, dtype=np.float64) ** (-s)
    w /= w.sum()
    return rng.choice(n_items, size=size, p=w).astype(np.int64) + 1


def _dict(codes: np.ndarray, name: str) -> HostColumn:
    return HostColumn.from_codes(codes, DICTIONARIES[name])


def generate(sf: float, skew: float = 0.0, seed: int = 0) -> Dataset:
    """Deterministic dataset for (sf, skew, seed); values identical to data.py:161."""
    if sf <= 0:
        raise DataError(f"scale factor must be positive, got {sf}")
    if skew < 0:
        raise DataError(f"skew exponent must be >= 0, got {skew}")
    rng = np.random.default_rng(seed)
    n_ord = max(1, round(1_500_000 * sf))
    n_cust = max(1, round(150_000 * sf))
    n_part = max(1, round(200_000 * sf))
    n_supp = max(1, round(10_000 * sf))
    i64 = np.int64

    # ---- orders: custkey, orderdate, priority -------------------------------
    if skew > 0:
        o_cust = _zipf(rng, n_cust, skew, n_ord)
    else:
        o_cust = rng.integers(1, n_cust + 1, size=n_ord, dtype=i64)
    o_date = narrow_host(rng.integers(_ORDERDATE_LO, _ORDERDATE_HI + 1, size=n_ord, dtype=i64))
    o_prio = rng.integers(0, len(ORDER_PRIORITIES), size=n_ord)
    orders = HostTable({
        "o_orderkey": HostColumn.int_range(1, n_ord + 1),
        "o_custkey": HostColumn.from_ints("int64", o_cust),
        "o_orderdate": HostColumn.from_ints("date32", o_date),
        "o_orderpriority": _dict(o_prio, "o_orderpriority"),
        "o_shippriority": HostColumn.from_ints("int64", np.zeros(n_ord, dtype=np.int8)),
    })
    del o_cust, o_prio

    # ---- lineitem ----------------------------------------------------------
    if skew > 0:
        n_li = max(1, round(6_000_000 * sf))
        l_ok = np.sort(_zipf(rng, n_ord, skew, n_li))
    else:
        lines_per_order = rng.integers(1, 8, size=n_ord, dtype=i64)
        l_ok = np.repeat(np.arange(1, n_ord + 1, dtype=i64), lines_per_order)
        n_li = len(l_ok)
        del lines_per_order
    if skew > 0:
        l_pk = _zipf(rng, n_part, skew, n_li)
    else:
        l_pk = rng.integers(1, n_part + 1, size=n_li, dtype=i64)
    qty = narrow_host(rng.integers(1, 51, size=n_li, dtype=i64))
    # extendedprice = qty * (900 + partkey % 1000): integral dollars -> cents
    ext_cents = (qty.astype(np.int32) * (900 + (l_pk % 1000)).astype(np.int32)) * np.int32(100)
    odate = o_date[(l_ok - 1)]
    ship = narrow_host(odate.astype(np.int32) + rng.integers(1, 122, size=n_li).astype(np.int32))
    commit = narrow_host(odate.astype(np.int32) + rng.integers(30, 91, size=n_li).astype(np.int32))
    del odate
    receipt = narrow_host(ship.astype(np.int32) + rng.integers(1, 31, size=n_li).astype(np.int32))
    disc = narrow_host(rng.integers(0, 11, size=n_li))
    tax = narrow_host(rng.integers(0, 9, size=n_li))
    rflag = rng.integers(0, len(RETURN_FLAGS), size=n_li)
    lineitem_cols = {
        "l_orderkey": _sorted(HostColumn.from_ints("int64", l_ok)),
        "l_partkey": HostColumn.from_ints("int64", l_pk),
        "l_quantity": HostColumn.from_ints("int64", qty),
        "l_extendedprice": HostColumn.decimal(ext_cents, 2),
        "l_discount": HostColumn.decimal(disc, 2),
        "l_tax": HostColumn.decimal(tax, 2),
        "l_returnflag": _dict(rflag, "l_returnflag"),
        "l_linestatus": _dict((ship <= _LINESTATUS_CUTOFF).astype(np.uint8), "l_linestatus"),
        "l_shipdate": HostColumn.from_ints("date32", ship),
        "l_commitdate": HostColumn.from_ints("date32", commit),
        "l_receiptdate": HostColumn.from_ints("date32", receipt),
    }
    del l_ok, l_pk, rflag
    lineitem_cols["l_shipinstruct"] = _dict(
        rng.integers(0, len(SHIP_INSTRUCTS), size=n_li), "l_shipinstruct")
    lineitem_cols["l_shipmode"] = _dict(
        rng.integers(0, len(SHIP_MODES), size=n_li), "l_shipmode")
    lineitem = HostTable(lineitem_cols)

    # ---- customer, part, partsupp, supplier -------------------------------
    customer = HostTable({
        "c_custkey": HostColumn.int_range(1, n_cust + 1),
        "c_mktsegment": _dict(rng.integers(0, len(MARKET_SEGMENTS), size=n_cust), "c_mktsegment"),
        "c_nationkey": HostColumn.from_ints("int64", rng.integers(0, 25, size=n_cust)),
    })
    part = HostTable({
        "p_partkey": HostColumn.int_range(1, n_part + 1),
        "p_brand": _dict(rng.integers(0, len(BRANDS), size=n_part), "p_brand"),
        "p_type": _dict(rng.integers(0, len(TYPES), size=n_part), "p_type"),
        "p_size": HostColumn.from_ints("int64", rng.integers(1, 51, size=n_part)),
        "p_container": _dict(rng.integers(0, len(CONTAINERS), size=n_part), "p_container"),
    })
    ps_supp = rng.integers(1, n_supp + 1, size=4 * n_part)
    ps_cost = rng.uniform(1.0, 1000.0, size=4 * n_part).round(2)
    partsupp = HostTable({
        "ps_partkey": HostColumn.from_ints(
            "int64", np.repeat(np.arange(1, n_part + 1, dtype=np.int64), 4)),
        "ps_suppkey": HostColumn.from_ints("int64", ps_supp),
        "ps_supplycost": HostColumn.from_float(ps_cost),
    })
    supplier = HostTable({
        "s_suppkey": HostColumn.int_range(1, n_supp + 1),
        "s_nationkey": HostColumn.from_ints("int64", rng.integers(0, 25, size=n_supp)),
    })
    nation = HostTable({
        "n_nationkey": HostColumn.int_range(0, 25),
        "n_name": _dict(np.arange(25), "n_name"),
        "n_regionkey": HostColumn.from_ints("int64", np.arange(25) % 5),
    })
    region = HostTable({
        "r_regionkey": HostColumn.int_range(0, 5),
        "r_name": _dict(np.arange(5), "r_name"),
    })
    extend_tpch(lineitem, orders, customer, part, partsupp, supplier, seed)
    return Dataset(
        tables={"lineitem": lineitem, "orders": orders, "customer": customer,
                "part": part, "partsupp": partsupp, "supplier": supplier,
                "nation": nation, "region": region},
        sf=sf, skew=skew, seed=seed,
    )


# ---------------------------------------------------------------------------
# TPC-H extension for the 16 queries the reference lacks
#
# Every new column comes from an RNG stream independent of the reference's
# ``default_rng(seed)`` (or is a deterministic function of reference
# columns), so the reference's columns stay bit-identical.  Free-text
# columns (names, comments) are dictionary-coded over small deterministic
# vocabularies: LIKE predicates resolve on the host dictionary into code
# bitmaps, exactly like the reference's ``_codes_where`` (queries.py:23-29).
# Identity columns the queries only print (c_name = "Customer#<key>",
# s_name, addresses, phones) are not materialised: results carry the key;
# c_phone's country code is c_nationkey + 10 (the dbgen rule).
# ---------------------------------------------------------------------------

COLORS = (
    "almond antique aquamarine azure beige bisque black blanched blue blush brown burlywood "
    "burnished chartreuse chiffon chocolate coral cornflower cornsilk cream cyan dark deep dim "
    "dodger drab firebrick floral forest frosted gainsboro ghost goldenrod green grey honeydew "
    "hot indian ivory khaki lace lavender lawn lemon light lime linen magenta maroon medium "
    "metallic midnight mint misty moccasin navajo navy olive orange orchid pale papaya peach "
    "peru pink plum powder puff purple red rose rosy royal saddle salmon sandy seashell sienna "
    "sky slate smoke snow spring steel tan thistle tomato turquoise violet wheat white yellow"
).split()
_WORDS = ("furiously quickly carefully blithely slyly fluffily regular final ironic express "
          "bold pending even silent unusual special requests deposits accounts packages "
          "instructions foxes ideas theodolites pinto beans platelets asymptotes dependencies "
          "excuses warthogs sheaves courts dolphins sentiments frets").split()
N_PART_NAMES = 1000
N_ORDER_COMMENTS = 1024
N_SUPP_COMMENTS = 256
ORDER_STATUSES = ("F", "O", "P")
MANUFACTURERS = tuple(f"Manufacturer#{i}" for i in range(1, 6))


def _vocab_rng(tag: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([2506, 9226, tag]))


def _part_names() -> tuple[str, ...]:
    r = _vocab_rng(1)
    names, seen = [], set()
    while len(names) < N_PART_NAMES:
        w = " ".join(COLORS[i] for i in r.choice(len(COLORS), 5, replace=False))
        if w not in seen:
            seen.add(w)
            names.append(w)
    return tuple(names)


def _comments(tag: int, n: int, plant: tuple[str, str], frac: float) -> tuple[str, ...]:
    """n distinct comments; about `frac` of them contain plant[0] ... plant[1]."""
    r = _vocab_rng(tag)
    out, seen = [], set()
    while len(out) < n:
        k = int(r.integers(4, 9))
        words = [_WORDS[i] for i in r.integers(0, len(_WORDS), k)]
        if r.random() < frac:
            i = int(r.integers(0, k - 1))
            words.insert(i, plant[0])
            words.insert(int(r.integers(i + 1, len(words) + 1)), plant[1])
        else:
            words = [w for w in words if w != plant[0]] or ["even"]
        c = " ".join(words)
        if c not in seen:
            seen.add(c)
            out.append(c)
    return tuple(out)


DICTIONARIES["p_name"] = _part_names()
DICTIONARIES["p_mfgr"] = MANUFACTURERS
DICTIONARIES["o_orderstatus"] = ORDER_STATUSES
DICTIONARIES["o_comment"] = _comments(2, N_ORDER_COMMENTS, ("special", "requests"), 0.02)
DICTIONARIES["s_comment"] = _comments(3, N_SUPP_COMMENTS, ("Customer", "Complaints"), 0.04)


def extend_tpch(lineitem: HostTable, orders: HostTable, customer: HostTable, part: HostTable,
                partsupp: HostTable, supplier: HostTable, seed: int) -> None:
    """Add the columns the 16 extra queries need (in place)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 22]))
    n_li, n_ord = lineitem.row_count, orders.row_count
    n_cust, n_part, n_supp = customer.row_count, part.row_count, supplier.row_count
    # l_suppkey: one of the part's four partsupp suppliers, so lineitem joins
    # partsupp on (partkey, suppkey) as in dbgen
    pk = lineitem.column("l_partkey").values.astype(np.int64)
    ps_supp = partsupp.column("ps_suppkey").values
    pick = rng.integers(0, 4, size=n_li)
    lineitem.columns["l_suppkey"] = HostColumn.from_ints("int64", ps_supp[(pk - 1) * 4 + pick])
    del pk, pick
    # o_totalprice = sum over lines of round(ext * (1 + tax) * (1 - disc)), cents
    ok = lineitem.column("l_orderkey").values
    line = (lineitem.column("l_extendedprice").values.astype(np.int64)
            * (100 + lineitem.column("l_tax").values.astype(np.int64))
            * (100 - lineitem.column("l_discount").values.astype(np.int64)))
    line = (line + 5000) // 10000
    starts = np.searchsorted(ok, np.arange(1, n_ord + 2, dtype=np.int64))
    cs = np.concatenate([[0], np.cumsum(line)])
    total = cs[starts[1:]] - cs[starts[:-1]]
    orders.columns["o_totalprice"] = HostColumn.decimal(total, 2)
    del line, cs, total
    # o_orderstatus: F if every line is F, O if every line is O, else P
    f = (lineitem.column("l_linestatus").values == LINE_STATUSES.index("F")).astype(np.int64)
    cf = np.concatenate([[0], np.cumsum(f)])
    nf = cf[starts[1:]] - cf[starts[:-1]]
    nl = starts[1:] - starts[:-1]
    status = np.where((nf == nl) & (nl > 0), 0, np.where(nf == 0, 1, 2))
    orders.columns["o_orderstatus"] = _dict(status, "o_orderstatus")
    del f, cf, nf, nl, status, starts
    orders.columns["o_comment"] = _dict(rng.integers(0, N_ORDER_COMMENTS, size=n_ord),
                                        "o_comment")
    customer.columns["c_acctbal"] = HostColumn.decimal(
        rng.integers(-99999, 1000000, size=n_cust), 2)
    part.columns["p_name"] = _dict(rng.integers(0, N_PART_NAMES, size=n_part), "p_name")
    # p_mfgr follows p_brand (Brand#MN is made by Manufacturer#M), as in dbgen
    brand = part.column("p_brand").values.astype(np.int64)
    mfgr = np.asarray([int(BRANDS[i][6]) - 1 for i in range(len(BRANDS))])[brand]
    part.columns["p_mfgr"] = _dict(mfgr, "p_mfgr")
    partsupp.columns["ps_availqty"] = HostColumn.from_ints(
        "int64", rng.integers(1, 10000, size=4 * n_part))
    supplier.columns["s_acctbal"] = HostColumn.decimal(
        rng.integers(-99999, 1000000, size=n_supp), 2)
    supplier.columns["s_comment"] = _dict(rng.integers(0, N_SUPP_COMMENTS, size=n_supp),
                                          "s_comment")
    for t in (lineitem, orders, customer, part, partsupp, supplier):
        t.row_count = next(iter(t.columns.values())).row_count


# ---------------------------------------------------------------------------
# on-disk cache of the narrowed columns (.npy + manifest), so SF100 is
# generated once per box and every rank of a job can mmap the same files
# (SURVEY.md §5 "cache the generated columns as .npy").  Loader-only: no
# timing depends on it.
# ---------------------------------------------------------------------------

def save_dataset(ds: Dataset, path: str) -> None:
    import json
    import os
    os.makedirs(path, exist_ok=True)
    meta = {"sf": ds.sf, "skew": ds.skew, "seed": ds.seed, "tables": {}}
    for tname, t in ds.tables.items():
        cols = {}
        for cname, c in t.columns.items():
            np.save(os.path.join(path, f"{tname}.{cname}.npy"), c.values)
            cols[cname] = {"kind": c.kind, "scale": c.scale, "lo": c.lo, "hi": c.hi,
                           "dictionary": list(c.dictionary) if c.dictionary else None,
                           "dense": bool(c.dense), "sorted": bool(c.sorted)}
        meta["tables"][tname] = cols
    tmp = os.path.join(path, "manifest.json.tmp")
    with open(tmp, "w") as fh:
        json.dump(meta, fh)
    os.replace(tmp, os.path.join(path, "manifest.json"))


def load_dataset(path: str, mmap: bool = True) -> Dataset:
    import json
    import os
    with open(os.path.join(path, "manifest.json")) as fh:
        meta = json.load(fh)
    tables = {}
    for tname, cols in meta["tables"].items():
        hc = {}
        for cname, m in cols.items():
            v = np.load(os.path.join(path, f"{tname}.{cname}.npy"),
                        mmap_mode="r" if mmap else None)
            hc[cname] = HostColumn(m["kind"], v, m["scale"],
                                   tuple(m["dictionary"]) if m["dictionary"] else None,
                                   m["lo"], m["hi"], bool(m.get("dense", False)),
                                   bool(m.get("sorted", cname == "l_orderkey")))
        tables[tname] = HostTable(hc)
    return Dataset(tables, meta["sf"], meta["skew"], meta["seed"])


def cached_generate(sf: float, skew: float = 0.0, seed: int = 0,
                    root: str = "/tmp/scx_data") -> Dataset:
    """generate() through the on-disk cache (validated by the manifest)."""
    import os
    path = os.path.join(root, f"sf{sf}_skew{skew}_seed{seed}")
    if os.path.exists(os.path.join(path, "manifest.json")):
        try:
            return load_dataset(path)
        except Exception:   # corrupt cache: regenerate
            pass
    ds = generate(sf, skew, seed)
    try:
        save_dataset(ds, path)
    except OSError:
        pass
    return ds


# ---------------------------------------------------------------------------
# host-side partition assignment (the GPU path lives in exchange.py)
# ---------------------------------------------------------------------------

@dataclass
class PartitionedDataset:
    """Per-worker table sets produced by one partitioning scheme (data.py:271-281)."""

    scheme: str
    n_workers: int
    workers: list[dict] = field(default_factory=list)
    source: Dataset | None = None

    def worker_tables(self, rank: int) -> dict:
        return self.workers[rank]


def fib_hash_host(keys: np.ndarray) -> np.ndarray:
    """Single-key Fibonacci hash, u64 wraparound (exchange.py:29-49).

    Host helper for metadata-scale work and for checking; bulk hashing runs
    in the ``scx_hash_partition`` kernel.
    """
    f = np.uint64(0x9E3779B97F4A7C15)
    with np.errstate(over="ignore"):
        return (keys.astype(np.int64).astype(np.uint64) * f) * f


def partition_rows(table: HostTable, scheme: str, key: str | None, n: int) -> list[np.ndarray]:
    """Row indices per worker for ``scheme`` (data.py:284-302), input order kept."""
    rows = table.row_count
    if scheme == "default_keys":
        b = fib_hash_host(table.column(key).to_int64()) % np.uint64(n)
        order = np.argsort(b, kind="stable")
        cuts = np.searchsorted(b[order], np.arange(n + 1, dtype=np.uint64))
        return [order[cuts[i]:cuts[i + 1]] for i in range(n)]
    if scheme == "unpartitioned":
        cuts = np.linspace(0, rows, n + 1).astype(np.int64)
        return [np.arange(cuts[i], cuts[i + 1]) for i in range(n)]
    idx = np.arange(rows)
    return [idx[idx % n == r] for r in range(n)]


def _sorted(c: HostColumn) -> HostColumn:
    """Mark a column generated in non-decreasing order (l_orderkey: orders'
    lines are emitted order by order, data.py:195-198 in the reference)."""
    c.sorted = True
    return c


def worker_rows(name: str, table: HostTable, scheme: str, n: int) -> list[np.ndarray]:
    """Row indices of table ``name`` per worker: the whole table on every
    worker for REPLICATED_TABLES, else partition_rows on its default key."""
    if name in REPLICATED_TABLES:
        return [np.arange(table.row_count)] * n
    return partition_rows(table, scheme, DEFAULT_PARTITION_KEYS[name], n)


def partition_dataset(ds: Dataset, n_workers: int, scheme: str = "default_keys") -> PartitionedDataset:
    """Host-side partitioning of a narrowed dataset (data.py:284).

    Used for small host datasets and by tests; ``engine.load_partition`` does
    the same assignment on the GPU for the bench path.
    """
    if n_workers < 1:
        raise DataError(f"need at least one worker, got {n_workers}")
    if scheme not in PARTITION_SCHEMES:
        raise DataError(f"unknown partitioning scheme {scheme!r}; choose from {PARTITION_SCHEMES}")
    workers: list[dict] = [{} for _ in range(n_workers)]
    for name, t in ds.tables.items():
        parts = worker_rows(name, t, scheme, n_workers)
        for r in range(n_workers):
            workers[r][name] = t.take(parts[r])
    return PartitionedDataset(scheme, n_workers, workers, ds)

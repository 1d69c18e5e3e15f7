"""Plan-specialised kernels (csrc/jit.cu): codegen + NVRTC for sm_100a, no GPU.

Hand-built descriptors covering every sink (dense registers / dense smem
table / hash group-by / compaction / count) and probe kind (direct / hash,
semi / anti / inner with payload) must generate CUDA that NVRTC compiles for
sm_100a without spilling.  The GPU parity suite then runs the same generator
on every TPC-H plan against the oracle.
"""

import ctypes as C
import os
import subprocess

import pytest

from paper_2506_09226_b200 import _lib as L


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    os.environ["SCX_JIT_CACHE"] = str(tmp_path_factory.mktemp("jit_cache"))
    return L.load()

def base(P, cols):
    P.n_base = len(cols); P.n_slots = len(cols)
    for i, dt in enumerate(cols):
        P.base[i] = L.Column_(0x10000 * (i + 1), dt, 0); P.slot_dtype[i] = dt

def _q6():
    P = L.Pipeline(); P.n_rows = 1000
    base(P, [L.SCX_I16, L.SCX_U8, L.SCX_I8, L.SCX_I32])
    atoms = [(0, 8766, 9130), (1, 5, 7), (2, -128, 23)]
    for i, (s, lo, hi) in enumerate(atoms):
        A = P.atoms[i]; A.op = L.ATOM_RANGE; A.slot = s; A.clause = 0; A.lo = lo; A.hi = hi
    P.pre.first_atom = 0; P.pre.n_atoms = 3; P.pre.clause_mask = 1
    S = P.sink; S.kind = L.SINK_AGG_DENSE; S.n_cells = 1; S.n_measures = 1
    m = S.m[0]; m.op = L.AGG_SUM; m.n_terms = 1; m.cond_atom = -1
    t = m.t[0]; t.coef = 1; t.n_factors = 2
    t.f[0].a, t.f[0].b, t.f[0].slot, t.f[0]._pad = 0, 1, 3, 1
    t.f[1].a, t.f[1].b, t.f[1].slot, t.f[1]._pad = 0, 1, 1, 1
    S.acc = 0x900000
    return P

def _q1():
    P = L.Pipeline(); P.n_rows = 1000
    # shipdate i16, rflag u8, lstatus u8, qty i8, ext i32, disc u8, tax u8
    base(P, [L.SCX_I16, L.SCX_U8, L.SCX_U8, L.SCX_I8, L.SCX_I32, L.SCX_U8, L.SCX_U8])
    A = P.atoms[0]; A.op = L.ATOM_RANGE; A.slot = 0; A.lo = -(1 << 40); A.hi = 10471
    P.pre.first_atom = 0; P.pre.n_atoms = 1; P.pre.clause_mask = 1
    S = P.sink; S.kind = L.SINK_AGG_DENSE; S.n_cells = 6; S.n_measures = 6
    S.gkey.n = 2; S.gkey.slot[0] = 1; S.gkey.slot[1] = 2; S.gcard[0] = 3; S.gcard[1] = 2
    S.glut[0] = 0; S.glut[1] = 3
    for i, x in enumerate([2, 0, 1, 1, 0]): P.lut[i] = x
    def fac(f, a, b, slot): f.a, f.b, f.slot, f._pad = a, b, slot, 1
    specs = [[(3,)], [(4,)], [(4,), ('1m', 5)], [(4,), ('1m', 5), ('1p', 6)], [(5,)], None]
    for i, sp in enumerate(specs):
        m = S.m[i]; m.cond_atom = -1
        if sp is None: m.op = L.AGG_COUNT; continue
        m.op = L.AGG_SUM; m.n_terms = 1; t = m.t[0]; t.coef = 1; t.n_factors = len(sp)
        for j, f in enumerate(sp):
            if len(f) == 1: fac(t.f[j], 0, 1, f[0])
            elif f[0] == '1m': fac(t.f[j], 100, -1, f[1])
            else: fac(t.f[j], 100, 1, f[1])
    S.acc = 0x900000
    return P

def _compact_probe(kind=L.HT_HASH, jk=L.JOIN_INNER):
    P = L.Pipeline(); P.n_rows = 1000
    base(P, [L.SCX_I32, L.SCX_I16, L.SCX_I32, L.SCX_U8])
    A = P.atoms[0]; A.op = L.ATOM_RANGE; A.slot = 1; A.lo = 9000; A.hi = 1 << 40
    P.pre.first_atom = 0; P.pre.n_atoms = 1; P.pre.clause_mask = 1
    P.n_probes = 1; pb = P.probe[0]; pb.kind = jk
    pb.key.n = 1; pb.key.slot[0] = 0; pb.key.bits[0] = 28; pb.key.lo[0] = 1
    pb.table.kind = kind; pb.table.keys = 0x5000; pb.table.vals = 0x6000; pb.table.cap = 1 << 20
    if jk == L.JOIN_INNER:
        pb.n_payload = 2; P.n_slots = 6
        pb.payload[0] = L.Column_(0x7000, L.SCX_I16, 0); pb.payload_slot[0] = 4; P.slot_dtype[4] = L.SCX_I16
        pb.payload[1] = L.Column_(0x8000, L.SCX_I64, 0); pb.payload_slot[1] = 5; P.slot_dtype[5] = L.SCX_I64
    S = P.sink; S.kind = L.SINK_COMPACT; S.n_out = 3
    for i, (s, dt) in enumerate([(0, L.SCX_I32), (2, L.SCX_I32), (5 if jk == L.JOIN_INNER else -1, L.SCX_I64)]):
        S.out_slot[i] = s; S.out[i] = L.Column_(0xa000 * (i + 1), dt, 0)
    S.status = 0xb000; S.count = 0xc000
    return P

def _prefetch_probe(kind):
    # monotone probe key (table._pad = 1): next-tile L2 prefetch of the build range
    P = _compact_probe(kind, L.JOIN_INNER)
    P.probe[0].table._pad = 1
    return P


def _hashgroup():
    P = _compact_probe()
    S = P.sink; S.kind = L.SINK_AGG_HASH; S.n_measures = 2
    S.gkey.n = 2; S.gkey.slot[0] = 0; S.gkey.slot[1] = 4; S.gkey.bits[0] = 28; S.gkey.bits[1] = 12
    S.gkey.shift[0] = 12; S.gkey.shift[1] = 0; S.gkey.lo[0] = 1; S.gkey.lo[1] = 8000; S.glut[0] = -1; S.glut[1] = -1
    m = S.m[0]; m.op = L.AGG_SUM; m.n_terms = 1; m.cond_atom = -1; t = m.t[0]; t.coef = 1; t.n_factors = 2
    t.f[0].a, t.f[0].b, t.f[0].slot, t.f[0]._pad = 0, 1, 2, 1
    t.f[1].a, t.f[1].b, t.f[1].slot, t.f[1]._pad = 100, -1, 3, 1
    S.m[1].op = L.AGG_COUNT; S.m[1].cond_atom = -1
    S.gkeys = 0x1000; S.acc = 0x2000; S.gcap = 1 << 20; S.flags = 0x3000
    return P


def _q1_packed():
    # SF100 bit budgets (measure._pad = 0x100 | bits): qty, ext, ext*(1-d),
    # ext*(1-d)*(1+t) (too wide), disc, count
    P = _q1()
    for i, b in enumerate([20, 38, 44, 0, 18, 14]):
        P.sink.m[i]._pad = (0x100 | b) if b else 0
    return P


def _hashgroup_narrow():
    # direct-addressed u32 sum / count table (sink.n_cells = 2), no key array
    P = _hashgroup()
    P.sink.n_cells = 2
    P.sink.gkeys = 0
    return P


def _dense_smem():
    P = _q1()
    P.sink.n_cells = 12
    P.sink.gcard[1] = 4
    return P


def _count():
    P = _q6()
    P.sink.kind = L.SINK_COUNT
    P.sink.count = 0xc000
    return P


def _bitmap_sink():
    P = _q6()
    S = P.sink
    S.kind = L.SINK_BITMAP
    S.gkey.n = 1
    S.gkey.slot[0] = 3
    S.gkey.bits[0] = 24
    S.gkey.lo[0] = 1
    S.gkeys = 0xd000
    S.gcap = 1 << 24
    return P


def _poly_left_year():
    P = _compact_probe(L.HT_DIRECT, L.JOIN_INNER)
    P.probe[0].kind = L.JOIN_LEFT
    A = P.atoms[1]
    A.op, A.slot, A.clause, A.lo, A.hi = L.ATOM_POLY, 0, 0, 1, 1 << 40
    P.pre.n_atoms = 1
    P.post.first_atom, P.post.n_atoms, P.post.clause_mask = 1, 1, 1
    m = P.polys[0]
    m.op, m.n_terms, m.cond_atom = L.AGG_SUM, 2, -1
    m.t[0].coef, m.t[0].n_factors = 5, 2
    m.t[0].f[0].a, m.t[0].f[0].b, m.t[0].f[0].slot, m.t[0].f[0]._pad = 0, 1, 1, 1
    m.t[0].f[1].a, m.t[0].f[1].b, m.t[0].f[1].slot, m.t[0].f[1]._pad = 0, 1, 4, 1
    m.t[1].coef, m.t[1].n_factors = -1, 1
    m.t[1].f[0].a, m.t[1].f[0].b, m.t[1].f[0].slot = 0, 1, 5
    S = P.sink
    S.kind = L.SINK_AGG_HASH
    S.n_measures = 1
    S.m[0].op, S.m[0].cond_atom = L.AGG_COUNT, -1
    S.gkey.n = 1
    S.gkey.slot[0] = 1
    S.gkey.bits[0] = 8
    S.gkey.lo[0] = 1992
    S.gkey.xform = L.XFORM_YEAR
    S.gkeys, S.acc, S.gcap, S.flags = 0x1000, 0x2000, 1 << 12, 0x3000
    return P


PLANS = {
    "bitmap_sink": _bitmap_sink,
    "semi_bitmap_probe": lambda: _compact_probe(L.HT_BITMAP, L.JOIN_SEMI),
    "poly_atom_left_join_year_key": _poly_left_year,
    "q6_dense1": _q6, "q1_dense6": _q1, "q1_dense6_packed": _q1_packed,
    "dense_smem": _dense_smem, "count": _count,
    "compact_inner_hash": _compact_probe,
    "compact_semi_direct": lambda: _compact_probe(L.HT_DIRECT, L.JOIN_SEMI),
    "compact_anti_hash": lambda: _compact_probe(L.HT_HASH, L.JOIN_ANTI),
    "hash_group": _hashgroup,
    "hash_group_direct_narrow": _hashgroup_narrow,
    "prefetch_identity_inner": lambda: _prefetch_probe(L.HT_IDENTITY),
    "prefetch_direct_inner": lambda: _prefetch_probe(L.HT_DIRECT),
}


@pytest.mark.parametrize("name", sorted(PLANS))
def test_codegen_compiles_for_sm100a(lib, name):
    P = PLANS[name]()
    n = lib.scx_pipeline_source(C.byref(P), None, 0)
    assert n > 0, lib.scx_last_error()
    buf = C.create_string_buffer(n + 1)
    lib.scx_pipeline_source(C.byref(P), buf, n + 1)
    src = buf.value.decode()
    assert "__global__" in src and "scx_pipe_" in src
    rc = lib.scx_pipeline_compile(C.byref(P))
    assert rc == 0, lib.scx_last_error().decode()
    cache = os.environ["SCX_JIT_CACHE"]
    cubins = [f for f in os.listdir(cache) if f.endswith(".cubin")]
    assert cubins
    kname = src.split("scx_pipe_")[1].split("(")[0]
    kname = "scx_pipe_" + kname
    res = subprocess.run(["cuobjdump", "-res-usage", os.path.join(cache, kname + ".cubin")],
                         capture_output=True, text=True)
    if res.returncode == 0:
        assert "LOCAL:0" in res.stdout and "STACK:0" in res.stdout, res.stdout   # no spills


def test_source_is_deterministic_and_pointer_free(lib):
    a, b = _q1(), _q1()
    b.base[0].ptr = 0x7770000
    b.sink.acc = 0x1230000
    sa, sb = C.create_string_buffer(1 << 16), C.create_string_buffer(1 << 16)
    lib.scx_pipeline_source(C.byref(a), sa, 1 << 16)
    lib.scx_pipeline_source(C.byref(b), sb, 1 << 16)
    assert sa.value == sb.value          # pointers are launch parameters, not code


def test_prefetch_emitted_only_for_monotone_probes(lib, monkeypatch):
    monkeypatch.setenv("SCX_GATHER_PF", "1")
    def src(P):
        n = lib.scx_pipeline_source(C.byref(P), None, 0)
        buf = C.create_string_buffer(n + 1)
        lib.scx_pipeline_source(C.byref(P), buf, n + 1)
        return buf.value.decode()
    assert "l2_prefetch((const void*)s0" in src(_prefetch_probe(L.HT_IDENTITY))
    assert "l2_prefetch((const void*)s0" not in src(_compact_probe(L.HT_DIRECT, L.JOIN_INNER))


def test_codegen_rejects_bad_descriptor(lib):
    P = _q6()
    P.base[0].ptr = 0x10001                # misaligned column
    assert lib.scx_pipeline_source(C.byref(P), None, 0) < 0
    assert b"aligned" in lib.scx_last_error()


def _chunk_two_probes(sink):
    # pre-predicate -> direct inner probe (a compaction point) -> semi bitmap
    # probe on a gathered payload -> sink: three levels in chunk mode
    P = _compact_probe(L.HT_DIRECT, L.JOIN_INNER)
    P.n_probes = 2
    pb = P.probe[1]
    pb.kind = L.JOIN_SEMI
    pb.key.n = 1; pb.key.slot[0] = 4; pb.key.bits[0] = 16; pb.key.lo[0] = 0
    pb.table.kind = L.HT_BITMAP; pb.table.vals = 0x9000; pb.table.cap = 1 << 16
    S = P.sink
    if sink == "count":
        S.kind = L.SINK_COUNT; S.count = 0xc000
    elif sink == "bitmap":
        S.kind = L.SINK_BITMAP; S.gkey.n = 1; S.gkey.slot[0] = 0; S.gkey.bits[0] = 28
        S.gkey.lo[0] = 1; S.gkeys = 0x1000; S.gcap = 1 << 28
    elif sink == "dense":
        S.kind = L.SINK_AGG_DENSE; S.n_cells = 1; S.n_measures = 1    # register accumulators
        m = S.m[0]; m.op = L.AGG_SUM; m.n_terms = 1; m.cond_atom = -1
        t = m.t[0]; t.coef = 1; t.n_factors = 1
        t.f[0].a, t.f[0].b, t.f[0].slot, t.f[0]._pad = 0, 1, 2, 1
        S.acc = 0x900000
    return P


@pytest.mark.parametrize("sink", ["compact", "count", "dense", "bitmap"])
def test_chunk_mode_levels_compile(lib, sink, monkeypatch):
    monkeypatch.setenv("SCX_CHUNK", "2")      # bitmap sinks only when forced
    P = _chunk_two_probes(sink)
    n = lib.scx_pipeline_source(C.byref(P), None, 0)
    assert n > 0, lib.scx_last_error()
    buf = C.create_string_buffer(n + 1)
    lib.scx_pipeline_source(C.byref(P), buf, n + 1)
    src = buf.value.decode()
    assert "// level 2" in src and "__ballot_sync" in src
    assert lib.scx_pipeline_compile(C.byref(P)) == 0, lib.scx_last_error().decode()


def test_chunk_tile_follows_selectivity_hint(lib):
    def v_of(P):
        n = lib.scx_pipeline_source(C.byref(P), None, 0)
        buf = C.create_string_buffer(n + 1)
        lib.scx_pipeline_source(C.byref(P), buf, n + 1)
        return int(buf.value.decode().split("constexpr int V = ")[1].split(";")[0])
    P = _chunk_two_probes("count")
    P._pad = 3          # 3% survive the pre-predicate
    assert v_of(P) == 8
    P._pad = 60
    assert v_of(P) == 4


def test_selectivity_estimate():
    from paper_2506_09226_b200 import relops as R
    from paper_2506_09226_b200.data import generate
    from paper_2506_09226_b200.table import Column, ColumnTable, date_to_days
    li = generate(0.001, 0.0, 0).tables["lineitem"]
    v = R.as_view(ColumnTable({n: Column.from_host_lazy(hc) for n, hc in li.columns.items()}))
    sd = v["l_shipdate"]
    month = R.filter_table(v, (sd >= date_to_days("1995-09-01")) & (sd < date_to_days("1995-10-01")))
    assert 0.005 < R._first_stage_survival(month) < 0.02
    modes = R.filter_table(v, v.isin("l_shipmode", ["AIR", "MAIL"]))
    assert abs(R._first_stage_survival(modes) - 2 / 7) < 1e-9


def test_chunk_late_columns(lib):
    # one selective semi probe feeding an aggregate: only the probe key is
    # staged; the measure's columns are read for the survivors at level 1
    P = _compact_probe(L.HT_BITMAP, L.JOIN_SEMI)
    P.pre.n_atoms = 0; P.pre.clause_mask = 0
    P._pad = 4
    S = P.sink
    S.kind = L.SINK_AGG_DENSE; S.n_cells = 1; S.n_measures = 1
    m = S.m[0]; m.op = L.AGG_SUM; m.n_terms = 1; m.cond_atom = -1
    t = m.t[0]; t.coef = 1; t.n_factors = 2
    t.f[0].a, t.f[0].b, t.f[0].slot, t.f[0]._pad = 0, 1, 2, 1
    t.f[1].a, t.f[1].b, t.f[1].slot, t.f[1]._pad = 0, 1, 3, 1
    S.acc = 0x900000
    n = lib.scx_pipeline_source(C.byref(P), None, 0)
    assert n > 0, lib.scx_last_error()
    buf = C.create_string_buffer(n + 1)
    lib.scx_pipeline_source(C.byref(P), buf, n + 1)
    src = buf.value.decode()
    assert "// level 1" in src and "__ldg((const i32*)a.p[" in src
    assert src.count("bulk_g2s(ring") == 1          # the key column only
    assert lib.scx_pipeline_compile(C.byref(P)) == 0, lib.scx_last_error().decode()

"""ctypes binding of libscx.so (include/scx.h).

The library is loaded lazily on first use and the struct layouts are
cross-checked against ``scx_sizeof`` so a header/binding drift fails loudly.
There is no fallback: if the .so is missing, every operator raises
``ScxError`` (the product path never runs numpy in place of a kernel).
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libscx.so")

# ---- constants (scx.h) ---------------------------------------------------
SCX_I8, SCX_I16, SCX_I32, SCX_I64, SCX_U8, SCX_U16, SCX_F64, SCX_U32 = range(8)
MAX_BASE, MAX_SLOTS, MAX_ATOMS, MAX_SETWORDS, MAX_LUT = 12, 32, 40, 128, 512
MAX_PROBES, MAX_PAYLOAD, MAX_MEASURES, MAX_GKEYS, MAX_OUT, MAX_KEYS = 8, 6, 8, 4, 16, 4
MAX_POLYS = 4
ATOM_RANGE, ATOM_SET, ATOM_DIFF, ATOM_POLY = 0, 1, 2, 3
XFORM_NONE, XFORM_YEAR = 0, 1
JOIN_SEMI, JOIN_ANTI, JOIN_INNER, JOIN_LEFT = 0, 1, 2, 3
HT_HASH, HT_DIRECT, HT_BITMAP, HT_IDENTITY = 0, 1, 2, 3
AGG_SUM, AGG_COUNT, AGG_MIN, AGG_MAX = 0, 1, 2, 3
SINK_AGG_DENSE, SINK_AGG_HASH, SINK_COMPACT, SINK_COUNT, SINK_BITMAP = 0, 1, 2, 3, 4
PACK_FOR, PACK_DELTA, PACK_IOTA = 0, 1, 2
EMPTY_KEY = 0xFFFFFFFFFFFFFFFF
NO_ROW = 0xFFFFFFFF

ERRORS = {-1: "SCX_EINVAL", -2: "SCX_ECUDA", -3: "SCX_ECAPACITY", -4: "SCX_EUNSUPPORTED"}

i32, i64, u32, u64, i16 = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_int16


class ScxError(RuntimeError):
    """A libscx call failed (or the library is missing)."""


class Column_(C.Structure):
    _fields_ = [("ptr", u64), ("dtype", i32), ("_pad", i32)]


class Atom(C.Structure):
    _fields_ = [("op", i32), ("slot", i32), ("slot2", i32), ("clause", i32),
                ("set_word", i32), ("negate", i32), ("lo", i64), ("hi", i64)]


class Pred(C.Structure):
    _fields_ = [("first_atom", i32), ("n_atoms", i32), ("clause_mask", u32), ("_pad", i32)]


class Factor(C.Structure):
    _fields_ = [("a", i64), ("b", i64), ("slot", i32), ("_pad", i32)]


class Term(C.Structure):
    _fields_ = [("coef", i64), ("n_factors", i32), ("_pad", i32), ("f", Factor * 3)]


class Measure(C.Structure):
    _fields_ = [("op", i32), ("n_terms", i32), ("cond_atom", i32), ("_pad", i32),
                ("t", Term * 2)]


class KeySpec(C.Structure):
    _fields_ = [("n", i32), ("slot", i32 * MAX_KEYS), ("shift", i32 * MAX_KEYS),
                ("bits", i32 * MAX_KEYS), ("xform", i32), ("lo", i64 * MAX_KEYS)]


class Lookup(C.Structure):
    _fields_ = [("kind", i32), ("_pad", i32), ("keys", u64), ("vals", u64), ("cap", u64)]


class Probe(C.Structure):
    _fields_ = [("kind", i32), ("n_payload", i32), ("key", KeySpec), ("table", Lookup),
                ("payload", Column_ * MAX_PAYLOAD), ("payload_slot", i32 * MAX_PAYLOAD),
                ("after", Pred)]


class Sink(C.Structure):
    _fields_ = [("kind", i32), ("n_measures", i32), ("m", Measure * MAX_MEASURES),
                ("gkey", KeySpec), ("gcard", i32 * MAX_GKEYS), ("glut", i32 * MAX_GKEYS),
                ("n_cells", i32), ("n_out", i32), ("acc", u64), ("gkeys", u64),
                ("gcap", u64), ("flags", u64), ("out_slot", i32 * MAX_OUT),
                ("out", Column_ * MAX_OUT), ("status", u64), ("count", u64)]


class Pipeline(C.Structure):
    _fields_ = [("n_rows", i64), ("n_base", i32), ("n_slots", i32), ("n_probes", i32),
                ("_pad", i32), ("base", Column_ * MAX_BASE), ("slot_dtype", i32 * MAX_SLOTS),
                ("pre", Pred), ("post", Pred), ("probe", Probe * MAX_PROBES), ("sink", Sink),
                ("atoms", Atom * MAX_ATOMS), ("polys", Measure * MAX_POLYS),
                ("setwords", u32 * MAX_SETWORDS),
                ("lut", i16 * MAX_LUT)]


_SIZE_CHECK = [(0, Pipeline), (1, Probe), (2, Sink), (3, Measure), (4, Atom), (5, KeySpec),
               (6, Lookup), (7, Column_)]

# exported symbol -> (restype, argtypes)
_vp = C.c_void_p
_PROTOS = {
    "scx_last_error": (C.c_char_p, []),
    "scx_abi_version": (C.c_int, []),
    "scx_launch_count": (u64, []),
    "scx_sizeof": (i64, [C.c_int]),
    "scx_device_info": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "scx_pipeline_run": (C.c_int, [C.POINTER(Pipeline), _vp]),
    "scx_pipeline_status_words": (i64, [C.POINTER(Pipeline)]),
    "scx_pipeline_source": (i64, [C.POINTER(Pipeline), C.c_char_p, i64]),
    "scx_pipeline_compile": (C.c_int, [C.POINTER(Pipeline)]),
    "scx_jit_stats": (C.c_int, [C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]),
    "scx_jit_clear_plans": (C.c_int, []),
    "scx_lookup_clear": (C.c_int, [C.POINTER(Lookup), _vp]),
    "scx_lookup_build": (C.c_int, [C.POINTER(Lookup), C.POINTER(Column_), C.c_int,
                                   C.POINTER(KeySpec), i64, _vp, _vp]),
    "scx_dense_reduce": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), _vp, _vp]),
    "scx_hash_agg_compact": (C.c_int, [_vp, _vp, i64, C.c_int, _vp, _vp, _vp, _vp]),
    "scx_i128_narrow": (C.c_int, [_vp, _vp, i64, _vp, _vp, _vp]),
    "scx_direct_agg_workspace": (i64, [i64]),
    "scx_direct_agg_compact": (C.c_int, [_vp, _vp, i64, C.c_int, _vp, _vp, _vp, _vp, _vp]),
    "scx_sorted_rank_workspace": (i64, [i64]),
    "scx_sorted_rank": (C.c_int, [C.POINTER(Column_), i64, i64, _vp, _vp, _vp, _vp, _vp]),
    "scx_direct_agg_compact_having": (C.c_int, [_vp, i64, C.c_int, C.c_int, C.c_int, i64, i64,
                                                _vp, _vp, _vp, _vp, _vp]),
    "scx_bitmap_coarsen": (C.c_int, [_vp, i64, C.c_int, _vp, _vp]),
    "scx_range_hist": (C.c_int, [_vp, i64, u64, u64, C.c_int, _vp, _vp]),
    "scx_select_below_workspace": (i64, [i64]),
    "scx_select_below": (C.c_int, [_vp, i64, u64, _vp, _vp, _vp, _vp, _vp]),
    "scx_is_sorted": (C.c_int, [C.POINTER(Column_), i64, _vp, _vp]),
    "scx_sorted_group_agg": (C.c_int, [C.POINTER(Column_), C.POINTER(Column_), C.POINTER(C.c_int),
                                       C.c_int, i64, C.c_int, i64, i64, _vp, _vp, i64, _vp, _vp,
                                       _vp]),
    "scx_widen_u32": (C.c_int, [_vp, i64, _vp, _vp]),
    "scx_direct_agg_select_having": (C.c_int, [_vp, i64, C.c_int, C.c_int, C.c_int, i64, i64,
                                               _vp, _vp, _vp, _vp]),
    "scx_direct_agg_compact_counted": (C.c_int, [_vp, i64, C.c_int, C.c_int, _vp, _vp, _vp, _vp,
                                                 _vp]),
    "scx_unpack_key": (C.c_int, [_vp, i64, C.c_int, u64, i64, Column_, _vp]),
    "scx_fixed_to_f64": (C.c_int, [_vp, i64, i64, C.c_int, _vp, i64, _vp, _vp]),
    "scx_sort_workspace": (i64, [i64]),
    "scx_sort_pairs": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, i64, C.c_int, _vp, _vp]),
    "scx_encode_sort_key": (C.c_int, [Column_, _vp, i64, i64, C.c_int, C.c_int, C.c_int,
                                      _vp, _vp, C.c_int, _vp]),
    "scx_minmax": (C.c_int, [Column_, i64, _vp, _vp]),
    "scx_gather": (C.c_int, [Column_, _vp, i64, Column_, _vp]),
    "scx_iota": (C.c_int, [_vp, i64, _vp]),
    "scx_fill_rows": (C.c_int, [_vp, i64, C.c_int, C.POINTER(i64), _vp]),
    "scx_fill_i64": (C.c_int, [_vp, i64, i64, i64, _vp]),
    "scx_write_mapped": (C.c_int, [_vp, _vp, i64, _vp]),
    "scx_hash_keys": (C.c_int, [C.POINTER(Column_), C.c_int, i64, _vp, _vp]),
    "scx_partition_workspace": (i64, [i64, C.c_int]),
    "scx_partition": (C.c_int, [C.POINTER(Column_), C.c_int, C.POINTER(Column_),
                                C.POINTER(Column_), C.c_int, i64, C.c_int, _vp, _vp, _vp]),
    "scx_part_workspace": (i64, [i64, C.c_int]),
    "scx_part_hist": (C.c_int, [C.POINTER(Column_), C.c_int, i64, C.c_int, _vp, _vp, _vp]),
    "scx_part_scatter": (C.c_int, [C.POINTER(Column_), C.c_int, C.POINTER(Column_), C.c_int, i64,
                                   C.c_int, _vp, _vp, _vp]),
    "scx_join_workspace": (i64, [i64]),
    "scx_join_match": (C.c_int, [_vp, i64, _vp, i64, _vp, _vp, _vp]),
    "scx_join_expand": (C.c_int, [_vp, i64, _vp, i64, _vp, _vp, _vp]),
    "scx_remap_codes": (C.c_int, [Column_, i64, _vp, C.c_int32, Column_, _vp, _vp]),
    "scx_nccl_version": (C.c_int, [C.POINTER(C.c_int)]),
    "scx_comm_id_bytes": (i64, []),
    "scx_comm_unique_id": (C.c_int, [_vp]),
    "scx_comm_init_rank": (C.c_int, [C.POINTER(_vp), C.c_int, _vp, C.c_int]),
    "scx_comm_init_all": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(_vp)]),
    "scx_comm_destroy": (C.c_int, [_vp]),
    "scx_alltoallv": (C.c_int, [_vp, _vp, C.POINTER(i64), C.POINTER(i64), _vp, C.POINTER(i64),
                                C.POINTER(i64), C.c_int, _vp]),
    "scx_bcast_group": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(i64), C.c_int, _vp]),
    "scx_allreduce_i64": (C.c_int, [_vp, _vp, _vp, i64, C.c_int, _vp]),
    "scx_gather_to0": (C.c_int, [_vp, _vp, i64, C.POINTER(_vp), C.POINTER(i64), _vp]),
    "scx_pack_words": (i64, [i64, C.c_int]),
    "scx_pack_delta_block": (i64, []),
    "scx_pack_host": (C.c_int, [_vp, C.c_int, i64, i64, C.c_int, C.c_int, _vp, _vp, C.c_int]),
    "scx_unpack": (C.c_int, [_vp, i64, C.c_int, i64, C.c_int, _vp, Column_, _vp]),
    "scx_unpack_diff": (C.c_int, [_vp, i64, C.c_int, i64, Column_, Column_, _vp]),
    "scx_unpack_fkdiff": (C.c_int, [_vp, i64, C.c_int, i64, Column_, i64, Column_, i64, Column_,
                                    _vp]),
    "scx_unpack_fkidx": (C.c_int, [_vp, i64, C.c_int, Column_, i64, i64, Column_, i64, Column_,
                                   _vp]),
}

EXPORTS = tuple(_PROTOS)

_lock = threading.Lock()
_lib = None


def load() -> C.CDLL:
    """Load and validate libscx.so; raises ScxError if absent or mismatched."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ScxError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2506_09226_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _PROTOS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        for which, cls in _SIZE_CHECK:
            got = lib.scx_sizeof(which)
            if got != C.sizeof(cls):
                raise ScxError(f"ABI mismatch: {cls.__name__} is {C.sizeof(cls)} B in ctypes, "
                               f"{got} B in libscx.so")
        _lib = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().scx_last_error().decode(errors="replace")
        raise ScxError(f"{what} failed: {ERRORS.get(rc, rc)}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


_TC = None


def stream_ptr(stream=None) -> C.c_void_p:
    """cudaStream_t of the given torch stream (current stream by default).

    The current stream is read through torch's C entry points: the Python
    torch.cuda.current_stream() wrapper cost ~15 us per kernel launch."""
    global _TC
    if stream is not None:
        return C.c_void_p(stream.cuda_stream)
    if _TC is None:
        import torch
        _TC = torch._C
    return C.c_void_p(_TC._cuda_getCurrentRawStream(_TC._cuda_getDevice()))

// pipeline.cu -- the fused scan pipeline (scx_pipeline_run).
//
// Persistent CTAs (occupancy x SMs) walk row tiles of a columnar table.
// Thread 0 of each CTA streams the touched columns of upcoming tiles into a
// ring of shared-memory stages with cp.async.bulk (TMA bulk copies, mbarrier
// complete_tx): whole-tile, fully coalesced, asynchronous HBM reads of the
// narrowed columns.  All 256 threads then run the query fragment
// column-at-a-time over the staged tile, R rows per thread:
//
//   pre-predicate   DNF over range / dictionary-set / column-difference atoms;
//                   each atom yields an R-bit mask (32-bit compares on the
//                   narrowed values, dtype dispatch hoisted out of the rows)
//   probes          up to 3 semi / anti / unique-inner lookups (direct or
//                   open-addressing tables); inner joins gather build-side
//                   payload columns into extra smem operand slots
//   post-predicate  same atoms, may reference payload slots
//   sink            dense group-by (per-thread register pre-aggregation, one
//                   128-bit global atomic per cell per CTA), hash group-by
//                   (global open addressing), stable compaction (decoupled
//                   look-back), or count
//
// Measures (sum_t coef * prod_f (a + b*v)) are evaluated in exact 64-bit
// fixed point.  On the fast path every factor fits int32 (host-proven from
// column ranges); its operand columns are widened once per tile into an
// int32 smem scratch so the unrolled per-measure code is switch-free.
//
// Replaces the numpy bodies of ColumnTable.filter/take (table.py:171-177),
// the driver predicates (queries.py:39,110-115,131-135,173,209-232),
// local_hash_join's probe (relops.py:73-94), group_aggregate
// (relops.py:97-160) and q1's np.add.at grid (queries.py:42-54).
#include <algorithm>
#include "common.cuh"

namespace scx {

#define SCX_DISPATCH(dt, ...)                                             \
  switch (dt) {                                                           \
    case SCX_I8:  { using T = int8_t;   __VA_ARGS__; } break;             \
    case SCX_I16: { using T = int16_t;  __VA_ARGS__; } break;             \
    case SCX_I32: { using T = int32_t;  __VA_ARGS__; } break;             \
    case SCX_U8:  { using T = uint8_t;  __VA_ARGS__; } break;             \
    case SCX_U16: { using T = uint16_t; __VA_ARGS__; } break;             \
    case SCX_U32: { using T = uint32_t; __VA_ARGS__; } break;             \
    default:      { using T = int64_t;  __VA_ARGS__; } break;             \
  }

// dtypes whose every value fits int32
#define SCX_DISPATCH32(dt, ...)                                           \
  switch (dt) {                                                           \
    case SCX_I8:  { using T = int8_t;   __VA_ARGS__; } break;             \
    case SCX_I16: { using T = int16_t;  __VA_ARGS__; } break;             \
    case SCX_U8:  { using T = uint8_t;  __VA_ARGS__; } break;             \
    case SCX_U16: { using T = uint16_t; __VA_ARGS__; } break;             \
    default:      { using T = int32_t;  __VA_ARGS__; } break;             \
  }

__host__ __device__ inline bool fits32(int dt) {
  return dt == SCX_I8 || dt == SCX_I16 || dt == SCX_I32 || dt == SCX_U8 || dt == SCX_U16;
}

constexpr int kMaxWide = 8;    // measure operand columns widened per tile

struct KParams {
  int64_t n_tiles;
  uint32_t stage_bytes;     // bytes of one stage (all base columns)
  uint32_t payload_off;     // smem offset of payload slot arrays
  uint32_t wide_off;        // smem offset of the int32 widened operand scratch
  uint32_t table_off;       // smem offset of the generic dense table
  uint32_t ring_off;        // smem offset of stage 0
  int32_t stages;
  int32_t n_wide;
  int32_t fast;             // measures on the int32 fast path
  uint32_t slot_off[SCX_MAX_SLOTS];  // base: offset within a stage; payload: absolute
  uint32_t base_col_off[SCX_MAX_BASE];
  int32_t wide_slot[kMaxWide];
  int8_t widx[SCX_MAX_SLOTS];        // slot -> wide index (or -1)
};

// fixed smem header
struct Header {
  uint64_t mbar[8];
  int32_t wcount[8 * kWarps];
  int64_t excl;
  uint32_t setwords[SCX_MAX_SETWORDS];
  int16_t lut[SCX_MAX_LUT];
};

template <int R>
struct Tile {
  static constexpr int kRows = kBlock * R;
  const char* stage;      // current stage base
  char* payload;          // payload base
  const int32_t* wide;    // widened operand scratch
  const KParams* kp;
  const scx_pipeline* P;
  __device__ __forceinline__ const char* slot_ptr(int s) const {
    return (s < P->n_base ? stage : payload) + kp->slot_off[s];
  }
  __device__ __forceinline__ int row(int r) const { return r * kBlock + threadIdx.x; }
  __device__ __forceinline__ const int32_t* wcol(int slot) const {
    return wide + kp->widx[slot] * kRows;
  }
};

// ---------------------------------------------------------------------------
// predicates: every atom yields an R-bit mask
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ uint32_t atom_mask(const Tile<R>& t, const scx_atom& A,
                                              const uint32_t* setw) {
  constexpr uint32_t kAll = (R == 32) ? 0xffffffffu : ((1u << R) - 1u);
  const int dt = t.P->slot_dtype[A.slot];
  const char* col = t.slot_ptr(A.slot);
  uint32_t m = 0;
  if (A.op == SCX_ATOM_RANGE) {
    if (fits32(dt)) {
      const int64_t lo = A.lo < (int64_t)INT32_MIN ? (int64_t)INT32_MIN : A.lo;
      const int64_t hi = A.hi > (int64_t)INT32_MAX ? (int64_t)INT32_MAX : A.hi;
      if (lo <= hi) {
        const int32_t lo32 = (int32_t)lo;
        const uint32_t span = (uint32_t)(hi - lo);
        SCX_DISPATCH32(dt,
          const T* c = reinterpret_cast<const T*>(col);
_Pragma("unroll")
          for (int r = 0; r < R; ++r) {
            const int32_t v = (int32_t)c[t.row(r)];
            m |= ((uint32_t)(v - lo32) <= span ? 1u : 0u) << r;
          })
      }
    } else {
      const int64_t lo = A.lo, hi = A.hi;
      SCX_DISPATCH(dt,
        const T* c = reinterpret_cast<const T*>(col);
_Pragma("unroll")
        for (int r = 0; r < R; ++r) {
          const int64_t v = (int64_t)c[t.row(r)];
          m |= ((v >= lo) & (v <= hi) ? 1u : 0u) << r;
        })
    }
  } else if (A.op == SCX_ATOM_SET) {
    const uint32_t* w = setw + A.set_word;
    const uint32_t nbits = (uint32_t)A.lo * 32u;
    SCX_DISPATCH(dt,
      const T* c = reinterpret_cast<const T*>(col);
_Pragma("unroll")
      for (int r = 0; r < R; ++r) {
        const uint32_t v = (uint32_t)c[t.row(r)];
        const bool ok = v < nbits && ((w[v >> 5] >> (v & 31)) & 1u);
        m |= (ok ? 1u : 0u) << r;
      })
  } else {  // DIFF: v[slot] - v[slot2]
    const int dt2 = t.P->slot_dtype[A.slot2];
    const char* col2 = t.slot_ptr(A.slot2);
    const int64_t lo = A.lo, hi = A.hi;
    if (dt == dt2 && (dt == SCX_I16 || dt == SCX_I32)) {
      SCX_DISPATCH32(dt,
        const T* a = reinterpret_cast<const T*>(col);
        const T* b = reinterpret_cast<const T*>(col2);
_Pragma("unroll")
        for (int r = 0; r < R; ++r) {
          const int64_t v = (int64_t)a[t.row(r)] - (int64_t)b[t.row(r)];
          m |= ((v >= lo) & (v <= hi) ? 1u : 0u) << r;
        })
    } else {
_Pragma("unroll")
      for (int r = 0; r < R; ++r) {
        const int64_t v = load_i64(col, dt, t.row(r)) - load_i64(col2, dt2, t.row(r));
        m |= ((v >= lo) & (v <= hi) ? 1u : 0u) << r;
      }
    }
  }
  return A.negate ? (m ^ kAll) : m;
}

// DNF: atoms are emitted clause by clause; pass = OR_clause AND_atom mask
template <int R>
__device__ __forceinline__ uint32_t eval_pred(const Tile<R>& t, const scx_pred& pr,
                                              const uint32_t* setw, uint32_t sel) {
  if (pr.clause_mask == 0 || sel == 0) return sel;
  constexpr uint32_t kAll = (R == 32) ? 0xffffffffu : ((1u << R) - 1u);
  uint32_t pass = 0, cur = kAll;
  int clause = t.P->atoms[pr.first_atom].clause;
  for (int a = pr.first_atom; a < pr.first_atom + pr.n_atoms; ++a) {
    const scx_atom& A = t.P->atoms[a];
    if (A.clause != clause) {
      pass |= cur;
      cur = kAll;
      clause = A.clause;
    }
    cur &= atom_mask<R>(t, A, setw);
  }
  pass |= cur;
  return sel & pass;
}

// ---------------------------------------------------------------------------
// keys
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ bool pack_key(const Tile<R>& t, const scx_keyspec& K, int r,
                                         const int16_t* lut, const int32_t* glut,
                                         uint64_t& out) {
  uint64_t k = 0;
  bool in = true;
  for (int i = 0; i < K.n; ++i) {
    const int s = K.slot[i];
    int64_t v = load_i64(t.slot_ptr(s), t.P->slot_dtype[s], t.row(r)) - K.lo[i];
    if (glut && glut[i] >= 0) v = lut[glut[i] + v];
    const uint64_t u = static_cast<uint64_t>(v);
    if (K.bits[i] < 64 && (u >> K.bits[i]) != 0) in = false;
    k |= u << K.shift[i];
  }
  out = k;
  return in;
}

// ---------------------------------------------------------------------------
// probes
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ uint32_t run_probe(const Tile<R>& t, const scx_probe& pb,
                                              uint32_t sel) {
  if (sel == 0) return sel;
  uint64_t key[R];
  uint32_t idx[R];
  bool live[R];
_Pragma("unroll")
  for (int r = 0; r < R; ++r) {
    live[r] = (sel >> r) & 1u;
    idx[r] = SCX_NO_ROW;
    key[r] = 0;
    if (live[r]) live[r] = pack_key<R>(t, pb.key, r, nullptr, nullptr, key[r]);
  }
  const uint32_t* vals = reinterpret_cast<const uint32_t*>(pb.table.vals);
  if (pb.table.kind == SCX_HT_DIRECT) {
    const uint64_t cap = pb.table.cap;
_Pragma("unroll")
    for (int r = 0; r < R; ++r)
      if (live[r] && key[r] < cap) idx[r] = __ldg(vals + key[r]);
  } else {
    // 16-byte {key, row} slots (tables.cu lookup_build_kernel)
    const uint64_t* slots = reinterpret_cast<const uint64_t*>(pb.table.keys);
    const uint64_t mask = pb.table.cap - 1;
    uint64_t h[R], k0[R];
    // issue all first probes before resolving any (memory-level parallelism)
_Pragma("unroll")
    for (int r = 0; r < R; ++r) {
      h[r] = mix64(key[r]) & mask;
      k0[r] = live[r] ? __ldg(slots + 2 * h[r]) : SCX_EMPTY_KEY;
    }
_Pragma("unroll")
    for (int r = 0; r < R; ++r) {
      if (!live[r]) continue;
      uint64_t hh = h[r], kk = k0[r];
      while (kk != key[r] && kk != SCX_EMPTY_KEY) {
        hh = (hh + 1) & mask;
        kk = __ldg(slots + 2 * hh);
      }
      if (kk == key[r]) idx[r] = (uint32_t)__ldg(slots + 2 * hh + 1);
    }
  }
_Pragma("unroll")
  for (int r = 0; r < R; ++r) {
    const bool found = idx[r] != SCX_NO_ROW;
    const bool keep = (pb.kind == SCX_JOIN_ANTI) ? !found : found;
    if (((sel >> r) & 1u) && !keep) sel &= ~(1u << r);
  }
  if (pb.kind == SCX_JOIN_INNER) {
    for (int j = 0; j < pb.n_payload; ++j) {
      const scx_column& pc = pb.payload[j];
      char* dst = const_cast<char*>(t.slot_ptr(pb.payload_slot[j]));
      SCX_DISPATCH(pc.dtype,
        const T* src = reinterpret_cast<const T*>(pc.ptr);
        T* d = reinterpret_cast<T*>(dst);
_Pragma("unroll")
        for (int r = 0; r < R; ++r)
          if ((sel >> r) & 1u) d[t.row(r)] = __ldg(src + idx[r]);)
    }
  }
  return sel;
}

// ---------------------------------------------------------------------------
// measures
// ---------------------------------------------------------------------------
// generic: any dtype, 64-bit factors
template <int R>
__device__ __forceinline__ void measure_generic(const Tile<R>& t, const scx_measure& M,
                                                const uint32_t* setw, int64_t (&mv)[R]) {
_Pragma("unroll")
  for (int r = 0; r < R; ++r) mv[r] = (M.op == SCX_AGG_COUNT) ? 1 : 0;
  if (M.op != SCX_AGG_COUNT) {
    for (int ti = 0; ti < M.n_terms; ++ti) {
      const scx_term& T_ = M.t[ti];
      int64_t tv[R];
_Pragma("unroll")
      for (int r = 0; r < R; ++r) tv[r] = T_.coef;
      for (int fi = 0; fi < T_.n_factors; ++fi) {
        const scx_factor& F = T_.f[fi];
        const int64_t a = F.a, b = F.b;
        if (F.slot < 0) {
_Pragma("unroll")
          for (int r = 0; r < R; ++r) tv[r] *= a;
        } else {
          SCX_DISPATCH(t.P->slot_dtype[F.slot],
            const T* c = reinterpret_cast<const T*>(t.slot_ptr(F.slot));
_Pragma("unroll")
            for (int r = 0; r < R; ++r) tv[r] *= a + b * (int64_t)c[t.row(r)];)
        }
      }
_Pragma("unroll")
      for (int r = 0; r < R; ++r) mv[r] += tv[r];
    }
  }
  if (M.cond_atom >= 0) {
    const uint32_t ok = atom_mask<R>(t, t.P->atoms[M.cond_atom], setw);
_Pragma("unroll")
    for (int r = 0; r < R; ++r) mv[r] = ((ok >> r) & 1u) ? mv[r] : 0;
  }
}

// fast: all factors int32 (host-proven), operands read from the int32 scratch
template <int R>
__device__ __forceinline__ void measure_fast(const Tile<R>& t, const scx_measure& M,
                                             const uint32_t* setw, int64_t (&mv)[R]) {
  if (M.op == SCX_AGG_COUNT) {
_Pragma("unroll")
    for (int r = 0; r < R; ++r) mv[r] = 1;
  } else {
_Pragma("unroll")
    for (int r = 0; r < R; ++r) mv[r] = 0;
    for (int ti = 0; ti < M.n_terms; ++ti) {
      const scx_term& T_ = M.t[ti];
      const int nf = T_.n_factors;
      int64_t p[R];
      if (nf == 0) {
_Pragma("unroll")
        for (int r = 0; r < R; ++r) p[r] = T_.coef;
      } else {
        const scx_factor& F0 = T_.f[0];
        const int32_t a0 = (int32_t)F0.a, b0 = (int32_t)F0.b;
        const int32_t* c0 = t.wcol(F0.slot);
        int32_t f0[R];
_Pragma("unroll")
        for (int r = 0; r < R; ++r) f0[r] = a0 + b0 * c0[t.row(r)];
        if (nf == 1) {
_Pragma("unroll")
          for (int r = 0; r < R; ++r) p[r] = f0[r];
        } else {
          const scx_factor& F1 = T_.f[1];
          const int32_t a1 = (int32_t)F1.a, b1 = (int32_t)F1.b;
          const int32_t* c1 = t.wcol(F1.slot);
_Pragma("unroll")
          for (int r = 0; r < R; ++r) p[r] = (int64_t)f0[r] * (int64_t)(a1 + b1 * c1[t.row(r)]);
          if (nf == 3) {
            const scx_factor& F2 = T_.f[2];
            const int32_t a2 = (int32_t)F2.a, b2 = (int32_t)F2.b;
            const int32_t* c2 = t.wcol(F2.slot);
_Pragma("unroll")
            for (int r = 0; r < R; ++r) p[r] *= (int64_t)(a2 + b2 * c2[t.row(r)]);
          }
        }
        if (T_.coef != 1) {
          const int64_t cf = T_.coef;
_Pragma("unroll")
          for (int r = 0; r < R; ++r) p[r] *= cf;
        }
      }
_Pragma("unroll")
      for (int r = 0; r < R; ++r) mv[r] += p[r];
    }
  }
  if (M.cond_atom >= 0) {
    const uint32_t ok = atom_mask<R>(t, t.P->atoms[M.cond_atom], setw);
_Pragma("unroll")
    for (int r = 0; r < R; ++r) mv[r] = ((ok >> r) & 1u) ? mv[r] : 0;
  }
}

template <int R>
__device__ __forceinline__ void widen_operands(const Tile<R>& t, int32_t* wide) {
  for (int w = 0; w < t.kp->n_wide; ++w) {
    const int s = t.kp->wide_slot[w];
    int32_t* dst = wide + w * Tile<R>::kRows;
    SCX_DISPATCH32(t.P->slot_dtype[s],
      const T* c = reinterpret_cast<const T*>(t.slot_ptr(s));
_Pragma("unroll")
      for (int r = 0; r < R; ++r) dst[t.row(r)] = (int32_t)c[t.row(r)];)
  }
}

__device__ __forceinline__ int64_t agg_identity(int op) {
  return op == SCX_AGG_MIN ? INT64_MAX : (op == SCX_AGG_MAX ? INT64_MIN : 0);
}
__device__ __forceinline__ int64_t agg_combine(int op, int64_t a, int64_t b) {
  return op == SCX_AGG_MIN ? min(a, b) : (op == SCX_AGG_MAX ? max(a, b) : a + b);
}

// dense cell id per row: mixed radix of (value - lo) or string rank
template <int R>
__device__ __forceinline__ void dense_cells(const Tile<R>& t, const scx_sink& S,
                                            const int16_t* lut, int (&cell)[R]) {
_Pragma("unroll")
  for (int r = 0; r < R; ++r) cell[r] = 0;
  for (int i = 0; i < S.gkey.n; ++i) {
    const int s = S.gkey.slot[i];
    const int32_t lo = (int32_t)S.gkey.lo[i];
    const int card = S.gcard[i];
    const int16_t* l = S.glut[i] >= 0 ? lut + S.glut[i] : nullptr;
    SCX_DISPATCH(t.P->slot_dtype[s],
      const T* c = reinterpret_cast<const T*>(t.slot_ptr(s));
_Pragma("unroll")
      for (int r = 0; r < R; ++r) {
        int v = (int)((int64_t)c[t.row(r)] - lo);
        if (l) v = l[v];
        cell[r] = cell[r] * card + v;
      })
  }
}

// global flush of one (cell, measure) partial
__device__ __forceinline__ void flush_dense(const scx_sink& S, int cell, int m, int64_t v) {
  int64_t* acc = reinterpret_cast<int64_t*>(S.acc) + 2 * ((int64_t)cell * S.n_measures + m);
  const int op = S.m[m].op;
  if (op == SCX_AGG_MIN) {
    if (v != INT64_MAX) atomicMin(reinterpret_cast<long long*>(acc), (long long)v);
  } else if (op == SCX_AGG_MAX) {
    if (v != INT64_MIN) atomicMax(reinterpret_cast<long long*>(acc), (long long)v);
  } else {
    atomic_add_i128(acc, v);
  }
}

// ---------------------------------------------------------------------------
// the kernel
//   NC > 0 : dense sink, fast measures, register accumulators [NC][NM]
//   NC == 0: generic sinks (COUNT / COMPACT / HASH / dense via smem table)
// ---------------------------------------------------------------------------
template <int R, int NC, int NM>
__global__ void __launch_bounds__(kBlock, 2)
pipeline_kernel(const __grid_constant__ scx_pipeline P, const __grid_constant__ KParams K) {
  extern __shared__ __align__(128) char smem[];
  Header& H = *reinterpret_cast<Header*>(smem);
  constexpr int TILE = kBlock * R;
  const int tid = threadIdx.x;
  const scx_sink& S = P.sink;

  for (int i = tid; i < SCX_MAX_SETWORDS; i += kBlock) H.setwords[i] = P.setwords[i];
  for (int i = tid; i < SCX_MAX_LUT; i += kBlock) H.lut[i] = P.lut[i];
  int64_t* dtab = reinterpret_cast<int64_t*>(smem + K.table_off);   // generic dense table
  const bool dense_generic = (NC == 0 && S.kind == SCX_SINK_AGG_DENSE);
  if (dense_generic) {
    for (int i = tid; i < S.n_cells * S.n_measures; i += kBlock)
      dtab[i] = agg_identity(S.m[i % S.n_measures].op);
  }

  const int64_t my_tiles = (K.n_tiles > blockIdx.x)
                               ? (K.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (tid == 0) {
    for (int s = 0; s < K.stages; ++s) mbar_init(&H.mbar[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](int64_t k) {  // thread 0: stream tile k of this CTA into its stage
    const int s = (int)(k % K.stages);
    const int64_t tile = blockIdx.x + k * gridDim.x;
    const int64_t row0 = tile * TILE;
    const uint32_t rows = (uint32_t)min((int64_t)TILE, P.n_rows - row0);
    uint32_t total = 0;
    for (int c = 0; c < P.n_base; ++c)
      total += (rows * dtype_size_d(P.base[c].dtype) + 15u) & ~15u;
    mbar_arrive_expect_tx(&H.mbar[s], total);
    char* dst = smem + K.ring_off + (size_t)s * K.stage_bytes;
    for (int c = 0; c < P.n_base; ++c) {
      const uint32_t w = dtype_size_d(P.base[c].dtype);
      bulk_g2s(dst + K.base_col_off[c],
               reinterpret_cast<const char*>(P.base[c].ptr) + row0 * w,
               (rows * w + 15u) & ~15u, &H.mbar[s]);
    }
  };

  if (tid == 0) {
    const int64_t pre = min((int64_t)K.stages, my_tiles);
    for (int64_t k = 0; k < pre; ++k) issue(k);
  }

  // ---- sink state ----
  int64_t racc[NC > 0 ? NC : 1][NM > 0 ? NM : 1];
  if constexpr (NC > 0) {
_Pragma("unroll")
    for (int m = 0; m < NM; ++m) {
      const int64_t id = (m < S.n_measures) ? agg_identity(S.m[m].op) : 0;
_Pragma("unroll")
      for (int c = 0; c < NC; ++c) racc[c][m] = id;
    }
  }

  uint64_t count_local = 0;
  Tile<R> tl;
  tl.P = &P;
  tl.kp = &K;
  tl.payload = smem + K.payload_off;
  int32_t* wide = reinterpret_cast<int32_t*>(smem + K.wide_off);
  tl.wide = wide;

  for (int64_t k = 0; k < my_tiles; ++k) {
    const int s = (int)(k % K.stages);
    const uint32_t parity = (uint32_t)((k / K.stages) & 1);
    const int64_t tile = blockIdx.x + k * gridDim.x;
    const int64_t row0 = tile * TILE;
    const int64_t rows = min((int64_t)TILE, P.n_rows - row0);
    mbar_wait(&H.mbar[s], parity);
    tl.stage = smem + K.ring_off + (size_t)s * K.stage_bytes;

    uint32_t sel = 0;
_Pragma("unroll")
    for (int r = 0; r < R; ++r) sel |= (tl.row(r) < rows) ? (1u << r) : 0u;

    sel = eval_pred<R>(tl, P.pre, H.setwords, sel);
    for (int p = 0; p < P.n_probes; ++p) {
      sel = run_probe<R>(tl, P.probe[p], sel);
      sel = eval_pred<R>(tl, P.probe[p].after, H.setwords, sel);
    }
    sel = eval_pred<R>(tl, P.post, H.setwords, sel);

    if constexpr (NC > 0) {
      widen_operands<R>(tl, wide);
      int cell[R];
      dense_cells<R>(tl, S, H.lut, cell);
_Pragma("unroll")
      for (int m = 0; m < NM; ++m) {
        if (m < S.n_measures) {
          int64_t mv[R];
          measure_fast<R>(tl, S.m[m], H.setwords, mv);
          const int op = S.m[m].op;
          if (op == SCX_AGG_SUM || op == SCX_AGG_COUNT) {
_Pragma("unroll")
            for (int r = 0; r < R; ++r) {
              const int64_t v = ((sel >> r) & 1u) ? mv[r] : 0;
              if constexpr (NC == 1) {
                racc[0][m] += v;
              } else {
                // branch-free masked adds: a predicated `if (cell == c)` gets
                // rewritten into a dynamically indexed (local-memory) store
_Pragma("unroll")
                for (int c = 0; c < NC; ++c)
                  racc[c][m] += v & -(int64_t)(cell[r] == c);
              }
            }
          } else {
_Pragma("unroll")
            for (int r = 0; r < R; ++r) {
_Pragma("unroll")
              for (int c = 0; c < NC; ++c) {
                const int64_t take =
                    -(int64_t)(((sel >> r) & 1u) && (NC == 1 || cell[r] == c));
                const int64_t cand = agg_combine(op, racc[c][m], mv[r]);
                racc[c][m] = (cand & take) | (racc[c][m] & ~take);
              }
            }
          }
        }
      }
    } else {
      if (S.kind == SCX_SINK_COUNT) {
        count_local += __popc(sel);
      } else if (S.kind == SCX_SINK_AGG_DENSE) {   // generic dense: smem table atomics
        int cell[R];
        dense_cells<R>(tl, S, H.lut, cell);
        for (int m = 0; m < S.n_measures; ++m) {
          int64_t mv[R];
          measure_generic<R>(tl, S.m[m], H.setwords, mv);
          const int op = S.m[m].op;
_Pragma("unroll")
          for (int r = 0; r < R; ++r) {
            if (!((sel >> r) & 1u)) continue;
            long long* a = reinterpret_cast<long long*>(dtab + cell[r] * S.n_measures + m);
            if (op == SCX_AGG_MIN) atomicMin(a, (long long)mv[r]);
            else if (op == SCX_AGG_MAX) atomicMax(a, (long long)mv[r]);
            else atomicAdd(reinterpret_cast<unsigned long long*>(a), (unsigned long long)mv[r]);
          }
        }
      } else if (S.kind == SCX_SINK_AGG_HASH) {
        uint64_t* gkeys = reinterpret_cast<uint64_t*>(S.gkeys);
        int64_t* acc = reinterpret_cast<int64_t*>(S.acc);
        const uint64_t mask = S.gcap - 1;
        uint64_t slot[R];
_Pragma("unroll")
        for (int r = 0; r < R; ++r) {
          slot[r] = ~0ull;
          if (!((sel >> r) & 1u)) continue;
          uint64_t key;
          pack_key<R>(tl, S.gkey, r, H.lut, S.glut, key);
          uint64_t h = mix64(key) & mask;
          for (uint64_t probes = 0; probes <= mask; ++probes) {
            uint64_t cur = gkeys[h];
            if (cur == SCX_EMPTY_KEY) {
              cur = atomicCAS(reinterpret_cast<unsigned long long*>(gkeys + h),
                              SCX_EMPTY_KEY, key);
              if (cur == SCX_EMPTY_KEY) cur = key;
            }
            if (cur == key) { slot[r] = h; break; }
            h = (h + 1) & mask;
          }
          if (slot[r] == ~0ull) atomicOr(reinterpret_cast<unsigned int*>(S.flags), 1u);
        }
        if (K.fast) widen_operands<R>(tl, wide);
        for (int m = 0; m < S.n_measures; ++m) {
          int64_t mv[R];
          if (K.fast) measure_fast<R>(tl, S.m[m], H.setwords, mv);
          else measure_generic<R>(tl, S.m[m], H.setwords, mv);
          const int op = S.m[m].op;
_Pragma("unroll")
          for (int r = 0; r < R; ++r) {
            if (slot[r] == ~0ull) continue;
            long long* a = reinterpret_cast<long long*>(acc + slot[r] * S.n_measures + m);
            if (op == SCX_AGG_MIN) atomicMin(a, (long long)mv[r]);
            else if (op == SCX_AGG_MAX) atomicMax(a, (long long)mv[r]);
            else atomicAdd(reinterpret_cast<unsigned long long*>(a), (unsigned long long)mv[r]);
          }
        }
      } else {  // COMPACT: stable order via per-(sub-tile, warp) ballots + look-back
        const int lane = tid & 31, warp = tid >> 5;
        int rank_in_warp[R];
_Pragma("unroll")
        for (int r = 0; r < R; ++r) {
          const uint32_t b = __ballot_sync(0xffffffffu, (sel >> r) & 1u);
          rank_in_warp[r] = __popc(b & ((1u << lane) - 1u));
          if (lane == 0) H.wcount[r * kWarps + warp] = __popc(b);
        }
        __syncthreads();
        if (tid == 0) {
          int run = 0;
          for (int i = 0; i < R * kWarps; ++i) {
            const int c = H.wcount[i];
            H.wcount[i] = run;
            run += c;
          }
          // decoupled look-back over tiles
          uint64_t* status = reinterpret_cast<uint64_t*>(S.status);
          const uint64_t kA = 1ull << 62, kP = 2ull << 62, kV = (1ull << 62) - 1;
          const uint64_t agg = (uint64_t)run;
          uint64_t excl = 0;
          if (tile == 0) {
            st_release(status, kP | agg);
          } else {
            st_release(status + tile, kA | agg);
            int64_t j = tile - 1;
            while (true) {
              const uint64_t w = ld_acquire(status + j);
              const uint64_t f = w & ~kV;
              if (f == 0) continue;
              excl += w & kV;
              if (f == kP) break;
              --j;
            }
            st_release(status + tile, kP | (excl + agg));
          }
          if (tile == K.n_tiles - 1)
            *reinterpret_cast<unsigned long long*>(S.count) = excl + agg;
          H.excl = (int64_t)excl;
        }
        __syncthreads();
        const int64_t base = H.excl;
        for (int o = 0; o < S.n_out; ++o) {
          const int s2 = S.out_slot[o];
          const scx_column& oc = S.out[o];
          if (s2 < 0) {
_Pragma("unroll")
            for (int r = 0; r < R; ++r)
              if ((sel >> r) & 1u)
                store_i64(reinterpret_cast<void*>(oc.ptr), oc.dtype,
                          base + H.wcount[r * kWarps + warp] + rank_in_warp[r],
                          row0 + tl.row(r));
          } else {
            SCX_DISPATCH(oc.dtype,
              T* dst = reinterpret_cast<T*>(oc.ptr);
              const T* src = reinterpret_cast<const T*>(tl.slot_ptr(s2));
_Pragma("unroll")
              for (int r = 0; r < R; ++r)
                if ((sel >> r) & 1u)
                  dst[base + H.wcount[r * kWarps + warp] + rank_in_warp[r]] = src[tl.row(r)];)
          }
        }
      }
    }

    __syncthreads();  // stage s fully consumed (and wcount reusable)
    if (tid == 0 && k + K.stages < my_tiles) issue(k + K.stages);
  }

  // ---- sink epilogues ----
  if constexpr (NC > 0) {
    __syncthreads();
    int64_t* red = reinterpret_cast<int64_t*>(smem + K.ring_off);  // ring is free now
    const int lane = tid & 31, warp = tid >> 5;
_Pragma("unroll")
    for (int m = 0; m < NM; ++m) {
      if (m < S.n_measures) {
        const int op = S.m[m].op;
_Pragma("unroll")
        for (int c = 0; c < NC; ++c) {
          int64_t v = racc[c][m];
          v = (op == SCX_AGG_MIN) ? warp_min_i64(v)
            : (op == SCX_AGG_MAX) ? warp_max_i64(v) : warp_sum_i64(v);
          if (lane == 0) red[(warp * NC + c) * NM + m] = v;
        }
      }
    }
    __syncthreads();
    const int ncells = S.n_cells < NC ? S.n_cells : NC;
    for (int i = tid; i < ncells * NM; i += kBlock) {
      const int c = i / NM, m = i % NM;
      if (m >= S.n_measures) continue;
      const int op = S.m[m].op;
      // combine per-warp partials in 128 bits before the global atomic
      if (op == SCX_AGG_SUM || op == SCX_AGG_COUNT) {
        int64_t lo = 0, hi = 0;
        for (int w = 0; w < kWarps; ++w) {
          const int64_t v = red[(w * NC + c) * NM + m];
          const uint64_t s2 = (uint64_t)lo + (uint64_t)v;
          hi += (v < 0 ? -1 : 0) + (s2 < (uint64_t)lo ? 1 : 0);
          lo = (int64_t)s2;
        }
        int64_t* acc = reinterpret_cast<int64_t*>(S.acc) + 2 * ((int64_t)c * S.n_measures + m);
        // (lo, hi) is an exact 128-bit partial: add lo unsigned, carry into hi
        const uint64_t old = lo != 0 ? (uint64_t)atomicAdd(reinterpret_cast<unsigned long long*>(acc),
                                                           (unsigned long long)lo) : 0ull;
        const int64_t h = hi + ((lo != 0 && old + (uint64_t)lo < old) ? 1 : 0);
        if (h != 0) atomicAdd(reinterpret_cast<unsigned long long*>(acc + 1), (unsigned long long)h);
      } else {
        int64_t v = agg_identity(op);
        for (int w = 0; w < kWarps; ++w) v = agg_combine(op, v, red[(w * NC + c) * NM + m]);
        flush_dense(S, c, m, v);
      }
    }
  } else {
    if (S.kind == SCX_SINK_COUNT) {
      unsigned long long wsum = (unsigned long long)count_local;
_Pragma("unroll")
      for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
      if ((tid & 31) == 0 && wsum) atomicAdd(reinterpret_cast<unsigned long long*>(S.count), wsum);
    } else if (dense_generic) {
      __syncthreads();
      for (int i = tid; i < S.n_cells * S.n_measures; i += kBlock)
        flush_dense(S, i / S.n_measures, i % S.n_measures, dtab[i]);
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct Launch {
  int R;
  size_t smem;
  KParams K;
  int grid;
  int nc, nm;   // template selection
};

static int64_t dtype_absmax(int dt) {
  switch (dt) {
    case SCX_I8: return 128;
    case SCX_U8: return 255;
    case SCX_I16: return 32768;
    case SCX_U16: return 65535;
    default: return (int64_t)1 << 31;
  }
}

// fast-path check: every measure factor flagged narrow by the host (factor
// _pad = 1: |a + b*v| < 2^31 over the column's range) on an int32-fitting slot
static bool measures_fast(const scx_pipeline& P, int8_t* widx, int32_t* wide_slot, int& n_wide) {
  const scx_sink& S = P.sink;
  n_wide = 0;
  for (int s = 0; s < SCX_MAX_SLOTS; ++s) widx[s] = -1;
  for (int m = 0; m < S.n_measures; ++m) {
    const scx_measure& M = S.m[m];
    if (M.op == SCX_AGG_COUNT) continue;
    if (M.n_terms < 0 || M.n_terms > 2) return false;
    for (int t = 0; t < M.n_terms; ++t) {
      const scx_term& T = M.t[t];
      if (T.n_factors < 0 || T.n_factors > 3) return false;
      for (int f = 0; f < T.n_factors; ++f) {
        const scx_factor& F = T.f[f];
        if (F.slot < 0 || F.slot >= P.n_slots) return false;
        if (!fits32(P.slot_dtype[F.slot]) || F._pad != 1) return false;
        if (F.a > INT32_MAX || F.a < INT32_MIN || F.b > INT32_MAX || F.b < INT32_MIN) return false;
        (void)dtype_absmax;
        if (widx[F.slot] < 0) {
          if (n_wide >= kMaxWide) return false;
          widx[F.slot] = (int8_t)n_wide;
          wide_slot[n_wide++] = F.slot;
        }
      }
    }
  }
  return true;
}

static int plan_launch(const scx_pipeline& P, Launch& L) {
  if (P.n_base < 0 || P.n_base > SCX_MAX_BASE || P.n_slots > SCX_MAX_SLOTS ||
      P.n_probes < 0 || P.n_probes > SCX_MAX_PROBES) {
    set_error("pipeline: descriptor counts out of range (base=%d slots=%d probes=%d)",
              P.n_base, P.n_slots, P.n_probes);
    return SCX_EINVAL;
  }
  // the interpreter predates poly atoms, key transforms and left joins
  for (int a = 0; a < SCX_MAX_ATOMS; ++a)
    if (P.atoms[a].op == SCX_ATOM_POLY) {
      set_error("interpreter: polynomial atoms need the JIT path (unset SCX_JIT=0)");
      return SCX_EUNSUPPORTED;
    }
  if (P.sink.kind == SCX_SINK_BITMAP) {
    set_error("interpreter: bitmap sinks need the JIT path (unset SCX_JIT=0)");
    return SCX_EUNSUPPORTED;
  }
  for (int p = 0; p < P.n_probes; ++p)
    if (P.probe[p].kind == SCX_JOIN_LEFT || P.probe[p].table.kind >= SCX_HT_BITMAP) {
      set_error("interpreter: left joins need the JIT path (unset SCX_JIT=0)");
      return SCX_EUNSUPPORTED;
    }
  if (P.sink.gkey.xform != 0) {
    set_error("interpreter: key transforms need the JIT path (unset SCX_JIT=0)");
    return SCX_EUNSUPPORTED;
  }
  uint32_t row_bytes = 0;
  for (int c = 0; c < P.n_base; ++c) {
    if (P.base[c].ptr % 16 != 0) {
      set_error("pipeline: base column %d not 16-byte aligned", c);
      return SCX_EINVAL;
    }
    if (P.slot_dtype[c] != P.base[c].dtype) {
      set_error("pipeline: slot %d dtype %d != base column dtype %d", c, P.slot_dtype[c],
                P.base[c].dtype);
      return SCX_EINVAL;
    }
    row_bytes += dtype_size(P.base[c].dtype);
  }
  uint32_t payload_row_bytes = 0;
  for (int s = P.n_base; s < P.n_slots; ++s) payload_row_bytes += dtype_size(P.slot_dtype[s]);

  KParams& K = L.K;
  memset(&K, 0, sizeof(K));
  const scx_sink& S = P.sink;
  const bool aggs = S.kind == SCX_SINK_AGG_DENSE || S.kind == SCX_SINK_AGG_HASH;
  K.fast = aggs && measures_fast(P, K.widx, K.wide_slot, K.n_wide) ? 1 : 0;
  if (!K.fast) {
    K.n_wide = 0;
    for (int s = 0; s < SCX_MAX_SLOTS; ++s) K.widx[s] = -1;
  }
  // template: register dense sinks need the fast measure path
  L.nc = 0;
  L.nm = 0;
  if (S.kind == SCX_SINK_AGG_DENSE && K.fast) {
    if (S.n_cells <= 1 && S.n_measures <= 8) { L.nc = 1; L.nm = 8; }
    else if (S.n_cells <= 8 && S.n_measures <= 6) { L.nc = 8; L.nm = 6; }
  }
  size_t dense_tbl = 0;
  if (S.kind == SCX_SINK_AGG_DENSE && L.nc == 0) {
    dense_tbl = (size_t)S.n_cells * S.n_measures * 8;
    if (dense_tbl > 64 * 1024) {
      set_error("pipeline: dense sink with %d cells x %d measures exceeds the smem table",
                S.n_cells, S.n_measures);
      return SCX_EUNSUPPORTED;
    }
  }

  int dev = 0;
  SCX_CUDA(cudaGetDevice(&dev));
  int smem_optin = 0, sms = 0, smem_sm = 0;
  SCX_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  SCX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  SCX_CUDA(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));

  const size_t header = (sizeof(Header) + 127) & ~size_t(127);
  auto round128 = [](size_t x) { return (x + 127) & ~size_t(127); };
  // target two resident CTAs per SM (16 warps) when the footprint allows
  const size_t budget2 = (size_t)smem_sm / 2 - 2048;
  const size_t budget1 = (size_t)smem_optin - 1024;
  int R = 0;
  size_t budget = budget2;
  for (int pass = 0; pass < 2 && R == 0; ++pass) {
    budget = pass == 0 ? budget2 : budget1;
    // register budget at 2 CTAs/SM (128 regs): [8 cells x 6] accumulators
    // leave room for R=2 rows/thread without spills, [1 x 8] for R=4
    for (int r = (L.nc == 8 ? 2 : (L.nc ? 4 : 8)); r >= 1; r >>= 1) {
      const size_t tile = (size_t)kBlock * r;
      const size_t stage = tile * row_bytes + 16 * P.n_base;
      const size_t fixed = header + round128(tile * payload_row_bytes + 16 * SCX_MAX_SLOTS) +
                           round128(tile * 4 * K.n_wide) + round128(dense_tbl);
      if (fixed + 2 * stage <= budget) { R = r; break; }
    }
  }
  if (R == 0) {
    set_error("pipeline: row too wide (%u B base + %u B payload)", row_bytes, payload_row_bytes);
    return SCX_EUNSUPPORTED;
  }
  const size_t tile = (size_t)kBlock * R;
  uint32_t off = 0;
  for (int c = 0; c < P.n_base; ++c) {
    K.base_col_off[c] = off;
    K.slot_off[c] = off;
    off += (uint32_t)((tile * dtype_size(P.base[c].dtype) + 15) & ~size_t(15));
  }
  K.stage_bytes = (off + 127) & ~127u;
  K.payload_off = (uint32_t)header;
  uint32_t poff = (uint32_t)header;
  for (int s = P.n_base; s < P.n_slots; ++s) {
    K.slot_off[s] = poff - K.payload_off;
    poff += (uint32_t)((tile * dtype_size(P.slot_dtype[s]) + 15) & ~size_t(15));
  }
  poff = (uint32_t)round128(poff);
  K.wide_off = poff;
  poff += (uint32_t)round128(tile * 4 * K.n_wide);
  K.table_off = poff;
  poff += (uint32_t)round128(dense_tbl);
  K.ring_off = poff;
  const size_t avail = budget > poff ? budget - poff : 0;
  int stages = K.stage_bytes ? (int)(avail / K.stage_bytes) : 2;
  if (stages > 6) stages = 6;
  if (stages < 1) stages = 1;
  // keep <= ~64 KB per CTA in flight: two resident CTAs cover HBM latency
  while (stages > 2 && (size_t)stages * K.stage_bytes > 64 * 1024) --stages;
  K.stages = stages;
  K.n_tiles = (P.n_rows + (int64_t)tile - 1) / (int64_t)tile;
  L.smem = K.ring_off + (size_t)stages * K.stage_bytes;
  L.R = R;
  L.grid = sms;   // refined with the occupancy query at launch
  return SCX_OK;
}

template <int R, int NC, int NM>
static int launch_one(const scx_pipeline& P, const Launch& L, cudaStream_t st) {
  auto kern = pipeline_kernel<R, NC, NM>;
  SCX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem));
  int occ = 0;
  SCX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kBlock, L.smem));
  if (occ < 1) {
    set_error("pipeline: kernel does not fit an SM (smem %zu)", L.smem);
    return SCX_EUNSUPPORTED;
  }
  // all CTAs co-resident: required by the compaction look-back
  const int64_t grid = std::min<int64_t>(L.K.n_tiles, (int64_t)L.grid * occ);
  kern<<<(int)grid, kBlock, L.smem, st>>>(P, L.K);
  SCX_CHECK_LAUNCH("pipeline_kernel");
  return SCX_OK;
}

template <int NC, int NM>
static int launch_r(const scx_pipeline& P, const Launch& L, cudaStream_t st) {
  switch (L.R) {
    case 8: return launch_one<8, NC, NM>(P, L, st);
    case 4: return launch_one<4, NC, NM>(P, L, st);
    case 2: return launch_one<2, NC, NM>(P, L, st);
    default: return launch_one<1, NC, NM>(P, L, st);
  }
}

}  // namespace scx

namespace scx {
// descriptor-interpreting path (SCX_JIT=0): kept as an A/B baseline for the
// plan-specialised kernels in jit.cu
int64_t interp_status_words(const scx_pipeline* d) {
  if (!d) return 0;
  scx::Launch L;
  if (scx::plan_launch(*d, L) != SCX_OK) return -1;
  return L.K.n_tiles;
}

int interp_pipeline_run(const scx_pipeline* d, void* stream) {
  if (!d) { set_error("pipeline: null descriptor"); return SCX_EINVAL; }
  const scx_pipeline& P = *d;
  if (P.n_rows < 0) { set_error("pipeline: negative n_rows"); return SCX_EINVAL; }
  if (P.n_rows == 0) {
    if (P.sink.kind == SCX_SINK_COMPACT || P.sink.kind == SCX_SINK_COUNT) {
      if (P.sink.count) SCX_CUDA(cudaMemsetAsync(reinterpret_cast<void*>(P.sink.count), 0, 8,
                                                 (cudaStream_t)stream));
    }
    return SCX_OK;
  }
  if (P.sink.kind == SCX_SINK_AGG_DENSE && P.sink.n_cells < 1) {
    set_error("pipeline: dense sink needs n_cells >= 1");
    return SCX_EINVAL;
  }
  if (P.sink.n_measures > SCX_MAX_MEASURES || P.sink.n_out > SCX_MAX_OUT) {
    set_error("pipeline: too many measures/outputs");
    return SCX_EINVAL;
  }
  Launch L;
  int rc = plan_launch(P, L);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  if (L.nc == 1) return launch_r<1, 8>(P, L, st);
  if (L.nc == 8) return launch_r<8, 6>(P, L, st);
  return launch_r<0, 0>(P, L, st);
}
}  // namespace scx

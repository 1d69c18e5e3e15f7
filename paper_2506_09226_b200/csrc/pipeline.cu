// pipeline.cu -- the fused scan pipeline (scx_pipeline_run).
//
// One persistent CTA per SM walks row tiles of a columnar table.  Thread 0
// streams the touched columns of upcoming tiles into a ring of shared-memory
// stages with cp.async.bulk (TMA bulk copies, mbarrier complete_tx), so HBM
// reads are whole-tile, fully coalesced and asynchronous.  All 256 threads
// then run the query fragment column-at-a-time over the staged tile:
//
//   pre-predicate (DNF of range / dictionary-set / column-difference atoms)
//   -> up to 3 probe stages (semi / anti / unique-inner lookups, payload
//      columns gathered into extra operand slots)
//   -> post-predicate
//   -> sink: dense group-agg (register pre-aggregation, one 128-bit global
//      atomic per cell per CTA), hash group-agg (global open addressing),
//      stable compaction (decoupled look-back) or count.
//
// Replaces the numpy bodies of ColumnTable.filter/take (table.py:171-177),
// the driver predicates (queries.py:39,110-115,131-135,173,209-232),
// local_hash_join's probe (relops.py:73-94), group_aggregate
// (relops.py:97-160) and q1's np.add.at grid (queries.py:42-54).
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

struct KParams {
  int64_t n_tiles;
  uint32_t stage_bytes;     // bytes of one stage (all base columns)
  uint32_t payload_off;     // smem offset of payload slot arrays
  uint32_t ring_off;        // smem offset of stage 0
  int32_t stages;
  uint32_t slot_off[SCX_MAX_SLOTS];  // base: offset within a stage; payload: absolute
  uint32_t base_col_off[SCX_MAX_BASE];
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
  const KParams* kp;
  const scx_pipeline* P;
  __device__ __forceinline__ const char* slot_ptr(int s) const {
    return (s < P->n_base ? stage : payload) + kp->slot_off[s];
  }
  __device__ __forceinline__ int row(int r) const { return r * kBlock + threadIdx.x; }
};

// ---------------------------------------------------------------------------
// predicate evaluation (column at a time; dtype switch hoisted out of rows)
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ void eval_atom(const Tile<R>& t, const scx_atom& A,
                                          const uint32_t* setw, bool (&ok)[R]) {
  const int dt = t.P->slot_dtype[A.slot];
  const char* col = t.slot_ptr(A.slot);
  if (A.op == SCX_ATOM_RANGE) {
    const int64_t lo = A.lo, hi = A.hi;
    SCX_DISPATCH(dt,
      const T* c = reinterpret_cast<const T*>(col);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        int64_t v = (int64_t)c[t.row(r)];
        ok[r] = (v >= lo) & (v <= hi);
      })
  } else if (A.op == SCX_ATOM_SET) {
    const uint32_t* w = setw + A.set_word;
    const int64_t nwords = A.lo;
    SCX_DISPATCH(dt,
      const T* c = reinterpret_cast<const T*>(col);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        int64_t v = (int64_t)c[t.row(r)];
        int64_t wi = v >> 5;
        ok[r] = (v >= 0) && (wi < nwords) && ((w[wi] >> (v & 31)) & 1u);
      })
  } else {  // DIFF
    const int dt2 = t.P->slot_dtype[A.slot2];
    const char* col2 = t.slot_ptr(A.slot2);
    const int64_t lo = A.lo, hi = A.hi;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      int64_t v = load_i64(col, dt, t.row(r)) - load_i64(col2, dt2, t.row(r));
      ok[r] = (v >= lo) & (v <= hi);
    }
  }
  if (A.negate) {
#pragma unroll
    for (int r = 0; r < R; ++r) ok[r] = !ok[r];
  }
}

template <int R>
__device__ __forceinline__ uint32_t eval_pred(const Tile<R>& t, const scx_pred& pr,
                                              const uint32_t* setw, uint32_t sel) {
  if (pr.clause_mask == 0 || sel == 0) return sel;
  uint32_t fail[R];
#pragma unroll
  for (int r = 0; r < R; ++r) fail[r] = 0;
  for (int a = pr.first_atom; a < pr.first_atom + pr.n_atoms; ++a) {
    const scx_atom& A = t.P->atoms[a];
    bool ok[R];
    eval_atom<R>(t, A, setw, ok);
    const uint32_t cbit = 1u << A.clause;
#pragma unroll
    for (int r = 0; r < R; ++r) fail[r] |= ok[r] ? 0u : cbit;
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (((~fail[r]) & pr.clause_mask) == 0) sel &= ~(1u << r);
  return sel;
}

// ---------------------------------------------------------------------------
// keys
// ---------------------------------------------------------------------------
// packed key of row r; returns false if a component is out of its range
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
#pragma unroll
  for (int r = 0; r < R; ++r) {
    live[r] = (sel >> r) & 1u;
    idx[r] = SCX_NO_ROW;
    if (live[r]) live[r] = pack_key<R>(t, pb.key, r, nullptr, nullptr, key[r]);
  }
  const uint32_t* vals = reinterpret_cast<const uint32_t*>(pb.table.vals);
  if (pb.table.kind == SCX_HT_DIRECT) {
    const uint64_t cap = pb.table.cap;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (live[r] && key[r] < cap) idx[r] = __ldg(vals + key[r]);
  } else {
    const uint64_t* keys = reinterpret_cast<const uint64_t*>(pb.table.keys);
    const uint64_t mask = pb.table.cap - 1;
    uint64_t h[R], k0[R];
    // issue all first probes before resolving any (memory-level parallelism)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      h[r] = mix64(key[r]) & mask;
      k0[r] = live[r] ? __ldg(keys + h[r]) : SCX_EMPTY_KEY;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (!live[r]) continue;
      uint64_t hh = h[r], kk = k0[r];
      while (kk != key[r] && kk != SCX_EMPTY_KEY) {
        hh = (hh + 1) & mask;
        kk = __ldg(keys + hh);
      }
      if (kk == key[r]) idx[r] = __ldg(vals + hh);
    }
  }
#pragma unroll
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
#pragma unroll
        for (int r = 0; r < R; ++r)
          if ((sel >> r) & 1u) d[t.row(r)] = __ldg(src + idx[r]);)
    }
  }
  return sel;
}

// ---------------------------------------------------------------------------
// measures: value per row = sum_t coef * prod_f (a + b*v), gated by cond
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ void eval_measure(const Tile<R>& t, const scx_measure& M,
                                             const uint32_t* setw, int64_t (&mv)[R]) {
#pragma unroll
  for (int r = 0; r < R; ++r) mv[r] = (M.op == SCX_AGG_COUNT) ? 1 : 0;
  if (M.op != SCX_AGG_COUNT) {
    for (int ti = 0; ti < M.n_terms; ++ti) {
      const scx_term& T_ = M.t[ti];
      int64_t tv[R];
#pragma unroll
      for (int r = 0; r < R; ++r) tv[r] = T_.coef;
      for (int fi = 0; fi < T_.n_factors; ++fi) {
        const scx_factor& F = T_.f[fi];
        const int64_t a = F.a, b = F.b;
        if (F.slot < 0) {
#pragma unroll
          for (int r = 0; r < R; ++r) tv[r] *= a;
        } else {
          SCX_DISPATCH(t.P->slot_dtype[F.slot],
            const T* c = reinterpret_cast<const T*>(t.slot_ptr(F.slot));
#pragma unroll
            for (int r = 0; r < R; ++r) tv[r] *= a + b * (int64_t)c[t.row(r)];)
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) mv[r] += tv[r];
    }
  }
  if (M.cond_atom >= 0) {
    bool ok[R];
    eval_atom<R>(t, t.P->atoms[M.cond_atom], setw, ok);
#pragma unroll
    for (int r = 0; r < R; ++r) mv[r] = ok[r] ? mv[r] : 0;
  }
}

__device__ __forceinline__ int64_t agg_identity(int op) {
  return op == SCX_AGG_MIN ? INT64_MAX : (op == SCX_AGG_MAX ? INT64_MIN : 0);
}
__device__ __forceinline__ int64_t agg_combine(int op, int64_t a, int64_t b) {
  return op == SCX_AGG_MIN ? min(a, b) : (op == SCX_AGG_MAX ? max(a, b) : a + b);
}

template <int R>
__device__ __forceinline__ int dense_cell(const Tile<R>& t, const scx_sink& S,
                                          const int16_t* lut, int r) {
  int cell = 0;
  for (int i = 0; i < S.gkey.n; ++i) {
    const int s = S.gkey.slot[i];
    int64_t v = load_i64(t.slot_ptr(s), t.P->slot_dtype[s], t.row(r)) - S.gkey.lo[i];
    if (S.glut[i] >= 0) v = lut[S.glut[i] + v];
    cell = cell * S.gcard[i] + (int)v;
  }
  return cell;
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
//   NC > 0 : dense sink with per-thread register accumulators [NC][NM]
//   NC == 0: generic sinks (COUNT / COMPACT / HASH / dense via smem atomics)
// ---------------------------------------------------------------------------
template <int R, int NC, int NM>
__global__ void __launch_bounds__(kBlock, 1)
pipeline_kernel(const __grid_constant__ scx_pipeline P, const __grid_constant__ KParams K) {
  extern __shared__ __align__(128) char smem[];
  Header& H = *reinterpret_cast<Header*>(smem);
  constexpr int TILE = kBlock * R;
  const int tid = threadIdx.x;
  const scx_sink& S = P.sink;

  for (int i = tid; i < SCX_MAX_SETWORDS; i += kBlock) H.setwords[i] = P.setwords[i];
  for (int i = tid; i < SCX_MAX_LUT; i += kBlock) H.lut[i] = P.lut[i];

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
    const int64_t rows = min((int64_t)TILE, P.n_rows - row0);
    uint32_t total = 0;
    uint32_t bytes[SCX_MAX_BASE];
    for (int c = 0; c < P.n_base; ++c) {
      const uint32_t w = dtype_size_d(P.base[c].dtype);
      bytes[c] = ((uint32_t)rows * w + 15u) & ~15u;
      total += bytes[c];
    }
    mbar_arrive_expect_tx(&H.mbar[s], total);
    char* dst = smem + K.ring_off + (size_t)s * K.stage_bytes;
    for (int c = 0; c < P.n_base; ++c) {
      const uint32_t w = dtype_size_d(P.base[c].dtype);
      bulk_g2s(dst + K.base_col_off[c],
               reinterpret_cast<const char*>(P.base[c].ptr) + row0 * w, bytes[c], &H.mbar[s]);
    }
  };

  if (tid == 0) {
    const int64_t pre = min((int64_t)K.stages, my_tiles);
    for (int64_t k = 0; k < pre; ++k) issue(k);
  }

  // ---- sink state ----
  int64_t racc[NC > 0 ? NC : 1][NM > 0 ? NM : 1];
  if constexpr (NC > 0) {
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      const int64_t id = (m < S.n_measures) ? agg_identity(S.m[m].op) : 0;
#pragma unroll
      for (int c = 0; c < NC; ++c) racc[c][m] = id;
    }
  }

  uint64_t count_local = 0;
  Tile<R> tl;
  tl.P = &P;
  tl.kp = &K;
  tl.payload = smem + K.payload_off;

  for (int64_t k = 0; k < my_tiles; ++k) {
    const int s = (int)(k % K.stages);
    const uint32_t parity = (uint32_t)((k / K.stages) & 1);
    const int64_t tile = blockIdx.x + k * gridDim.x;
    const int64_t row0 = tile * TILE;
    const int64_t rows = min((int64_t)TILE, P.n_rows - row0);
    mbar_wait(&H.mbar[s], parity);
    tl.stage = smem + K.ring_off + (size_t)s * K.stage_bytes;

    uint32_t sel = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) sel |= (tl.row(r) < rows) ? (1u << r) : 0u;

    sel = eval_pred<R>(tl, P.pre, H.setwords, sel);
    for (int p = 0; p < P.n_probes; ++p) sel = run_probe<R>(tl, P.probe[p], sel);
    sel = eval_pred<R>(tl, P.post, H.setwords, sel);

    if constexpr (NC > 0) {
      int cell[R];
#pragma unroll
      for (int r = 0; r < R; ++r) cell[r] = (S.gkey.n > 0) ? dense_cell<R>(tl, S, H.lut, r) : 0;
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        if (m < S.n_measures) {
          int64_t mv[R];
          eval_measure<R>(tl, S.m[m], H.setwords, mv);
          const int op = S.m[m].op;
          if (op == SCX_AGG_SUM || op == SCX_AGG_COUNT) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
              const int64_t v = ((sel >> r) & 1u) ? mv[r] : 0;
#pragma unroll
              for (int c = 0; c < NC; ++c) racc[c][m] += (cell[r] == c) ? v : 0;
            }
          } else {
#pragma unroll
            for (int r = 0; r < R; ++r)
              if ((sel >> r) & 1u) {
#pragma unroll
                for (int c = 0; c < NC; ++c)
                  if (cell[r] == c) racc[c][m] = agg_combine(op, racc[c][m], mv[r]);
              }
          }
        }
      }
    } else {
      if (S.kind == SCX_SINK_COUNT) {
        count_local += __popc(sel);
      } else if (S.kind == SCX_SINK_AGG_HASH) {
        uint64_t* gkeys = reinterpret_cast<uint64_t*>(S.gkeys);
        int64_t* acc = reinterpret_cast<int64_t*>(S.acc);
        const uint64_t mask = S.gcap - 1;
        uint64_t slot[R];
#pragma unroll
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
        for (int m = 0; m < S.n_measures; ++m) {
          int64_t mv[R];
          eval_measure<R>(tl, S.m[m], H.setwords, mv);
          const int op = S.m[m].op;
#pragma unroll
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
#pragma unroll
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
          const int s = S.out_slot[o];
          const scx_column& oc = S.out[o];
          if (s < 0) {
#pragma unroll
            for (int r = 0; r < R; ++r)
              if ((sel >> r) & 1u)
                store_i64(reinterpret_cast<void*>(oc.ptr), oc.dtype,
                          base + H.wcount[r * kWarps + warp] + rank_in_warp[r],
                          row0 + tl.row(r));
          } else {
            SCX_DISPATCH(oc.dtype,
              T* dst = reinterpret_cast<T*>(oc.ptr);
              const T* src = reinterpret_cast<const T*>(tl.slot_ptr(s));
#pragma unroll
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
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      if (m < S.n_measures) {
        const int op = S.m[m].op;
#pragma unroll
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
        if (lo != 0) atomic_add_i128(acc, lo);
        if (hi != 0) atomicAdd(reinterpret_cast<unsigned long long*>(acc + 1), (unsigned long long)hi);
      } else {
        int64_t v = agg_identity(op);
        for (int w = 0; w < kWarps; ++w) v = agg_combine(op, v, red[(w * NC + c) * NM + m]);
        flush_dense(S, c, m, v);
      }
    }
  } else {
    if (S.kind == SCX_SINK_COUNT) {
      __syncthreads();
      const unsigned long long c = (unsigned long long)count_local;
      unsigned long long wsum = c;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
      if ((tid & 31) == 0 && wsum) atomicAdd(reinterpret_cast<unsigned long long*>(S.count), wsum);
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
};

static int plan_launch(const scx_pipeline& P, Launch& L) {
  if (P.n_base < 0 || P.n_base > SCX_MAX_BASE || P.n_slots > SCX_MAX_SLOTS ||
      P.n_probes < 0 || P.n_probes > SCX_MAX_PROBES) {
    set_error("pipeline: descriptor counts out of range (base=%d slots=%d probes=%d)",
              P.n_base, P.n_slots, P.n_probes);
    return SCX_EINVAL;
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

  int dev = 0;
  SCX_CUDA(cudaGetDevice(&dev));
  int smem_optin = 0;
  SCX_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  int sms = 0;
  SCX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));

  const size_t header = (sizeof(Header) + 127) & ~size_t(127);
  const size_t dense_tbl = 0;
  const size_t budget = (size_t)smem_optin - 1024;

  // pick rows/thread: largest R whose ring (>= 2 stages) + payload fits
  int R = 8;
  for (; R >= 1; R >>= 1) {
    const size_t tile = (size_t)kBlock * R;
    const size_t stage = tile * row_bytes;
    const size_t pay = ((tile * payload_row_bytes + 127) & ~size_t(127)) + ((dense_tbl + 127) & ~size_t(127));
    if (header + pay + 2 * stage <= budget) break;
  }
  if (R < 1) {
    set_error("pipeline: row too wide (%u B base + %u B payload)", row_bytes, payload_row_bytes);
    return SCX_EUNSUPPORTED;
  }
  const size_t tile = (size_t)kBlock * R;
  KParams& K = L.K;
  memset(&K, 0, sizeof(K));
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
  poff = (poff + 127) & ~127u;
  K.ring_off = poff;
  const size_t avail = budget - poff;
  int stages = K.stage_bytes ? (int)(avail / K.stage_bytes) : 1;
  if (stages > 6) stages = 6;
  if (stages < 1) stages = 1;
  // keep ~96 KB in flight per SM; more stages do not help a streaming scan
  while (stages > 2 && (size_t)(stages - 1) * K.stage_bytes > 160 * 1024) --stages;
  K.stages = stages;
  K.n_tiles = (P.n_rows + (int64_t)tile - 1) / (int64_t)tile;
  L.smem = K.ring_off + (size_t)stages * K.stage_bytes;
  L.R = R;
  L.grid = (int)std::min<int64_t>(K.n_tiles, (int64_t)sms);
  return SCX_OK;
}

template <int R, int NC, int NM>
static int launch_one(const scx_pipeline& P, const Launch& L, cudaStream_t st) {
  auto kern = pipeline_kernel<R, NC, NM>;
  SCX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.smem));
  kern<<<L.grid, kBlock, L.smem, st>>>(P, L.K);
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


extern "C" int64_t scx_pipeline_status_words(const scx_pipeline* d) {
  if (!d) return 0;
  scx::Launch L;
  if (scx::plan_launch(*d, L) != SCX_OK) return -1;
  return L.K.n_tiles;
}

extern "C" int scx_pipeline_run(const scx_pipeline* d, void* stream) {
  using namespace scx;
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
  if (P.sink.kind == SCX_SINK_AGG_DENSE && P.sink.n_cells <= 1 && P.sink.n_measures <= 8)
    return launch_r<1, 8>(P, L, st);
  if (P.sink.kind == SCX_SINK_AGG_DENSE && P.sink.n_cells <= 8 && P.sink.n_measures <= 6)
    return launch_r<8, 6>(P, L, st);
  if (P.sink.kind == SCX_SINK_AGG_DENSE) {
    set_error("pipeline: dense sink with %d cells x %d measures not supported yet",
              P.sink.n_cells, P.sink.n_measures);
    return SCX_EUNSUPPORTED;
  }
  return launch_r<0, 0>(P, L, st);
}

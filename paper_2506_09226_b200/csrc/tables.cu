// tables.cu -- lookup-table build (join build side), group-table compaction,
// exact dense-aggregate reduction, key unpack, fixed-point -> f64, gather.
//
// Build side of local_hash_join (relops.py:81-84: the reference's stable
// argsort + searchsorted becomes an open-addressing insert), the output
// assembly of group_aggregate (relops.py:115-160) and Column.take
// (table.py:76-77).
#include <algorithm>

#include "common.cuh"

namespace scx {

// HASH tables are one array of 16-byte slots {u64 key, u64 row}: a probe
// reads key and row in one sector (separate key / row arrays cost a second
// dependent random access per hit).  DIRECT: vals[key] = row.
__global__ void lookup_clear_kernel(uint64_t* slots, uint32_t* vals, uint64_t cap) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (slots) {
      slots[2 * i] = SCX_EMPTY_KEY;
      slots[2 * i + 1] = SCX_NO_ROW;
    } else {
      vals[i] = SCX_NO_ROW;
    }
  }
}

struct BuildCols {
  scx_column c[SCX_MAX_KEYS];
};

__device__ __forceinline__ bool build_key(const BuildCols& C, const scx_keyspec& K, int64_t i,
                                          uint64_t& out) {
  uint64_t k = 0;
  bool in = true;
  for (int j = 0; j < K.n; ++j) {
    const scx_column& col = C.c[K.slot[j]];
    const uint64_t u = static_cast<uint64_t>(load_i64(reinterpret_cast<const void*>(col.ptr),
                                                      col.dtype, i) - K.lo[j]);
    if (K.bits[j] < 64 && (u >> K.bits[j]) != 0) in = false;
    k |= u << K.shift[j];
  }
  out = k;
  return in;
}

__global__ void lookup_build_kernel(scx_lookup T, BuildCols C, scx_keyspec K, int64_t n,
                                    uint32_t* flags) {
  uint32_t* vals = reinterpret_cast<uint32_t*>(T.vals);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t key;
    if (!build_key(C, K, i, key)) { atomicOr(flags + 2, 1u); continue; }
    // clustered build sides (lineitem by orderkey) repeat keys in runs: the
    // first row of a run inserts, the rest only report the duplicate
    uint64_t prev;
    if (i > 0 && build_key(C, K, i - 1, prev) && prev == key) { atomicOr(flags + 1, 1u); continue; }
    if (T.kind == SCX_HT_BITMAP) {
      if (key >= T.cap) { atomicOr(flags + 2, 1u); continue; }
      atomicOr(vals + (key >> 5), 1u << (key & 31));
    } else if (T.kind == SCX_HT_DIRECT) {
      if (key >= T.cap) { atomicOr(flags + 2, 1u); continue; }
      const uint32_t prev = atomicExch(vals + key, (uint32_t)i);
      if (prev != SCX_NO_ROW) atomicOr(flags + 1, 1u);
    } else {
      uint64_t* slots = reinterpret_cast<uint64_t*>(T.keys);
      const uint64_t mask = T.cap - 1;
      uint64_t h = mix64(key) & mask;
      for (uint64_t p = 0; p <= mask; ++p) {
        const unsigned long long prev =
            atomicCAS(reinterpret_cast<unsigned long long*>(slots + 2 * h), SCX_EMPTY_KEY, key);
        if (prev == SCX_EMPTY_KEY) { slots[2 * h + 1] = (uint64_t)i; break; }
        if (prev == key) { atomicOr(flags + 1, 1u); break; }   // duplicate key
        h = (h + 1) & mask;
      }
    }
  }
}

// exact reduction of n_ranks partial {lo,hi} accumulators into 3 x 42-bit
// signed limbs is unnecessary on one device: we emit {lo, hi} summed.
struct ReduceOps {
  int8_t op[SCX_MAX_MEASURES];             // 0 = 128-bit sum, 1 = min, 2 = max
};

// Cross-rank fold of dense group-by accumulators: cell (c, m) is an exact
// {lo, hi} 128-bit sum, or for a min / max measure an int64 in lo (hi = 0).
__global__ void dense_reduce_kernel(const int64_t* acc, int n_ranks, int64_t words, int m,
                                    ReduceOps ops, int64_t* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= words / 2) return;
  const int op = ops.op[i % m];
  if (op != 0) {
    int64_t v = acc[2 * i];
    for (int r = 1; r < n_ranks; ++r) {
      const int64_t x = acc[r * words + 2 * i];
      v = op == 1 ? (x < v ? x : v) : (x > v ? x : v);
    }
    out[2 * i] = v;
    out[2 * i + 1] = 0;
    return;
  }
  uint64_t lo = 0;
  int64_t hi = 0;
  for (int r = 0; r < n_ranks; ++r) {
    const uint64_t l = (uint64_t)acc[r * words + 2 * i];
    const int64_t h = acc[r * words + 2 * i + 1];
    const uint64_t s = lo + l;
    hi += h + (s < lo ? 1 : 0);
    lo = s;
  }
  out[2 * i] = (int64_t)lo;
  out[2 * i + 1] = hi;
}

// Occupied slots of an open-addressing group table -> dense (key, measures)
// arrays (any order; the caller sorts when the output must be ordered).  A
// CTA reserves its output range with ONE atomic per 2048 slots: a per-warp
// atomic on the single counter serialised at L2 (Q16: 32M slots, 0.79 ms).
constexpr int kCompactPer = 8;
__global__ void __launch_bounds__(256) hash_agg_compact_kernel(
    const uint64_t* __restrict__ gkeys, const int64_t* __restrict__ acc, int64_t cap, int m,
    uint64_t* __restrict__ out_keys, int64_t* __restrict__ out_acc, unsigned long long* count) {
  __shared__ uint32_t wsum[8];
  __shared__ unsigned long long cbase;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t span = 256 * kCompactPer;
  for (int64_t base = blockIdx.x * span; base < cap; base += (int64_t)gridDim.x * span) {
    uint64_t k[kCompactPer];
    uint32_t masks[kCompactPer];
    uint32_t mine = 0;
#pragma unroll
    for (int s = 0; s < kCompactPer; ++s) {
      const int64_t i = base + s * 256 + threadIdx.x;
      k[s] = i < cap ? gkeys[i] : SCX_EMPTY_KEY;
      masks[s] = __ballot_sync(0xffffffffu, k[s] != SCX_EMPTY_KEY);
      mine += __popc(masks[s]);             // warp total, identical in every lane
    }
    if (lane == 0) wsum[w] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (int j = 0; j < 8; ++j) { const uint32_t c = wsum[j]; wsum[j] = t; t += c; }
      cbase = t ? atomicAdd(count, (unsigned long long)t) : 0ull;
    }
    __syncthreads();
    int64_t o = (int64_t)cbase + wsum[w];
#pragma unroll
    for (int s = 0; s < kCompactPer; ++s) {
      const int64_t i = base + s * 256 + threadIdx.x;
      if (k[s] != SCX_EMPTY_KEY) {
        const int64_t d = o + __popc(masks[s] & ((1u << lane) - 1u));
        out_keys[d] = k[s];
        for (int j = 0; j < m; ++j) out_acc[j * cap + d] = acc[i * m + j];
      }
      o += __popc(masks[s]);
    }
    __syncthreads();                        // wsum / cbase reuse
  }
}

// 128-bit {lo, hi} -> int64 with an overflow flag (hash-group wide sums)
__global__ void i128_narrow_kernel(const int64_t* lo, const int64_t* hi, int64_t n, int64_t* out,
                                   uint32_t* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = lo[i];
    if (hi[i] != (lo[i] >> 63)) atomicOr(flag, 1u);
  }
}

__global__ void unpack_key_kernel(const uint64_t* packed, int64_t n, int shift, uint64_t mask,
                                  int64_t lo, scx_column out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = (int64_t)((packed[i] >> shift) & mask) + lo;
    store_i64(reinterpret_cast<void*>(out.ptr), out.dtype, i, v);
  }
}

__device__ __forceinline__ double pow10d(int s) {
  double p = 1.0;
  for (int i = 0; i < s; ++i) p *= 10.0;
  return p;
}

// exact integer -> correctly rounded double, then one correctly rounded
// division by 10^scale (the numpy reference computes the same quotient
// in float64 up to summation-order rounding).
__global__ void fixed_to_f64_kernel(const int64_t* in, int64_t stride, int64_t n, int scale,
                                    const int64_t* cnt, int64_t cstride, double* out) {
  const double p = pow10d(scale);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = (double)in[i * stride];
    v = scale ? v / p : v;
    if (cnt) {
      int64_t c = cnt[i * cstride];
      v = v / (double)(c > 1 ? c : 1);
    }
    out[i] = v;
  }
}

__global__ void gather_kernel(scx_column in, const uint32_t* idx, int64_t n, scx_column out) {
  const int w = dtype_size_d(in.dtype);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx[i];
    const char* s = reinterpret_cast<const char*>(in.ptr);
    char* d = reinterpret_cast<char*>(out.ptr);
    switch (w) {
      case 1: d[i] = s[j]; break;
      case 2: reinterpret_cast<int16_t*>(d)[i] = reinterpret_cast<const int16_t*>(s)[j]; break;
      case 4: reinterpret_cast<int32_t*>(d)[i] = reinterpret_cast<const int32_t*>(s)[j]; break;
      default: reinterpret_cast<int64_t*>(d)[i] = reinterpret_cast<const int64_t*>(s)[j]; break;
    }
  }
}

__global__ void fill_i64_kernel(int64_t* p, int64_t n, int64_t stride, int64_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i * stride] = v;
}

struct RowPattern {
  int64_t v[16];
};

// p[r * w + j] = pattern[j]: one coalesced pass over a row-major table
__global__ void fill_rows_kernel(int64_t* p, int64_t words, int w, RowPattern pat) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < words;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = pat.v[i % w];
}

__global__ void iota_kernel(uint32_t* idx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    idx[i] = (uint32_t)i;
}

// order-preserving key of one sort column (table.py:198-214).  F64 columns
// map IEEE bits to a monotone u64; integers are offset by `lo`.
__global__ void encode_sort_key_kernel(scx_column col, const uint32_t* idx, int64_t n,
                                       int64_t lo, int n_bits, int desc, int shift,
                                       const int32_t* lut, uint64_t* key, int accumulate) {
  const uint64_t mask = n_bits >= 64 ? ~0ull : ((1ull << n_bits) - 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = idx ? (int64_t)idx[i] : i;
    uint64_t u;
    if (col.dtype == SCX_F64) {   // n_bits == 64 enforced by the host entry
      const uint64_t b = reinterpret_cast<const uint64_t*>(col.ptr)[j];
      u = (b >> 63) ? ~b : (b | (1ull << 63));
    } else {
      int64_t v = load_i64(reinterpret_cast<const void*>(col.ptr), col.dtype, j) - lo;
      if (lut) v = lut[v];
      u = (uint64_t)v;
    }
    u &= mask;
    if (desc) u = mask - u;
    u <<= shift;
    key[i] = accumulate ? (key[i] | u) : u;
  }
}

__global__ void minmax_kernel(scx_column col, int64_t n, int64_t* out) {
  int64_t mn = INT64_MAX, mx = INT64_MIN;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = load_i64(reinterpret_cast<const void*>(col.ptr), col.dtype, i);
    mn = min(mn, v);
    mx = max(mx, v);
  }
  mn = warp_min_i64(mn);
  mx = warp_max_i64(mx);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(reinterpret_cast<long long*>(out), (long long)mn);
    atomicMax(reinterpret_cast<long long*>(out + 1), (long long)mx);
  }
}


// ---- small result reads without a copy engine ------------------------------
// The kernel stores straight into mapped pinned host memory over PCIe: a
// query's few result bytes reach the host while the copy engines are busy
// with a multi-GB upload (a D2H cudaMemcpyAsync queued behind it).
__global__ void write_mapped_kernel(const uint8_t* src, uint8_t* dst, int64_t n) {
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t st = (int64_t)gridDim.x * blockDim.x;
  if ((((uintptr_t)src | (uintptr_t)dst | (uintptr_t)n) & 15) == 0) {
    for (int64_t i = i0; i < n / 16; i += st)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  } else {
    for (int64_t i = i0; i < n; i += st) dst[i] = src[i];
  }
}

}  // namespace scx

extern "C" int scx_write_mapped(const void* src_dev, void* dst_host, int64_t nbytes,
                                void* stream) {
  using namespace scx;
  if (nbytes < 0 || (nbytes && (!src_dev || !dst_host))) {
    set_error("write_mapped: bad arguments");
    return SCX_EINVAL;
  }
  if (nbytes == 0) return SCX_OK;
  void* dptr = nullptr;
  SCX_CUDA(cudaHostGetDevicePointer(&dptr, dst_host, 0));
  const int64_t work = (nbytes + 15) / 16;
  const int grid = (int)(work < 256 * 64 ? (work + 255) / 256 : 64);
  write_mapped_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const uint8_t*>(src_dev), reinterpret_cast<uint8_t*>(dptr), nbytes);
  SCX_CHECK_LAUNCH("write_mapped_kernel");
  return SCX_OK;
}

using namespace scx;

extern "C" int scx_minmax(scx_column col, int64_t n, int64_t* out, void* stream) {
  if (n == 0) return SCX_OK;
  if (!col.ptr || !out || col.dtype == SCX_F64) { set_error("minmax: bad arguments"); return SCX_EINVAL; }
  minmax_kernel<<<grid_for(n, 256, 148 * 8), 256, 0, (cudaStream_t)stream>>>(col, n, out);
  SCX_CHECK_LAUNCH("minmax_kernel");
  return SCX_OK;
}

static int launch_grid(int64_t n) { return grid_for(n, 256, 148 * 16); }

extern "C" int scx_lookup_clear(const scx_lookup* T, void* stream) {
  if (!T || (T->kind != SCX_HT_HASH && !T->vals) ||
      (T->kind == SCX_HT_HASH && (!T->keys || (T->cap & (T->cap - 1))))) {
    set_error("lookup_clear: bad table (hash capacity must be a power of two)");
    return SCX_EINVAL;
  }
  if (T->kind == SCX_HT_BITMAP) {
    SCX_CUDA(cudaMemsetAsync(reinterpret_cast<void*>(T->vals), 0, 4 * ((T->cap + 31) / 32),
                             (cudaStream_t)stream));
    return SCX_OK;
  }
  lookup_clear_kernel<<<launch_grid(T->cap), 256, 0, (cudaStream_t)stream>>>(
      T->kind == SCX_HT_HASH ? reinterpret_cast<uint64_t*>(T->keys) : nullptr,
      reinterpret_cast<uint32_t*>(T->vals), T->cap);
  SCX_CHECK_LAUNCH("lookup_clear_kernel");
  return SCX_OK;
}

extern "C" int scx_lookup_build(const scx_lookup* T, const scx_column* cols, int n_cols,
                                const scx_keyspec* K, int64_t n, uint32_t* flags,
                                void* stream) {
  if (!T || !cols || !K || !flags || n_cols < 1 || n_cols > SCX_MAX_KEYS || K->n < 1 ||
      K->n > SCX_MAX_KEYS) {
    set_error("lookup_build: bad arguments");
    return SCX_EINVAL;
  }
  if (n > 0xFFFFFFFEll) { set_error("lookup_build: >2^32-2 build rows"); return SCX_EUNSUPPORTED; }
  BuildCols C;
  memset(&C, 0, sizeof(C));
  for (int i = 0; i < n_cols; ++i) C.c[i] = cols[i];
  for (int i = 0; i < K->n; ++i)
    if (K->slot[i] < 0 || K->slot[i] >= n_cols) { set_error("lookup_build: key slot"); return SCX_EINVAL; }
  if (n == 0) return SCX_OK;
  lookup_build_kernel<<<launch_grid(n), 256, 0, (cudaStream_t)stream>>>(*T, C, *K, n, flags);
  SCX_CHECK_LAUNCH("lookup_build_kernel");
  return SCX_OK;
}

extern "C" int scx_dense_reduce(const int64_t* acc, int n_ranks, int cells, int m,
                                const int* ops_host, int64_t* out, void* stream) {
  if (!acc || !out || !ops_host || n_ranks < 1 || cells < 1 || m < 1 || m > SCX_MAX_MEASURES) {
    set_error("dense_reduce: bad arguments");
    return SCX_EINVAL;
  }
  ReduceOps ops;
  for (int j = 0; j < m; ++j) {
    if (ops_host[j] < 0 || ops_host[j] > 2) {
      set_error("dense_reduce: measure %d has op %d (0 sum, 1 min, 2 max)", j, ops_host[j]);
      return SCX_EINVAL;
    }
    ops.op[j] = (int8_t)ops_host[j];
  }
  const int64_t words = 2ll * cells * m;
  dense_reduce_kernel<<<(int)((words / 2 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      acc, n_ranks, words, m, ops, out);
  SCX_CHECK_LAUNCH("dense_reduce_kernel");
  return SCX_OK;
}

extern "C" int scx_hash_agg_compact(const uint64_t* gkeys, const int64_t* acc, int64_t cap, int m,
                                    uint64_t* out_keys, int64_t* out_acc, uint64_t* count,
                                    void* stream) {
  if (!gkeys || !out_keys || !count || (m > 0 && (!acc || !out_acc))) {
    set_error("hash_agg_compact: bad arguments");
    return SCX_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  SCX_CUDA(cudaMemsetAsync(count, 0, 8, st));
  if (cap == 0) return SCX_OK;
  hash_agg_compact_kernel<<<launch_grid((cap + kCompactPer - 1) / kCompactPer), 256, 0, st>>>(
      gkeys, acc, cap, m, out_keys, out_acc, reinterpret_cast<unsigned long long*>(count));
  SCX_CHECK_LAUNCH("hash_agg_compact_kernel");
  return SCX_OK;
}

extern "C" int scx_unpack_key(const uint64_t* packed, int64_t n, int shift, uint64_t mask,
                              int64_t lo, scx_column out, void* stream) {
  if (n == 0) return SCX_OK;
  if (!packed || !out.ptr || shift < 0 || shift > 63) { set_error("unpack_key: bad arguments"); return SCX_EINVAL; }
  unpack_key_kernel<<<launch_grid(n), 256, 0, (cudaStream_t)stream>>>(packed, n, shift, mask, lo, out);
  SCX_CHECK_LAUNCH("unpack_key_kernel");
  return SCX_OK;
}

extern "C" int scx_i128_narrow(const int64_t* lo, const int64_t* hi, int64_t n, int64_t* out,
                               uint32_t* flag, void* stream) {
  if (n == 0) return SCX_OK;
  if (!lo || !hi || !out || !flag) { set_error("i128_narrow: null pointer"); return SCX_EINVAL; }
  i128_narrow_kernel<<<launch_grid(n), 256, 0, (cudaStream_t)stream>>>(lo, hi, n, out, flag);
  SCX_CHECK_LAUNCH("i128_narrow_kernel");
  return SCX_OK;
}

extern "C" int scx_fixed_to_f64(const int64_t* in, int64_t stride, int64_t n, int scale,
                                const int64_t* cnt, int64_t cstride, double* out, void* stream) {
  if (n == 0) return SCX_OK;
  if (!in || !out || scale < 0 || scale > 18) { set_error("fixed_to_f64: bad arguments"); return SCX_EINVAL; }
  fixed_to_f64_kernel<<<launch_grid(n), 256, 0, (cudaStream_t)stream>>>(in, stride, n, scale, cnt,
                                                                       cstride, out);
  SCX_CHECK_LAUNCH("fixed_to_f64_kernel");
  return SCX_OK;
}

extern "C" int scx_gather(scx_column in, const uint32_t* idx, int64_t n, scx_column out,
                          void* stream) {
  if (n == 0) return SCX_OK;
  if (!in.ptr || !out.ptr || !idx || dtype_size(in.dtype) != dtype_size(out.dtype)) {
    set_error("gather: bad arguments");
    return SCX_EINVAL;
  }
  gather_kernel<<<launch_grid(n), 256, 0, (cudaStream_t)stream>>>(in, idx, n, out);
  SCX_CHECK_LAUNCH("gather_kernel");
  return SCX_OK;
}

extern "C" int scx_fill_i64(int64_t* p, int64_t n, int64_t stride, int64_t value, void* stream) {
  if (n == 0) return SCX_OK;
  if (!p || stride < 1) { set_error("fill_i64: bad arguments"); return SCX_EINVAL; }
  fill_i64_kernel<<<launch_grid(n), 256, 0, (cudaStream_t)stream>>>(p, n, stride, value);
  SCX_CHECK_LAUNCH("fill_i64_kernel");
  return SCX_OK;
}

extern "C" int scx_fill_rows(int64_t* p, int64_t rows, int w, const int64_t* pattern_host,
                             void* stream) {
  if (rows == 0) return SCX_OK;
  if (!p || !pattern_host || w < 1 || w > 16) { set_error("fill_rows: bad arguments"); return SCX_EINVAL; }
  RowPattern pat;
  for (int j = 0; j < w; ++j) pat.v[j] = pattern_host[j];
  fill_rows_kernel<<<launch_grid(rows * w), 256, 0, (cudaStream_t)stream>>>(p, rows * w, w, pat);
  SCX_CHECK_LAUNCH("fill_rows_kernel");
  return SCX_OK;
}

extern "C" int scx_iota(uint32_t* idx, int64_t n, void* stream) {
  if (n == 0) return SCX_OK;
  if (!idx) { set_error("iota: null"); return SCX_EINVAL; }
  iota_kernel<<<launch_grid(n), 256, 0, (cudaStream_t)stream>>>(idx, n);
  SCX_CHECK_LAUNCH("iota_kernel");
  return SCX_OK;
}

extern "C" int scx_encode_sort_key(scx_column col, const uint32_t* idx, int64_t n, int64_t lo,
                                   int n_bits, int descending, int shift, const int32_t* lut,
                                   uint64_t* key, int accumulate, void* stream) {
  if (n == 0) return SCX_OK;
  if (!col.ptr || !key || n_bits < 1 || n_bits > 64 || shift < 0 || shift + n_bits > 64 ||
      (col.dtype == SCX_F64 && n_bits != 64)) {
    set_error("encode_sort_key: bad arguments (bits=%d shift=%d)", n_bits, shift);
    return SCX_EINVAL;
  }
  encode_sort_key_kernel<<<launch_grid(n), 256, 0, (cudaStream_t)stream>>>(
      col, idx, n, lo, n_bits, descending, shift, lut, key, accumulate);
  SCX_CHECK_LAUNCH("encode_sort_key_kernel");
  return SCX_OK;
}

// ---- coarse membership bitmap (shared-memory prefilter of bitmap probes) ---
// coarse bit j = OR of fine bits [j << shift, (j + 1) << shift): a probe whose
// coarse bit is clear is a non-member without touching the fine bitmap, so a
// selective semi join (Q17: 0.1% of parts) is answered from shared memory for
// most rows instead of one random L2 access per row.
namespace scx {
__global__ void bitmap_coarsen_kernel(const uint32_t* fine, int64_t nbits, int shift,
                                      uint32_t* coarse, int64_t cbits) {
  const int lane = threadIdx.x & 31;
  for (int64_t j0 = (int64_t)blockIdx.x * blockDim.x; j0 < cbits; j0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = j0 + threadIdx.x;
    bool any = false;
    if (j < cbits) {
      const int64_t b0 = j << shift, b1 = min((j + 1) << shift, nbits);
      if (shift >= 5) {
        for (int64_t w = b0 >> 5; w < (b1 + 31) >> 5; ++w) any |= fine[w] != 0u;
      } else {
        const uint32_t word = fine[b0 >> 5];
        const uint32_t m = (shift == 0 ? 1u : ((1u << (1 << shift)) - 1u)) << (b0 & 31);
        any = (word & m) != 0u;
      }
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, any);
    if (lane == 0 && j < cbits) coarse[j >> 5] = bal;
  }
}
}  // namespace scx

extern "C" int scx_bitmap_coarsen(const uint32_t* fine, int64_t nbits, int shift,
                                  uint32_t* coarse, void* stream) {
  if (!fine || !coarse || nbits < 0 || shift < 0 || shift > 40) {
    set_error("bitmap_coarsen: bad arguments");
    return SCX_EINVAL;
  }
  const int64_t cbits = nbits > 0 ? ((nbits - 1) >> shift) + 1 : 0;
  if (cbits == 0) return SCX_OK;
  const int64_t padded = (cbits + 31) & ~int64_t(31);     // whole warps -> whole words
  scx::bitmap_coarsen_kernel<<<(int)std::min<int64_t>((padded + 255) / 256, 2368), 256, 0,
                               (cudaStream_t)stream>>>(fine, nbits, shift, coarse, padded);
  SCX_CHECK_LAUNCH("bitmap_coarsen_kernel");
  return SCX_OK;
}


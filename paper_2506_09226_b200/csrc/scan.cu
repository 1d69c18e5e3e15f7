// scan.cu -- multi-CTA exclusive scan and the ordered compaction of
// direct-addressed group tables.
//
// * scan_u32_excl: reduce -> scan of tile sums -> rescan (3 launches, all
//   CTAs busy); replaces the single-CTA scan of the radix passes, which was
//   the top kernel of the sort-heavy queries (profiles/r1_kprof_*).
// * scx_direct_agg_compact: occupied slots of a direct-addressed group table
//   (slot = packed key) in slot order -- i.e. already sorted by group key --
//   so group_aggregate (relops.py:97-160, output sorted by keys) skips the
//   radix sort entirely for dense-key groupings (orderkey, custkey, ...).
#include "common.cuh"

namespace scx {

constexpr int kScanItems = 16;
constexpr int kScanTile = kBlock * kScanItems;   // 4096 elements per CTA

// block-wide exclusive scan of one u32 per thread; returns the block total
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t& excl) {
  __shared__ uint32_t warp_tot[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += y;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  uint32_t wofs = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const uint32_t t = warp_tot[w];
    wofs += (w < warp) ? t : 0;
    tot += t;
  }
  __syncthreads();
  excl = wofs + inc - v;
  return tot;
}

__global__ void tile_sum_kernel(const uint32_t* in, int64_t m, uint64_t* part) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) s += (base + i < m) ? in[base + i] : 0u;
  uint32_t excl;
  const uint32_t tot = block_excl_scan(s, excl);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

// exclusive scan of nb u64 tile sums in one CTA (nb <= 1024 * 64)
__global__ void small_scan_kernel(uint64_t* part, int64_t nb) {
  __shared__ uint64_t s[1024];
  const int t = threadIdx.x;
  const int64_t per = (nb + 1023) / 1024;
  const int64_t b = t * per, e = min(nb, b + per);
  uint64_t sum = 0;
  for (int64_t i = b; i < e; ++i) sum += part[i];
  s[t] = sum;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const uint64_t v = (t >= o) ? s[t - o] : 0;
    __syncthreads();
    s[t] += v;
    __syncthreads();
  }
  uint64_t run = s[t] - sum;
  for (int64_t i = b; i < e; ++i) {
    const uint64_t x = part[i];
    part[i] = run;
    run += x;
  }
  if (t == 1023) part[nb] = s[1023];
}

__global__ void tile_scan_kernel(const uint32_t* in, int64_t m, const uint64_t* part,
                                 uint64_t* out) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t v[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < m) ? in[base + i] : 0u;
    s += v[i];
  }
  uint32_t excl;
  block_excl_scan(s, excl);
  uint64_t run = part[blockIdx.x] + excl;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < m) out[base + i] = run;
    run += v[i];
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == kBlock - 1) out[m] = part[gridDim.x];
}

int64_t scan_tmp_words(int64_t m) { return (m + kScanTile - 1) / kScanTile + 2; }

// out[i] = sum in[0..i), out[m] = total; tmp: scan_tmp_words(m) u64
int scan_u32_excl(const uint32_t* in, uint64_t* out, int64_t m, uint64_t* tmp, cudaStream_t st) {
  const int64_t nb = (m + kScanTile - 1) / kScanTile;
  if (nb > 1024 * 64) { set_error("scan: %lld elements exceed the scan capacity", (long long)m); return SCX_EUNSUPPORTED; }
  if (m == 0) {
    SCX_CUDA(cudaMemsetAsync(out, 0, 8, st));
    return SCX_OK;
  }
  tile_sum_kernel<<<(int)nb, kBlock, 0, st>>>(in, m, tmp);
  SCX_CHECK_LAUNCH("tile_sum_kernel");
  small_scan_kernel<<<1, 1024, 0, st>>>(tmp, nb);
  SCX_CHECK_LAUNCH("small_scan_kernel");
  tile_scan_kernel<<<(int)nb, kBlock, 0, st>>>(in, m, tmp, out);
  SCX_CHECK_LAUNCH("tile_scan_kernel");
  return SCX_OK;
}

// ---- ordered compaction of a direct-addressed group table -----------------
// A CTA owns 4096 consecutive slots, visited as 16 rounds of 256 (thread t
// reads slot round*256 + t: coalesced).  Each round's ranks come from warp
// ballots; the round's accumulator rows (256 x W words, row-major) are staged
// through shared memory so both the read and the measure-major write are
// coalesced.
// occupancy of slot e: gkeys[e] != EMPTY, or (gkeys == nullptr) the group's
// count word acc[e*m + occ_word] > 0 -- direct tables keyed by the slot need
// no key array at all (the packed key IS the slot)
struct Occ {
  const uint64_t* gkeys;
  const int64_t* acc;
  int m, occ_word;
  int hv_word;               // HAVING on a measure word: keep iff hv_lo <= acc <= hv_hi (-1: none)
  int64_t hv_lo, hv_hi;
  __device__ __forceinline__ bool keep(const int64_t* row) const {
    return row[occ_word] > 0 && (hv_word < 0 || (row[hv_word] >= hv_lo && row[hv_word] <= hv_hi));
  }
  __device__ __forceinline__ bool operator()(int64_t e) const {
    return gkeys ? gkeys[e] != SCX_EMPTY_KEY : keep(acc + e * m);
  }
  __device__ __forceinline__ uint64_t key(int64_t e) const { return gkeys ? gkeys[e] : (uint64_t)e; }
};

__global__ void occ_count_kernel(Occ O, int64_t cap, uint64_t* part) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  uint32_t s = 0;
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) {
    const int64_t e = base + it * kBlock + threadIdx.x;
    s += (e < cap && O(e));
  }
  uint32_t excl;
  const uint32_t tot = block_excl_scan(s, excl);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kBlock) occ_write_kernel(
    Occ O, const int64_t* acc, int64_t cap, int m, const uint64_t* part,
    uint64_t* out_keys, int64_t* out_acc, uint64_t* count) {
  __shared__ int64_t tile[kBlock * 16];
  __shared__ uint32_t wcnt[kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * kScanTile;
  uint64_t pos0 = part[blockIdx.x];
  for (int it = 0; it < kScanItems; ++it) {
    const int64_t r0 = base + (int64_t)it * kBlock;
    if (r0 >= cap) break;
    const int64_t e = r0 + tid;
    const int64_t rows = min((int64_t)kBlock, cap - r0);
    for (int64_t x = tid; x < rows * m; x += kBlock) tile[x] = acc[r0 * m + x];
    __syncthreads();
    const bool occ = e < cap && (O.gkeys ? O.gkeys[e] != SCX_EMPTY_KEY : O.keep(tile + tid * m));
    const uint32_t b = __ballot_sync(0xffffffffu, occ);
    if (lane == 0) wcnt[warp] = __popc(b);
    __syncthreads();
    uint32_t wofs = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      wofs += (w < warp) ? wcnt[w] : 0;
      tot += wcnt[w];
    }
    if (occ) {
      const uint64_t pos = pos0 + wofs + __popc(b & ((1u << lane) - 1u));
      out_keys[pos] = O.key(e);
      for (int j = 0; j < m; ++j) out_acc[(int64_t)j * cap + (int64_t)pos] = tile[tid * m + j];
    }
    pos0 += tot;
    __syncthreads();
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *count = part[gridDim.x];
}

// ---- finishing a staged stable compaction (jit COMPACT sink) ---------------
// One launch moves every output column (blockIdx.z = column): CTA b's staged
// rows [0, cnt_b) of column j go to rows [prefix_b, prefix_b + cnt_b).
constexpr int kRegionCols = 16;
struct RegionCols {
  const char* src[kRegionCols];
  char* dst[kRegionCols];
  int w[kRegionCols];
};

// 16 bytes of src starting at byte offset m (0..15) of the aligned pair {a, b}
__device__ __forceinline__ uint4 byte_window(const uint4 a, const uint4 b, int m) {
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  const int q = m >> 2, sh = (m & 3) * 8;
  uint32_t o[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) {     // o[k] = w[q + k], q in 0..3, without local memory
    uint32_t v = w[k];
    v = q == 1 ? w[k + 1 < 8 ? k + 1 : 7] : v;
    v = q == 2 ? w[k + 2 < 8 ? k + 2 : 7] : v;
    v = q == 3 ? w[k + 3 < 8 ? k + 3 : 7] : v;
    o[k] = v;
  }
  return make_uint4(__funnelshift_r(o[0], o[1], sh), __funnelshift_r(o[1], o[2], sh),
                    __funnelshift_r(o[2], o[3], sh), __funnelshift_r(o[3], o[4], sh));
}

// A region is a byte range: [s, s + cnt * w) -> [d, d + cnt * w).  The staged
// source is 16-byte aligned (region_rows * w and every column's stage are
// multiples of 16), the destination starts at any byte, so each thread writes
// one aligned 16-byte destination chunk from a byte window of two aligned
// source vectors; the first and last chunks (shared with the neighbouring
// regions) are written byte by byte.
__global__ void region_copy_kernel(RegionCols R, const uint64_t* prefix, int64_t region_rows) {
  const int j = blockIdx.z, w = R.w[j];
  const int64_t b = blockIdx.y;
  const uint64_t start = prefix[b], nb = (prefix[b + 1] - start) * (uint64_t)w;
  if (nb == 0) return;
  const uint8_t* s = reinterpret_cast<const uint8_t*>(R.src[j]) + (size_t)b * region_rows * w;
  uint8_t* d = reinterpret_cast<uint8_t*>(R.dst[j]) + (size_t)start * w;
  const uintptr_t da = reinterpret_cast<uintptr_t>(d), d0 = da & ~uintptr_t(15);
  const uint64_t nchunks = (da + nb - d0 + 15) / 16;
  const int m = (int)((16 - (da & 15)) & 15);      // source offset of each chunk, mod 16
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < nchunks;
       c += (uint64_t)gridDim.x * blockDim.x) {
    const uintptr_t x0 = d0 + c * 16;
    if (x0 >= da && x0 + 16 <= da + nb) {
      const uint64_t so = x0 - da;                   // so % 16 == m
      const uint4* sp = reinterpret_cast<const uint4*>(s + (so - m));
      const uint4 lo = sp[0];
      const uint4 hi = m ? sp[1] : lo;
      *reinterpret_cast<uint4*>(x0) = byte_window(lo, hi, m);
    } else {
      for (int i = 0; i < 16; ++i) {
        const uintptr_t x = x0 + i;
        if (x >= da && x < da + nb) *reinterpret_cast<uint8_t*>(x) = s[x - da];
      }
    }
  }
}

// status[0..grid) = per-CTA selected counts -> exclusive prefix (+ total at
// status[grid]); each CTA's staged rows move to their final position
int compact_finish(uint64_t* status, int64_t grid, char* stage, int64_t stage_rows,
                   const scx_column* outs, int n_out, int64_t region_rows, uint64_t* count,
                   cudaStream_t st) {
  small_scan_kernel<<<1, 1024, 0, st>>>(status, grid);
  SCX_CHECK_LAUNCH("small_scan_kernel");
  SCX_CUDA(cudaMemcpyAsync(count, status + grid, 8, cudaMemcpyDeviceToDevice, st));
  char* src = stage;
  for (int j0 = 0; j0 < n_out; j0 += kRegionCols) {
    RegionCols R{};
    const int m = n_out - j0 < kRegionCols ? n_out - j0 : kRegionCols;
    for (int j = 0; j < m; ++j) {
      const int w = dtype_size(outs[j0 + j].dtype);
      R.src[j] = src;
      R.dst[j] = reinterpret_cast<char*>(outs[j0 + j].ptr);
      R.w[j] = w;
      src += (stage_rows * w + 15) & ~int64_t(15);
    }
    region_copy_kernel<<<dim3(8, (unsigned)grid, (unsigned)m), 256, 0, st>>>(R, status,
                                                                            region_rows);
    SCX_CHECK_LAUNCH("region_copy_kernel");
  }
  return SCX_OK;
}

// ---- dense ranks of a sorted (non-decreasing) key column --------------------
// head(i) = i == 0 || key[i] != key[i-1]; rank(i) = #heads in [0, i] - 1.
// A group-by on a clustered key (lineitem / a materialised lineitem subset by
// l_orderkey) then addresses a table of exactly #distinct-keys slots,
// sequentially, instead of hashing into a table sized by the row count.
__device__ __forceinline__ uint32_t is_head(const scx_column& c, int64_t i) {
  const void* p = reinterpret_cast<const void*>(c.ptr);
  return i == 0 || load_i64(p, c.dtype, i) != load_i64(p, c.dtype, i - 1);
}

__global__ void rank_count_kernel(scx_column c, int64_t n, uint64_t* part, uint64_t* unsorted) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  const void* p = reinterpret_cast<const void*>(c.ptr);
  uint32_t s = 0, bad = 0;
  int64_t prev = base > 0 && base < n ? load_i64(p, c.dtype, base - 1) : 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) {
      const int64_t k = load_i64(p, c.dtype, base + i);
      s += (base + i == 0 || k != prev);
      bad += (base + i > 0 && k < prev);
      prev = k;
    }
  }
  uint32_t excl;
  const uint32_t tot = block_excl_scan(s, excl);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
  if (bad) atomicAdd(reinterpret_cast<unsigned long long*>(unsorted), (unsigned long long)bad);
}

__global__ void rank_write_kernel(scx_column c, int64_t n, int64_t lo, const uint64_t* part,
                                  uint32_t* rank, uint64_t* keys_by_rank, uint64_t* count) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  const void* p = reinterpret_cast<const void*>(c.ptr);
  uint32_t h[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    h[i] = (base + i < n) ? is_head(c, base + i) : 0u;
    s += h[i];
  }
  uint32_t excl;
  block_excl_scan(s, excl);
  uint64_t run = part[blockIdx.x] + excl;   // heads before this thread's rows
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i >= n) break;
    run += h[i];
    rank[base + i] = (uint32_t)(run - 1);
    if (h[i]) keys_by_rank[run - 1] = (uint64_t)(load_i64(p, c.dtype, base + i) - lo);
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == kBlock - 1) *count = part[gridDim.x];
}

// ---- stream aggregation over a sorted key ---------------------------------------
// Rows of one key are contiguous; the thread holding a group's FIRST row
// aggregates the whole group (reading past its own rows when the group runs
// on), so every group is produced exactly once with no table, no atomics on
// accumulators and no merge pass.  HAVING is applied before the write; the
// output is compacted with one warp-aggregated atomic (unordered).
struct SortedAggArgs {
  scx_column key;
  scx_column val[SCX_MAX_MEASURES];
  int op[SCX_MAX_MEASURES];          // SCX_AGG_SUM / COUNT / MIN / MAX
  int m;
  int hv;                            // measure index of the HAVING range, -1 = none
  int64_t hv_lo, hv_hi;
};

constexpr int kSortedChunk = 4096;      // rows per warp
constexpr int kSortedUnroll = 4;        // 32-row windows loaded ahead

__device__ __forceinline__ int64_t agg_op(int op, int64_t a, int64_t b) {
  return op == SCX_AGG_MIN ? (b < a ? b : a) : op == SCX_AGG_MAX ? (b > a ? b : a) : a + b;
}
__device__ __forceinline__ int64_t agg_ident(int op) {
  return op == SCX_AGG_MIN ? INT64_MAX : op == SCX_AGG_MAX ? INT64_MIN : 0;
}

// Each warp owns kSortedChunk consecutive rows and walks them 32 at a time
// (coalesced loads): head flags from the neighbouring lane's key, a segmented
// inclusive warp scan per measure, and the lane that ends a segment emits the
// group.  A group still open at lane 31 is carried into the next window; rows
// of the group that began before the chunk belong to the previous warp; the
// group open at the chunk end is followed past it until its key changes.
template <int M>
__device__ __forceinline__ bool having_ok(const SortedAggArgs& A, const int64_t (&x)[M]) {
  if (A.hv < 0) return true;
  int64_t h = 0;
#pragma unroll
  for (int j = 0; j < M; ++j)
    if (j == A.hv) h = x[j];
  return h >= A.hv_lo && h <= A.hv_hi;
}

template <int M>
__global__ void __launch_bounds__(256) sorted_agg_kernel(SortedAggArgs A, int64_t n, int64_t* out_keys,
                                                         int64_t* out_acc, int64_t cap,
                                                         unsigned long long* count, uint32_t* overflow) {
  const void* kp = reinterpret_cast<const void*>(A.key.ptr);
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t start = warp * kSortedChunk;
  if (start >= n) return;
  const int64_t cend = start + kSortedChunk < n ? start + kSortedChunk : n;
  const bool skip_first = start > 0;
  const int64_t kfirst_prev = skip_first ? load_i64(kp, A.key.dtype, start - 1) : 0;
  const int64_t kend = load_i64(kp, A.key.dtype, cend - 1);   // key open at the chunk end
  bool carry = false;
  int64_t ckey = 0, cacc[M];
  int64_t prev_last = kfirst_prev;                            // key of row s-1
  const uint32_t lt = (1u << lane) - 1u;
  bool done = false;
  for (int64_t s0 = start; s0 < n && !done; s0 += 32 * kSortedUnroll) {
    // loads of kSortedUnroll windows in flight before any is processed
    int64_t kk[kSortedUnroll], vv[kSortedUnroll][M];
#pragma unroll
    for (int u = 0; u < kSortedUnroll; ++u) {
      const int64_t i = s0 + 32 * u + lane;
      kk[u] = i < n ? load_i64(kp, A.key.dtype, i) : 0;
#pragma unroll
      for (int j = 0; j < M; ++j)
        vv[u][j] = (i < n && A.op[j] != SCX_AGG_COUNT)
                       ? load_i64(reinterpret_cast<const void*>(A.val[j].ptr), A.val[j].dtype, i) : 1;
    }
#pragma unroll
  for (int u = 0; u < kSortedUnroll; ++u) {
    const int64_t s = s0 + 32 * u;
    if (done || s >= n) { done = true; break; }
    const int64_t k = kk[u];
    if (s >= cend) {
      // past the chunk: only rows continuing the open group remain
      if (!carry || __shfl_sync(0xffffffffu, k, 0) != ckey) { done = true; break; }
    }
    const int64_t i = s + lane;
    const bool in = i < n;
    bool act = in && !(skip_first && k == kfirst_prev) && (i < cend || k == kend);
    int64_t up = __shfl_up_sync(0xffffffffu, k, 1);
    if (lane == 0) up = prev_last;
    const bool head_raw = (i == 0) || k != up;
    // a segment starts at an active row whose predecessor is another key, or
    // at the first active row of the window that does not continue the carry
    bool prev_act = __shfl_up_sync(0xffffffffu, act, 1);
    if (lane == 0) prev_act = carry;
    bool head = act && (head_raw || !prev_act);
    // the carry is complete if the window's first row does not continue it
    const bool cont0 = __shfl_sync(0xffffffffu, act && !head, 0);
    if (carry && !cont0) {
      if (lane == 0) {
        const bool ok = having_ok<M>(A, cacc);
        if (ok) {
          const unsigned long long o = atomicAdd(count, 1ull);
          if ((int64_t)o < cap) {
            out_keys[o] = ckey;
            _Pragma("unroll") for (int j = 0; j < M; ++j) out_acc[(int64_t)j * cap + (int64_t)o] = cacc[j];
          } else {
            atomicOr(overflow, 1u);
          }
        }
      }
      carry = false;
    }
    int64_t v[M];
    _Pragma("unroll") for (int j = 0; j < M; ++j) v[j] = act ? vv[u][j] : agg_ident(A.op[j]);
    // segmented inclusive scan (segments start at `head`)
    bool f = head;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const bool fu = __shfl_up_sync(0xffffffffu, f, d);
      _Pragma("unroll") for (int j = 0; j < M; ++j) {
        const int64_t vu = __shfl_up_sync(0xffffffffu, v[j], d);
        if (lane >= d && !f) v[j] = agg_op(A.op[j], v[j], vu);
      }
      if (lane >= d) f = f || fu;
    }
    // rows of the first segment continue the carry
    if (carry && act && !f)
      _Pragma("unroll") for (int j = 0; j < M; ++j) v[j] = agg_op(A.op[j], v[j], cacc[j]);
    // segment ends: the next lane starts another segment or is inactive
    const bool nact = __shfl_down_sync(0xffffffffu, act, 1);
    const bool nhead = __shfl_down_sync(0xffffffffu, head, 1);
    const bool end_here = act && lane < 31 && (!nact || nhead);
    bool emit = end_here && having_ok<M>(A, v);
    const uint32_t bal = __ballot_sync(0xffffffffu, emit);
    if (bal) {
      unsigned long long base = 0;
      const int leader = __ffs(bal) - 1;
      if (lane == leader) base = atomicAdd(count, (unsigned long long)__popc(bal));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (emit) {
        const int64_t o = (int64_t)base + __popc(bal & lt);
        if (o < cap) {
          out_keys[o] = k;
          _Pragma("unroll") for (int j = 0; j < M; ++j) out_acc[(int64_t)j * cap + o] = v[j];
        } else {
          atomicOr(overflow, 1u);
        }
      }
    }
    // lane 31's segment stays open -> carry (all lanes keep the same state)
    const bool act31 = __shfl_sync(0xffffffffu, act, 31);
    carry = act31;
    if (act31) {
      ckey = __shfl_sync(0xffffffffu, k, 31);
      _Pragma("unroll") for (int j = 0; j < M; ++j) cacc[j] = __shfl_sync(0xffffffffu, v[j], 31);
    }
    prev_last = __shfl_sync(0xffffffffu, k, 31);
    if (!__shfl_sync(0xffffffffu, in, 31)) { done = true; break; }
  }
  }
  if (carry && lane == 0) {
    const bool ok = having_ok<M>(A, cacc);
    if (ok) {
      const unsigned long long o = atomicAdd(count, 1ull);
      if ((int64_t)o < cap) {
        out_keys[o] = ckey;
        _Pragma("unroll") for (int j = 0; j < M; ++j) out_acc[(int64_t)j * cap + (int64_t)o] = cacc[j];
      } else {
        atomicOr(overflow, 1u);
      }
    }
  }
}

// non-decreasing check of a column: *bad = number of i with key[i] < key[i-1]
__global__ void sorted_check_kernel(scx_column c, int64_t n, unsigned long long* bad) {
  const void* p = reinterpret_cast<const void*>(c.ptr);
  unsigned long long cnt = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    cnt += load_i64(p, c.dtype, i) < load_i64(p, c.dtype, i - 1);
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(bad, cnt);
}

// ---- top-k support: digit histogram of keys in a range, stable select-below --
__global__ void range_hist_kernel(const uint64_t* keys, int64_t n, uint64_t lo, uint64_t hi,
                                  int shift, uint32_t* counts) {
  __shared__ uint32_t h[256];
  for (int d = threadIdx.x; d < 256; d += blockDim.x) h[d] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    if (k >= lo && k < hi) atomicAdd(&h[((k - lo) >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += blockDim.x)
    if (h[d]) atomicAdd(&counts[d], h[d]);
}

__global__ void below_count_kernel(const uint64_t* keys, int64_t n, uint64_t T, uint64_t* part) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) s += (base + i < n && keys[base + i] < T);
  uint32_t excl;
  const uint32_t tot = block_excl_scan(s, excl);
  if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void below_write_kernel(const uint64_t* keys, int64_t n, uint64_t T, const uint64_t* part,
                                   uint64_t* out_keys, uint32_t* out_idx, uint64_t* count) {
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t f[kScanItems];
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    f[i] = base + i < n && keys[base + i] < T;
    s += f[i];
  }
  uint32_t excl;
  block_excl_scan(s, excl);
  uint64_t o = part[blockIdx.x] + excl;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (f[i]) {
      out_keys[o] = keys[base + i];
      out_idx[o] = (uint32_t)(base + i);
      ++o;
    }
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == kBlock - 1) *count = part[gridDim.x];
}

}  // namespace scx

using namespace scx;

extern "C" int scx_range_hist(const uint64_t* keys, int64_t n, uint64_t lo, uint64_t hi, int shift,
                              uint32_t* counts, void* stream) {
  if (!keys || !counts || n < 0 || shift < 0 || shift > 63) {
    set_error("range_hist: bad arguments");
    return SCX_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  SCX_CUDA(cudaMemsetAsync(counts, 0, 256 * sizeof(uint32_t), st));
  if (n == 0) return SCX_OK;
  range_hist_kernel<<<grid_for(n, 256, 1184), 256, 0, st>>>(keys, n, lo, hi, shift, counts);
  SCX_CHECK_LAUNCH("range_hist_kernel");
  return SCX_OK;
}

extern "C" int64_t scx_select_below_workspace(int64_t n) { return 8 * scan_tmp_words(n); }

extern "C" int scx_select_below(const uint64_t* keys, int64_t n, uint64_t T, uint64_t* out_keys,
                                uint32_t* out_idx, uint64_t* count, void* temp, void* stream) {
  if (!keys || !out_keys || !out_idx || !count || (n > 0 && !temp) || n < 0 ||
      n > (int64_t)0xFFFFFFFFll) {
    set_error("select_below: bad arguments");
    return SCX_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0) {
    SCX_CUDA(cudaMemsetAsync(count, 0, 8, st));
    return SCX_OK;
  }
  const int64_t nb = (n + kScanTile - 1) / kScanTile;
  if (nb > 1024 * 64) { set_error("select_below: input too long"); return SCX_EUNSUPPORTED; }
  uint64_t* part = static_cast<uint64_t*>(temp);
  below_count_kernel<<<(int)nb, kBlock, 0, st>>>(keys, n, T, part);
  SCX_CHECK_LAUNCH("below_count_kernel");
  small_scan_kernel<<<1, 1024, 0, st>>>(part, nb);
  SCX_CHECK_LAUNCH("small_scan_kernel");
  below_write_kernel<<<(int)nb, kBlock, 0, st>>>(keys, n, T, part, out_keys, out_idx, count);
  SCX_CHECK_LAUNCH("below_write_kernel");
  return SCX_OK;
}

extern "C" int64_t scx_sorted_rank_workspace(int64_t n) { return 8 * scan_tmp_words(n); }

extern "C" int scx_sorted_rank(const scx_column* key, int64_t n, int64_t lo, uint32_t* rank,
                               uint64_t* keys_by_rank, uint64_t* count, void* temp,
                               void* stream) {
  if (!key || !rank || !keys_by_rank || !count || (n > 0 && !temp) || n < 0 ||
      n > (int64_t)0xFFFFFFFFll) {
    set_error("sorted_rank: bad arguments");
    return SCX_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 0) {
    SCX_CUDA(cudaMemsetAsync(count, 0, 16, st));
    return SCX_OK;
  }
  const int64_t nb = (n + kScanTile - 1) / kScanTile;
  if (nb > 1024 * 64) { set_error("sorted_rank: column too long"); return SCX_EUNSUPPORTED; }
  uint64_t* part = static_cast<uint64_t*>(temp);
  SCX_CUDA(cudaMemsetAsync(count + 1, 0, 8, st));
  rank_count_kernel<<<(int)nb, kBlock, 0, st>>>(*key, n, part, count + 1);
  SCX_CHECK_LAUNCH("rank_count_kernel");
  small_scan_kernel<<<1, 1024, 0, st>>>(part, nb);
  SCX_CHECK_LAUNCH("small_scan_kernel");
  rank_write_kernel<<<(int)nb, kBlock, 0, st>>>(*key, n, lo, part, rank, keys_by_rank, count);
  SCX_CHECK_LAUNCH("rank_write_kernel");
  return SCX_OK;
}

extern "C" int64_t scx_direct_agg_workspace(int64_t cap) { return 8 * scan_tmp_words(cap); }

static int direct_compact(const Occ& O, const int64_t* acc, int64_t cap, int m,
                          uint64_t* out_keys, int64_t* out_acc, uint64_t* count, void* temp,
                          cudaStream_t st) {
  if (cap == 0) {
    SCX_CUDA(cudaMemsetAsync(count, 0, 8, st));
    return SCX_OK;
  }
  const int64_t nb = (cap + kScanTile - 1) / kScanTile;
  if (nb > 1024 * 64) { set_error("direct_agg_compact: table too large"); return SCX_EUNSUPPORTED; }
  uint64_t* part = static_cast<uint64_t*>(temp);
  occ_count_kernel<<<(int)nb, kBlock, 0, st>>>(O, cap, part);
  SCX_CHECK_LAUNCH("occ_count_kernel");
  small_scan_kernel<<<1, 1024, 0, st>>>(part, nb);
  SCX_CHECK_LAUNCH("small_scan_kernel");
  occ_write_kernel<<<(int)nb, kBlock, 0, st>>>(O, acc, cap, m, part, out_keys, out_acc, count);
  SCX_CHECK_LAUNCH("occ_write_kernel");
  return SCX_OK;
}

extern "C" int scx_direct_agg_compact(const uint64_t* gkeys, const int64_t* acc, int64_t cap,
                                      int m, uint64_t* out_keys, int64_t* out_acc,
                                      uint64_t* count, void* temp, void* stream) {
  if (!gkeys || !out_keys || !count || !temp || m > 16 || (m > 0 && (!acc || !out_acc))) {
    set_error("direct_agg_compact: bad arguments");
    return SCX_EINVAL;
  }
  Occ O{gkeys, acc, m, 0, -1, 0, 0};
  return direct_compact(O, acc, cap, m, out_keys, out_acc, count, temp, (cudaStream_t)stream);
}

extern "C" int scx_direct_agg_compact_counted(const int64_t* acc, int64_t cap, int m,
                                              int occ_word, uint64_t* out_keys,
                                              int64_t* out_acc, uint64_t* count, void* temp,
                                              void* stream) {
  if (!acc || !out_keys || !out_acc || !count || !temp || m < 1 || m > 16 || occ_word < 0 ||
      occ_word >= m) {
    set_error("direct_agg_compact_counted: bad arguments");
    return SCX_EINVAL;
  }
  Occ O{nullptr, acc, m, occ_word, -1, 0, 0};
  return direct_compact(O, acc, cap, m, out_keys, out_acc, count, temp, (cudaStream_t)stream);
}

extern "C" int scx_direct_agg_compact_having(const int64_t* acc, int64_t cap, int m,
                                             int occ_word, int hv_word, int64_t hv_lo,
                                             int64_t hv_hi, uint64_t* out_keys,
                                             int64_t* out_acc, uint64_t* count, void* temp,
                                             void* stream) {
  if (!acc || !out_keys || !out_acc || !count || !temp || m < 1 || m > 16 || occ_word < 0 ||
      occ_word >= m || hv_word < 0 || hv_word >= m) {
    set_error("direct_agg_compact_having: bad arguments");
    return SCX_EINVAL;
  }
  Occ O{nullptr, acc, m, occ_word, hv_word, hv_lo, hv_hi};
  return direct_compact(O, acc, cap, m, out_keys, out_acc, count, temp, (cudaStream_t)stream);
}

extern "C" int scx_is_sorted(const scx_column* col, int64_t n, uint64_t* bad, void* stream) {
  if (!col || !bad || n < 0) {
    set_error("is_sorted: bad arguments");
    return SCX_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  SCX_CUDA(cudaMemsetAsync(bad, 0, 8, st));
  if (n < 2) return SCX_OK;
  sorted_check_kernel<<<grid_for(n, 256, 2368), 256, 0, st>>>(*col, n, reinterpret_cast<unsigned long long*>(bad));
  SCX_CHECK_LAUNCH("sorted_check_kernel");
  return SCX_OK;
}

extern "C" int scx_sorted_group_agg(const scx_column* key, const scx_column* vals, const int* ops,
                                    int m, int64_t n, int hv, int64_t hv_lo, int64_t hv_hi,
                                    int64_t* out_keys, int64_t* out_acc, int64_t cap,
                                    uint64_t* count, uint32_t* overflow, void* stream) {
  if (!key || m < 0 || m > SCX_MAX_MEASURES || (m > 0 && (!vals || !ops)) || n < 0 ||
      hv >= m || !out_keys || (m > 0 && !out_acc) || !count || !overflow) {
    set_error("sorted_group_agg: bad arguments");
    return SCX_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  SCX_CUDA(cudaMemsetAsync(count, 0, 8, st));
  SCX_CUDA(cudaMemsetAsync(overflow, 0, 4, st));
  if (n == 0) return SCX_OK;
  SortedAggArgs A;
  memset(&A, 0, sizeof(A));
  A.key = *key;
  A.m = m;
  for (int j = 0; j < m; ++j) {
    A.val[j] = vals[j];
    A.op[j] = ops[j];
    if (ops[j] < SCX_AGG_SUM || ops[j] > SCX_AGG_MAX) {
      set_error("sorted_group_agg: unknown aggregate op %d", ops[j]);
      return SCX_EINVAL;
    }
  }
  A.hv = hv;
  A.hv_lo = hv_lo;
  A.hv_hi = hv_hi;
  const int64_t warps = (n + kSortedChunk - 1) / kSortedChunk;
  const int grid = (int)((warps * 32 + 255) / 256);
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(count);
  switch (m) {   // measures in registers: one instantiation per count
    case 1: sorted_agg_kernel<1><<<grid, 256, 0, st>>>(A, n, out_keys, out_acc, cap, cnt, overflow); break;
    case 2: sorted_agg_kernel<2><<<grid, 256, 0, st>>>(A, n, out_keys, out_acc, cap, cnt, overflow); break;
    case 3: sorted_agg_kernel<3><<<grid, 256, 0, st>>>(A, n, out_keys, out_acc, cap, cnt, overflow); break;
    case 4: sorted_agg_kernel<4><<<grid, 256, 0, st>>>(A, n, out_keys, out_acc, cap, cnt, overflow); break;
    default:
      set_error("sorted_group_agg: supports 1..4 measures (got %d)", m);
      return SCX_EUNSUPPORTED;
  }
  SCX_CHECK_LAUNCH("sorted_agg_kernel");
  return SCX_OK;
}

// u32 group-table words -> int64 (narrow direct tables, before compaction)
__global__ void widen_u32_kernel(const uint32_t* in, int64_t n, int64_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)in[i];
}

extern "C" int scx_widen_u32(const uint32_t* in, int64_t n, int64_t* out, void* stream) {
  if ((n > 0 && (!in || !out)) || n < 0) {
    set_error("widen_u32: bad arguments");
    return SCX_EINVAL;
  }
  if (n == 0) return SCX_OK;
  widen_u32_kernel<<<grid_for(n, 256, 2368), 256, 0, (cudaStream_t)stream>>>(in, n, out);
  SCX_CHECK_LAUNCH("widen_u32_kernel");
  return SCX_OK;
}

// One-pass unordered selection of a direct table's groups passing HAVING
// (warp-aggregated atomics): for selective HAVING the ordered two-pass
// compaction reads the whole table twice to write a handful of rows.
__global__ void direct_select_kernel(Occ O, const int64_t* acc, int64_t cap, int m,
                                     uint64_t* out_keys, int64_t* out_acc,
                                     unsigned long long* count) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < cap;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = base + threadIdx.x;
    const bool keep = e < cap && O.keep(acc + e * m);
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (!bal) continue;
    unsigned long long o = 0;
    const int leader = __ffs(bal) - 1;
    if (lane == leader) o = atomicAdd(count, (unsigned long long)__popc(bal));
    o = __shfl_sync(0xffffffffu, o, leader) + __popc(bal & ((1u << lane) - 1u));
    if (keep) {
      out_keys[o] = (uint64_t)e;
      for (int j = 0; j < m; ++j) out_acc[(int64_t)j * cap + (int64_t)o] = acc[e * m + j];
    }
  }
}

extern "C" int scx_direct_agg_select_having(const int64_t* acc, int64_t cap, int m, int occ_word,
                                            int hv_word, int64_t hv_lo, int64_t hv_hi,
                                            uint64_t* out_keys, int64_t* out_acc,
                                            uint64_t* count, void* stream) {
  if (!acc || !out_keys || !out_acc || !count || m < 1 || m > 16 || occ_word < 0 ||
      occ_word >= m || hv_word < 0 || hv_word >= m || cap < 0) {
    set_error("direct_agg_select_having: bad arguments");
    return SCX_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  SCX_CUDA(cudaMemsetAsync(count, 0, 8, st));
  if (cap == 0) return SCX_OK;
  Occ O{nullptr, acc, m, occ_word, hv_word, hv_lo, hv_hi};
  direct_select_kernel<<<grid_for(cap, 256, 148 * 16), 256, 0, st>>>(
      O, acc, cap, m, out_keys, out_acc, reinterpret_cast<unsigned long long*>(count));
  SCX_CHECK_LAUNCH("direct_select_kernel");
  return SCX_OK;
}


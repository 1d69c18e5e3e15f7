// partition.cu -- hash partitioning of a table into n_parts destinations
// (exchange.py:52-70 partition_indices / hash_partition: the reference takes
// a STABLE argsort of `hash_keys(t, keys) % n` and then `take`s every column;
// exchange.py:131-174 shuffle_table sends part j to worker j).
//
// Two passes over CTA tiles of kTile rows (256 threads, 16 rows per thread,
// warp w owns the contiguous rows [512w, 512w + 512) of the tile):
//
//   pass 1  part_hist_kernel : bucket per row from the key columns (read
//           straight from HBM, coalesced); a warp-aggregated histogram
//           (__match_any_sync -> one shared-memory atomic per distinct bucket
//           per 32 rows) -> per-(part, tile) counts.  A part-major exclusive
//           scan of those gives every tile, for every part, the position of
//           its first row of that part; part totals go to counts_dev.
//   pass 2  part_scatter_kernel : the tile's columns are staged into shared
//           memory by TMA bulk copies (cp.async.bulk + mbarrier; 16-byte
//           aligned bodies, tails by plain loads), the buckets are recomputed
//           from the staged key column (the key is read from HBM only by
//           pass 1 and the copy itself), rows are ranked stably within the
//           tile (per-warp running counters + __match_any_sync ranks, then a
//           per-part scan over warps), and the inverse permutation
//           `src_of[local position]` is built in shared memory.  Each column
//           is then written part by part as contiguous runs: consecutive
//           threads store consecutive destination addresses, so every
//           part's run of the tile leaves as full coalesced lines.
//
// Destinations: `contig` mode writes part d of column c at
// outs[c] + (part start + rank) * width (hash_partition's layout);
// destination mode writes it at dst[c * n_parts + d] + rank_in_part * width
// where dst holds arbitrary device byte addresses: a local receive buffer,
// another virtual worker's buffer on the same device, or a peer GPU's HBM
// (P2P over NVLink) -- the partition kernel IS the send of a shuffle.
#include <stdlib.h>
#include <string.h>

#include <type_traits>

#include "common.cuh"

namespace scx {

int scan_u32_excl(const uint32_t* in, uint64_t* out, int64_t m, uint64_t* tmp, cudaStream_t st);
int64_t scan_tmp_words(int64_t m);

namespace part {

constexpr int kT = 256;                    // threads per CTA
constexpr int kW = kT / 32;                // warps
constexpr int kPer = 8;                    // rows per thread
constexpr int kTile = kT * kPer;           // 2048 rows per tile
constexpr int kSeg = kTile / kW;           // 256 rows per warp segment
constexpr int kMaxParts = 64;
constexpr uint64_t kFib2 = kFib * kFib;    // single key: (0 ^ v*F) * F == v * F^2

struct Keys {
  scx_column k[SCX_MAX_KEYS];
  int n;
  uint32_t np;
  uint64_t magic;                          // floor((2^64 - 1) / np) for h % np
  int staged;                              // single key == payload column 0 (staged by TMA)
  int nbits;                               // bits of a bucket id: ceil(log2(np))
};
struct Cols {
  scx_column in[SCX_MAX_OUT];
  uint64_t out[SCX_MAX_OUT];               // contig mode: output column base
  int orig[SCX_MAX_OUT];                   // dst mode: the column's index in dst
  int n;
};

__device__ __forceinline__ uint32_t bucket(const Keys& K, uint64_t h) {
  if ((K.np & (K.np - 1)) == 0) return (uint32_t)h & (K.np - 1);
  // h mod np by multiply-high: q is floor(h / np) or one less
  const uint64_t q = __umul64hi(h, K.magic);
  uint64_t r = h - q * K.np;
  if (r >= K.np) r -= K.np;
  return (uint32_t)r;
}

__device__ __forceinline__ uint64_t hash_generic(const Keys& K, int64_t i) {
  if (K.n == 1)
    return (uint64_t)load_i64(reinterpret_cast<const void*>(K.k[0].ptr), K.k[0].dtype, i) * kFib2;
  uint64_t acc = 0;
  for (int j = 0; j < K.n; ++j)
    acc = fib_step(acc, load_i64(reinterpret_cast<const void*>(K.k[j].ptr), K.k[j].dtype, i));
  return acc;
}

// Buckets of `cnt` rows {base + s * 32 + lane} (s < kPer) of one warp.  KT is
// the single key's physical type: all kPer loads are issued before any use
// (no per-row branch between them); void = generic (multi-key / switch).
template <typename KT>
__device__ __forceinline__ void warp_buckets(const Keys& K, int64_t base, int64_t n, int lane,
                                             uint32_t (&d)[kPer]) {
  if constexpr (!std::is_void<KT>::value) {
    const KT* k = reinterpret_cast<const KT*>(K.k[0].ptr);
    KT v[kPer];
    if (base + (kPer - 1) * 32 + 31 < n) {
#pragma unroll
      for (int s = 0; s < kPer; ++s) v[s] = __ldg(k + base + s * 32 + lane);
    } else {
#pragma unroll
      for (int s = 0; s < kPer; ++s) {
        const int64_t i = base + s * 32 + lane;
        v[s] = i < n ? __ldg(k + i) : KT(0);
      }
    }
#pragma unroll
    for (int s = 0; s < kPer; ++s)
      d[s] = base + s * 32 + lane < n ? bucket(K, (uint64_t)(int64_t)v[s] * kFib2) : 0xFFFFFFFFu;
  } else {
#pragma unroll
    for (int s = 0; s < kPer; ++s) {
      const int64_t i = base + s * 32 + lane;
      d[s] = i < n ? bucket(K, hash_generic(K, i)) : 0xFFFFFFFFu;
    }
  }
}

// pass 1: per-(part, tile) row counts.  Each warp keeps a private histogram
// in shared memory (no cross-warp contention); lanes add with shared-memory
// atomics.  Grid-strided over tiles so the key loads of the next tile are
// issued while the last tile's counts are written.
template <typename KT>
__global__ void __launch_bounds__(kT) part_hist_kernel(const __grid_constant__ Keys K, int64_t n,
                                                       uint32_t* cnt, int64_t nb) {
  __shared__ uint32_t h[kW][kMaxParts];
  const int np = (int)K.np;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t t = blockIdx.x; t < nb; t += gridDim.x) {
    for (int j = threadIdx.x; j < kW * kMaxParts; j += kT) (&h[0][0])[j] = 0;
    __syncthreads();
    uint32_t d[kPer];
    warp_buckets<KT>(K, t * kTile + w * kSeg, n, lane, d);
#pragma unroll
    for (int s = 0; s < kPer; ++s)
      if (d[s] != 0xFFFFFFFFu) atomicAdd(&h[w][d[s]], 1u);
    __syncthreads();
    for (int p = threadIdx.x; p < np; p += kT) {
      uint32_t c = 0;
#pragma unroll
      for (int ww = 0; ww < kW; ++ww) c += h[ww][p];
      cnt[(int64_t)p * nb + t] = c;
    }
    __syncthreads();
  }
}

__global__ void part_totals_kernel(const uint64_t* offs, int np, int64_t nb, uint64_t* counts) {
  for (int p = threadIdx.x; p < np; p += blockDim.x)
    counts[p] = offs[(int64_t)(p + 1) * nb] - offs[(int64_t)p * nb];
}

struct alignas(128) Smem {
  uint64_t stage[2][kTile];                // TMA ring: two column tiles, source row order
  uint64_t perm[kTile];                    // one column tile in partition order
  uint16_t pos[kTile];                     // tile row -> tile-local partition-order position
  union {                                  // (wcnt while ranking, pid while moving columns)
    uint32_t wcnt[kW][kMaxParts];          // per-warp running counts -> warp prefix
    uint8_t pid[kTile];                    // tile-local position -> its part
  };
  uint64_t dptr[kMaxParts];                // this column: byte address of position 0's slot in part p
  uint32_t lbase[kMaxParts + 1];           // tile-local start of each part
  int64_t rel[kMaxParts];                  // destination row of tile-local position 0 of part p
  uint64_t bar[2];
};

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Stage column c's rows [t0, t0 + rows) into `buf`: a 16-byte aligned source
// moves its aligned body by one bulk copy (thread 0 issues; completion on
// `bar`), the < 16-byte tail -- or all of an unaligned source (a column
// view at an odd offset) -- by plain loads from every thread.
__device__ __forceinline__ void stage_column(const scx_column& c, int64_t t0, int rows, void* buf,
                                             uint64_t* bar) {
  const int w = dtype_size_d(c.dtype);
  const uint64_t src = c.ptr + (uint64_t)t0 * w;
  const uint32_t bytes = (uint32_t)rows * w;
  const uint32_t body = (src & 15) ? 0u : (bytes & ~15u);
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, body);
    if (body) bulk_g2s(buf, reinterpret_cast<const void*>(src), body, bar);
  }
  unsigned char* d = static_cast<unsigned char*>(buf);
  const unsigned char* g = reinterpret_cast<const unsigned char*>(src);
  for (uint32_t b = body + threadIdx.x; b < bytes; b += kT) d[b] = __ldg(g + b);
}

// Column tile: staged (source order) -> perm (partition order) in shared
// memory, then out part-run by part-run: thread j writes position j, so a
// warp's 32 stores are consecutive destination addresses.
template <typename T>
__device__ __forceinline__ void move_column(Smem& S, const T* stage, int rows) {
  const int tid = threadIdx.x;
  T* perm = reinterpret_cast<T*>(S.perm);
#pragma unroll
  for (int s = 0; s < kPer; ++s) {
    const int r = s * kT + tid;            // conflict-free linear reads
    if (r < rows) perm[S.pos[r]] = stage[r];
  }
  __syncthreads();
  // position j belongs to part pid[j]; its slot is dptr[p] + j (dptr folds
  // the part's destination base and the tile's offset inside the part)
#pragma unroll
  for (int s = 0; s < kPer; ++s) {
    const int j = s * kT + tid;
    if (j < rows) reinterpret_cast<T*>(S.dptr[S.pid[j]])[j] = perm[j];
  }
}

// pass 2.  dst == nullptr: contiguous layout (C.out, part-major, exactly
// hash_partition's); else dst[orig(c) * np + p] is the byte address where
// this source's part-p rows of column c begin.
template <typename KT>
__global__ void __launch_bounds__(kT, 4) part_scatter_kernel(const __grid_constant__ Keys K,
                                                             const __grid_constant__ Cols C,
                                                             int64_t n,
                                                             const uint64_t* __restrict__ offs,
                                                             int64_t nb,
                                                             const uint64_t* __restrict__ dst) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int np = (int)K.np;
  // persistent: this CTA walks tiles blockIdx.x, + gridDim.x, ...; the TMA
  // ring runs over the flattened (tile, column) sequence q, so the next
  // tile's first columns are in flight while this tile is written out
  const int64_t my_tiles = (nb - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int64_t Q = my_tiles * C.n;
  auto issue = [&](int64_t q) {
    if (q >= Q) return;
    const int64_t tq = blockIdx.x + (q / C.n) * (int64_t)gridDim.x;
    const int rq = (int)min((int64_t)kTile, n - tq * kTile);
    stage_column(C.in[q % C.n], tq * kTile, rq, S.stage[q & 1], &S.bar[q & 1]);
  };
  if (tid == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  issue(0);
  issue(1);

  for (int64_t it = 0; it < my_tiles; ++it) {
    const int64_t tile = blockIdx.x + it * (int64_t)gridDim.x;
    const int64_t t0 = tile * kTile;
    const int rows = (int)min((int64_t)kTile, n - t0);
    const int64_t q0 = it * C.n;
    for (int j = tid; j < kW * kMaxParts; j += kT) (&S.wcnt[0][0])[j] = 0;
    __syncthreads();

    // ---- buckets + stable ranks (warp w: tile rows [256w, 256w + 256) in order)
    uint32_t d[kPer];
    if (K.staged) {                        // the key is payload column 0: read its staged tile
      mbar_wait(&S.bar[q0 & 1], (q0 >> 1) & 1);
      __syncthreads();                     // plain-loaded tail bytes
      const void* kt = S.stage[q0 & 1];
#pragma unroll
      for (int s = 0; s < kPer; ++s) {
        const int r = w * kSeg + s * 32 + lane;
        d[s] = r < rows ? bucket(K, (uint64_t)load_i64(kt, K.k[0].dtype, r) * kFib2)
                        : 0xFFFFFFFFu;
      }
    } else {
      warp_buckets<KT>(K, t0 + w * kSeg, n, lane, d);
    }
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t rk[kPer];
#pragma unroll
    for (int s = 0; s < kPer; ++s) {
      // lanes with the same bucket: one ballot per bucket bit (np <= 64:
      // at most 6) instead of match.any
      const bool valid = d[s] != 0xFFFFFFFFu;
      const uint32_t vb = __ballot_sync(0xffffffffu, valid);
      uint32_t peers = valid ? vb : ~vb;
      for (int k = 0; k < K.nbits; ++k) {
        const bool bit = (d[s] >> k) & 1u;
        const uint32_t b = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? b : ~b;
      }
      uint32_t before = 0;
      if (d[s] != 0xFFFFFFFFu) before = S.wcnt[w][d[s]];
      __syncwarp();
      if (d[s] != 0xFFFFFFFFu && (peers & lt) == 0) S.wcnt[w][d[s]] = before + __popc(peers);
      __syncwarp();
      rk[s] = before + __popc(peers & lt);
    }
    __syncthreads();
    for (int p = tid; p < np; p += kT) {   // per part: exclusive scan over warps
      uint32_t run = 0;
#pragma unroll
      for (int ww = 0; ww < kW; ++ww) { const uint32_t c = S.wcnt[ww][p]; S.wcnt[ww][p] = run; run += c; }
      S.lbase[p + 1] = run;                // part total, scanned below
    }
    __syncthreads();
    if (w == 0) {                          // exclusive scan of part totals (np <= 64)
      uint32_t carry = 0;
      for (int p0 = 0; p0 < np; p0 += 32) {
        const int p = p0 + lane;
        const uint32_t v = p < np ? S.lbase[p + 1] : 0;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (p < np) S.lbase[p] = carry + x - v;
        carry += __shfl_sync(0xffffffffu, x, 31);
      }
      if (lane == 0) {
        S.lbase[np] = carry;               // == rows
        for (int p = np + 1; p <= kMaxParts; ++p) S.lbase[p] = 0xFFFFFFFFu;
      }
    }
    __syncthreads();
    for (int p = tid; p < np; p += kT) {
      const int64_t o = (int64_t)offs[(int64_t)p * nb + tile];
      S.rel[p] = (dst ? o - (int64_t)offs[(int64_t)p * nb] : o) - (int64_t)S.lbase[p];
    }
#pragma unroll
    for (int s = 0; s < kPer; ++s)
      if (d[s] != 0xFFFFFFFFu) rk[s] += S.lbase[d[s]] + S.wcnt[w][d[s]];
    __syncthreads();                       // wcnt is dead: its bytes become pid
#pragma unroll
    for (int s = 0; s < kPer; ++s)
      if (d[s] != 0xFFFFFFFFu) {
        S.pos[w * kSeg + s * 32 + lane] = (uint16_t)rk[s];
        S.pid[rk[s]] = (uint8_t)d[s];
      }

    // ---- every column: TMA-staged tile -> partition order -> part runs
    for (int c = 0; c < C.n; ++c) {
      const int64_t q = q0 + c;
      const int b = (int)(q & 1);
      {
        const int wdt = dtype_size_d(C.in[c].dtype);
        for (int p = tid; p < np; p += kT)
          S.dptr[p] = (dst ? dst[(int64_t)C.orig[c] * np + p] : C.out[c]) + (uint64_t)(S.rel[p] * wdt);
      }
      mbar_wait(&S.bar[b], (q >> 1) & 1);
      __syncthreads();                     // pos / pid / dptr / plain-loaded tail bytes visible
      switch (dtype_size_d(C.in[c].dtype)) {
        case 1: move_column(S, reinterpret_cast<const uint8_t*>(S.stage[b]), rows); break;
        case 2: move_column(S, reinterpret_cast<const uint16_t*>(S.stage[b]), rows); break;
        case 4: move_column(S, reinterpret_cast<const uint32_t*>(S.stage[b]), rows); break;
        default: move_column(S, reinterpret_cast<const uint64_t*>(S.stage[b]), rows); break;
      }
      // stage[b] was consumed before move_column's barrier: refill it with q + 2
      if (tid == 0) fence_proxy_async_smem();
      issue(q + 2);
      __syncthreads();                     // perm / dptr reuse
    }
  }
}

// pass 2, direct variant: no shared-memory staging of the data at all.
// Each lane keeps the bucket and stable rank of its 8 rows in registers;
// after one CTA-wide prefix of the per-warp part counts every row's final
// slot is known and each column is loaded (coalesced) and stored straight to
// it.  A warp's 32 rows of one step land in at most np contiguous runs, one
// per part, and neighbouring warps extend the same runs, so L2 merges the
// partial sectors at run ends before they reach HBM.
struct DirectSmem {
  uint32_t wcnt[2][kW][kMaxParts];         // per-warp part counts -> warp prefix (tile parity)
  int64_t tb[2][kMaxParts];                // tile's first slot of part p (within the part / global)
  uint64_t base[SCX_MAX_OUT][kMaxParts];   // destination byte address of slot 0 of part p
};

template <typename T>
__device__ __forceinline__ void direct_column(const scx_column& in, const DirectSmem& S, int c,
                                              int64_t r0, int64_t n, int lane,
                                              const uint32_t (&d)[kPer],
                                              const uint64_t (&slot)[kPer]) {
  const T* src = reinterpret_cast<const T*>(in.ptr);
  T v[kPer];
#pragma unroll
  for (int s = 0; s < kPer; ++s) {
    const int64_t i = r0 + s * 32 + lane;
    v[s] = i < n ? __ldg(src + i) : T(0);
  }
#pragma unroll
  for (int s = 0; s < kPer; ++s)
    if (d[s] != 0xFFFFFFFFu) {
      T* dstp = reinterpret_cast<T*>(S.base[c][d[s]]);
      __stcs(dstp + slot[s], v[s]);
    }
}

template <typename KT>
__global__ void __launch_bounds__(kT, 4) part_scatter_direct_kernel(const __grid_constant__ Keys K,
                                                                    const __grid_constant__ Cols C,
                                                                    int64_t n,
                                                                    const uint64_t* __restrict__ offs,
                                                                    int64_t nb,
                                                                    const uint64_t* __restrict__ dst) {
  __shared__ DirectSmem S;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int np = (int)K.np;
  for (int j = tid; j < 2 * kW * kMaxParts; j += kT) (&S.wcnt[0][0][0])[j] = 0;
  for (int j = tid; j < C.n * np; j += kT) {
    const int c = j / np, p = j % np;
    S.base[c][p] = dst ? dst[(int64_t)C.orig[c] * np + p] : C.out[c];
  }
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
  int par = 0;
  for (int64_t tile = blockIdx.x; tile < nb; tile += gridDim.x, par ^= 1) {
    const int64_t r0 = tile * kTile + w * kSeg;
    uint32_t d[kPer];
    warp_buckets<KT>(K, r0, n, lane, d);
    uint32_t rk[kPer];
#pragma unroll
    for (int s = 0; s < kPer; ++s) {
      const bool valid = d[s] != 0xFFFFFFFFu;
      const uint32_t vb = __ballot_sync(0xffffffffu, valid);
      uint32_t peers = valid ? vb : ~vb;
      for (int k = 0; k < K.nbits; ++k) {
        const bool bit = (d[s] >> k) & 1u;
        const uint32_t b = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? b : ~b;
      }
      uint32_t before = 0;
      if (valid) before = S.wcnt[par][w][d[s]];
      __syncwarp();
      if (valid && (peers & lt) == 0) S.wcnt[par][w][d[s]] = before + __popc(peers);
      __syncwarp();
      rk[s] = before + __popc(peers & lt);
    }
    __syncthreads();
    for (int p = tid; p < np; p += kT) {
      uint32_t run = 0;
#pragma unroll
      for (int ww = 0; ww < kW; ++ww) { const uint32_t c = S.wcnt[par][ww][p]; S.wcnt[par][ww][p] = run; run += c; }
      const int64_t o = (int64_t)offs[(int64_t)p * nb + tile];
      S.tb[par][p] = dst ? o - (int64_t)offs[(int64_t)p * nb] : o;
    }
    for (int j = tid; j < kW * kMaxParts; j += kT) (&S.wcnt[par ^ 1][0][0])[j] = 0;
    __syncthreads();
    uint64_t slot[kPer];             // 64-bit: a 64 GiB table has 2^32 rows
#pragma unroll
    for (int s = 0; s < kPer; ++s)
      slot[s] = d[s] != 0xFFFFFFFFu ? (uint64_t)(S.tb[par][d[s]] + S.wcnt[par][w][d[s]] + rk[s]) : 0ull;
    for (int c = 0; c < C.n; ++c) {
      switch (dtype_size_d(C.in[c].dtype)) {
        case 1: direct_column<uint8_t>(C.in[c], S, c, r0, n, lane, d, slot); break;
        case 2: direct_column<uint16_t>(C.in[c], S, c, r0, n, lane, d, slot); break;
        case 4: direct_column<uint32_t>(C.in[c], S, c, r0, n, lane, d, slot); break;
        default: direct_column<uint64_t>(C.in[c], S, c, r0, n, lane, d, slot); break;
      }
    }
  }
}

// launch `F<KT>` for the single key's physical type (generic otherwise)
template <template <typename> class F, typename... A>
static void by_key_type(const Keys& K, A&&... a) {
  if (K.n != 1) return F<void>::run(a...);
  switch (K.k[0].dtype) {
    case SCX_I8: return F<int8_t>::run(a...);
    case SCX_U8: return F<uint8_t>::run(a...);
    case SCX_I16: return F<int16_t>::run(a...);
    case SCX_U16: return F<uint16_t>::run(a...);
    case SCX_I32: return F<int32_t>::run(a...);
    case SCX_U32: return F<uint32_t>::run(a...);
    case SCX_I64: return F<int64_t>::run(a...);
    default: return F<void>::run(a...);
  }
}

static int g_sms = 0;

template <typename KT>
struct HistLaunch {
  static void run(const Keys& K, int64_t n, uint32_t* cnt, int64_t nb, cudaStream_t st) {
    const int64_t cap = (int64_t)(g_sms > 0 ? g_sms : 148) * 8;
    part_hist_kernel<KT><<<(unsigned)(nb < cap ? nb : cap), kT, 0, st>>>(K, n, cnt, nb);
  }
};

template <typename KT>
struct ScatterLaunch {
  static void run(const Keys& K, const Cols& C, int64_t n, const uint64_t* offs, int64_t nb,
                  const uint64_t* dst, cudaStream_t st) {
    static bool attr = false;              // idempotent; racing threads set the same value
    if (!attr) {
      cudaFuncSetAttribute(part_scatter_kernel<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)sizeof(Smem));
      attr = true;
    }
    static const int64_t per_sm = getenv("SCX_PART_CTAS") ? atoll(getenv("SCX_PART_CTAS")) : 4;
    const int64_t cap = per_sm > 0 ? (int64_t)(g_sms > 0 ? g_sms : 148) * per_sm : nb;
    // direct stores coalesce while a warp's 32 rows fall into few parts:
    // measured (1 GiB, 16-byte rows) 8 parts 0.626 vs 0.742 ms staged, 64
    // parts 2.29 vs 0.84 ms -- the staged kernel takes the wide fan-outs
    const char* env = getenv("SCX_PART_DIRECT");
    const bool direct = env ? env[0] != '0' : K.np <= 8;
    if (direct) {
      const int64_t dcap = (int64_t)(g_sms > 0 ? g_sms : 148) * 8;
      part_scatter_direct_kernel<KT><<<(unsigned)(nb < dcap ? nb : dcap), kT, 0, st>>>(
          K, C, n, offs, nb, dst);
      return;
    }
    part_scatter_kernel<KT><<<(unsigned)(nb < cap ? nb : cap), kT, sizeof(Smem), st>>>(
        K, C, n, offs, nb, dst);
  }
};

static int64_t tiles(int64_t n) { return (n + kTile - 1) / kTile; }

// ws: counts u32[np * nb] (256-B padded) | offs u64[np * nb + 1] | scan scratch
static int64_t ws_bytes(int64_t n, int np) {
  const int64_t nb = tiles(n) > 0 ? tiles(n) : 1;
  const int64_t m = (int64_t)np * nb;
  return ((m * 4 + 255) / 256) * 256 + (m + 1) * 8 + 8 * scan_tmp_words(m) + 256;
}

static int load_keys(const scx_column* keys, int n_keys, int np, Keys& K) {
  if (!keys || n_keys < 1 || n_keys > SCX_MAX_KEYS) {
    set_error("partition: %d key columns (1..%d)", n_keys, SCX_MAX_KEYS);
    return SCX_EINVAL;
  }
  memset(&K, 0, sizeof(K));
  K.n = n_keys;
  K.np = (uint32_t)np;
  K.magic = ~0ull / (uint64_t)np;
  K.staged = 0;
  K.nbits = 0;
  while ((1 << K.nbits) < np) ++K.nbits;
  for (int i = 0; i < n_keys; ++i) {
    if (dtype_size(keys[i].dtype) == 0) {
      set_error("partition: key %d has bad dtype %d", i, keys[i].dtype);
      return SCX_EINVAL;
    }
    K.k[i] = keys[i];
  }
  return SCX_OK;
}

static uint64_t* offs_of(void* ws, int64_t nb, int np) {
  return reinterpret_cast<uint64_t*>(static_cast<char*>(ws) + ((np * nb * 4 + 255) / 256) * 256);
}

static int hist(const Keys& K, int64_t n, void* ws, uint64_t* counts, cudaStream_t st) {
  const int np = (int)K.np;
  const int64_t nb = tiles(n);
  uint32_t* cnt = static_cast<uint32_t*>(ws);
  uint64_t* offs = offs_of(ws, nb, np);
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  by_key_type<HistLaunch>(K, K, n, cnt, nb, st);
  SCX_CHECK_LAUNCH("part_hist_kernel");
  int rc = scan_u32_excl(cnt, offs, np * nb, offs + np * nb + 1, st);
  if (rc) return rc;
  part_totals_kernel<<<1, 256, 0, st>>>(offs, np, nb, counts);
  SCX_CHECK_LAUNCH("part_totals_kernel");
  return SCX_OK;
}

static int scatter(Keys K, const scx_column* cols, const scx_column* outs, int n_cols,
                   int64_t n, const uint64_t* dst, const void* ws, cudaStream_t st) {
  if (n_cols < 0 || n_cols > SCX_MAX_OUT || (n_cols > 0 && !cols)) {
    set_error("partition: %d columns (0..%d)", n_cols, SCX_MAX_OUT);
    return SCX_EINVAL;
  }
  // a payload column that IS the single key goes first: its staged tile
  // feeds the hash, so the key is not read from HBM a second time
  int first = -1;
  if (K.n == 1)
    for (int i = 0; i < n_cols; ++i)
      if (cols[i].ptr == K.k[0].ptr && cols[i].dtype == K.k[0].dtype) { first = i; break; }
  K.staged = first >= 0;
  Cols C;
  memset(&C, 0, sizeof(C));
  C.n = n_cols;
  int j = 0;
  for (int pass = 0; pass < 2; ++pass)
    for (int i = 0; i < n_cols; ++i) {
      if ((pass == 0) != (i == first)) continue;
      const int wdt = dtype_size(cols[i].dtype);
      if (wdt == 0 || (outs && dtype_size(outs[i].dtype) != wdt)) {
        set_error("partition: column %d bad dtype / in-out width mismatch", i);
        return SCX_EINVAL;
      }
      C.in[j] = cols[i];
      C.out[j] = outs ? outs[i].ptr : 0;
      C.orig[j] = i;
      ++j;
    }
  if (n_cols == 0 || n == 0) return SCX_OK;
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t nb = tiles(n);
  by_key_type<ScatterLaunch>(K, K, C, n, offs_of(const_cast<void*>(ws), nb, (int)K.np), nb, dst, st);
  SCX_CHECK_LAUNCH("part_scatter_kernel");
  return SCX_OK;
}

}  // namespace part
}  // namespace scx

using namespace scx;

extern "C" int64_t scx_part_workspace(int64_t n, int n_parts) {
  return part::ws_bytes(n, n_parts < 1 ? 1 : n_parts);
}

extern "C" int scx_part_hist(const scx_column* keys, int n_keys, int64_t n, int n_parts,
                             void* ws_dev, uint64_t* counts_dev, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n < 0 || n_parts < 1 || n_parts > part::kMaxParts || !counts_dev || (n > 0 && !ws_dev)) {
    set_error("scx_part_hist: bad arguments (n=%lld parts=%d)", (long long)n, n_parts);
    return SCX_EINVAL;
  }
  part::Keys K;
  int rc = part::load_keys(keys, n_keys, n_parts, K);
  if (rc) return rc;
  if (n == 0) {
    SCX_CUDA(cudaMemsetAsync(counts_dev, 0, 8 * (size_t)n_parts, st));
    return SCX_OK;
  }
  return part::hist(K, n, ws_dev, counts_dev, st);
}

extern "C" int scx_part_scatter(const scx_column* keys, int n_keys, const scx_column* cols,
                                int n_cols, int64_t n, int n_parts, const uint64_t* dst_dev,
                                const void* ws_dev, void* stream) {
  if (n < 0 || n_parts < 1 || n_parts > part::kMaxParts || (n > 0 && (!ws_dev || !dst_dev))) {
    set_error("scx_part_scatter: bad arguments (n=%lld parts=%d)", (long long)n, n_parts);
    return SCX_EINVAL;
  }
  part::Keys K;
  int rc = part::load_keys(keys, n_keys, n_parts, K);
  if (rc) return rc;
  return part::scatter(K, cols, nullptr, n_cols, n, dst_dev, ws_dev,
                       static_cast<cudaStream_t>(stream));
}

extern "C" int64_t scx_partition_workspace(int64_t n, int n_parts) {
  return part::ws_bytes(n, n_parts < 1 ? 1 : n_parts);
}

extern "C" int scx_partition(const scx_column* keys, int n_keys, const scx_column* cols,
                             const scx_column* outs, int n_cols, int64_t n, int n_parts,
                             uint64_t* counts, void* temp, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n < 0 || n_parts < 1 || n_parts > part::kMaxParts || !counts || (n > 0 && !temp) ||
      (n_cols > 0 && !outs)) {
    set_error("partition: bad arguments (cols=%d parts=%d)", n_cols, n_parts);
    return SCX_EINVAL;
  }
  part::Keys K;
  int rc = part::load_keys(keys, n_keys, n_parts, K);
  if (rc) return rc;
  if (n == 0) {
    SCX_CUDA(cudaMemsetAsync(counts, 0, 8 * (size_t)n_parts, st));
    return SCX_OK;
  }
  rc = part::hist(K, n, temp, counts, st);
  if (rc) return rc;
  return part::scatter(K, cols, outs, n_cols, n, nullptr, temp, st);
}

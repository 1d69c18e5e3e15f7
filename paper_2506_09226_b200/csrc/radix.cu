// radix.cu -- stable 8-bit-digit counting passes shared by
//   * scx_sort_pairs   : LSD radix sort (ColumnTable.sort_by, table.py:198-214)
//   * scx_hash_keys    : raw Fibonacci hashes (exchange.py:35-49)
//
// Each CTA owns a contiguous chunk of kChunk rows processed as 16 sub-tiles of
// 256 rows in order.  Stability within a sub-tile comes from a per-warp
// __match_any_sync rank plus a per-(warp, digit) exclusive scan in shared
// memory; across CTAs from a digit-major exclusive scan of the per-CTA
// histograms.  So every element's output position is the same as a stable
// sort by digit, which is exactly partition_indices' stable argsort.
#include "common.cuh"

namespace scx {

constexpr int kDigits = 256;
constexpr int kItems = 16;
constexpr int kChunk = kBlock * kItems;   // 4096 rows per CTA

struct PartKeys {
  scx_column k[SCX_MAX_KEYS];
  int n;
};

__device__ __forceinline__ uint64_t fib_hash_row(const PartKeys& K, int64_t i) {
  uint64_t acc = 0;
  for (int j = 0; j < K.n; ++j)
    acc = fib_step(acc, load_i64(reinterpret_cast<const void*>(K.k[j].ptr), K.k[j].dtype, i));
  return acc;
}

__device__ __forceinline__ uint32_t bucket_of(const PartKeys& K, int64_t i, uint32_t nparts) {
  const uint64_t h = fib_hash_row(K, i);
  return (nparts & (nparts - 1)) == 0 ? (uint32_t)(h & (nparts - 1)) : (uint32_t)(h % nparts);
}

// digit source: sort pass (key >> shift) & 255, or partition bucket
struct DigitSrc {
  const uint64_t* keys;
  int shift;
  PartKeys pk;
  uint32_t nparts;
  __device__ __forceinline__ uint32_t operator()(int64_t i) const {
    return keys ? (uint32_t)((keys[i] >> shift) & 255u) : bucket_of(pk, i, nparts);
  }
};

__global__ void hist_kernel(DigitSrc D, int64_t n, int ndig, uint32_t* counts, int nblocks) {
  __shared__ uint32_t h[kDigits];
  for (int d = threadIdx.x; d < kDigits; d += kBlock) h[d] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  for (int it = 0; it < kItems; ++it) {
    const int64_t i = base + it * kBlock + threadIdx.x;
    if (i < n) atomicAdd(&h[D(i)], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < ndig; d += kBlock) counts[(int64_t)d * nblocks + blockIdx.x] = h[d];
}

// stable scatter; `emit(i, pos)` writes element i to pos
template <typename Emit>
__device__ __forceinline__ void scatter_chunk(const DigitSrc& D, int64_t n, int ndig,
                                              const uint64_t* offs, int nblocks, Emit emit) {
  __shared__ uint32_t wc[kWarps][kDigits];
  __shared__ uint64_t run[kDigits];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int d = tid; d < kDigits; d += kBlock)
    run[d] = d < ndig ? offs[(int64_t)d * nblocks + blockIdx.x] : 0;
  const int64_t base = (int64_t)blockIdx.x * kChunk;
  for (int it = 0; it < kItems; ++it) {
    // only the ndig live digit columns (8 for an 8-way partition, 256 for sort)
    for (int j = tid; j < kWarps * ndig; j += kBlock) wc[j / ndig][j % ndig] = 0;
    __syncthreads();
    const int64_t i = base + it * kBlock + tid;
    const bool valid = i < n;
    const uint32_t d = valid ? D(i) : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (valid && rank == 0) wc[warp][d] = __popc(peers);
    __syncthreads();
    // per digit: exclusive scan over warps (thread d owns digit d)
    for (int dd = tid; dd < ndig; dd += kBlock) {
      uint32_t s = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) { const uint32_t c = wc[w][dd]; wc[w][dd] = s; s += c; }
      // stash total in run after positions are computed: use a second pass
      // (run is read below before being advanced)
      (void)s;
    }
    __syncthreads();
    uint64_t pos = 0;
    if (valid) pos = run[d] + wc[warp][d] + rank;
    __syncthreads();
    if (valid) emit(i, pos);
    // advance run[d] by this sub-tile's count of digit d: the last element of
    // each digit group (highest warp, highest rank) knows the total.
    if (valid && (peers >> lane) == 1u) {
      // am I the last lane of my peer group in the highest warp holding d?
      // total = wc[warp][d] + popc(peers) only if no later warp has digit d;
      // resolved with an atomic max on the candidate end position instead.
      atomicMax(reinterpret_cast<unsigned long long*>(&run[d]), (unsigned long long)(pos + 1));
    }
    __syncthreads();
  }
}

__global__ void sort_scatter_kernel(DigitSrc D, int64_t n, const uint64_t* offs, int nblocks,
                                    const uint64_t* kin, const uint32_t* vin, uint64_t* kout,
                                    uint32_t* vout) {
  scatter_chunk(D, n, kDigits, offs, nblocks, [&](int64_t i, uint64_t pos) {
    kout[pos] = kin[i];
    vout[pos] = vin[i];
  });
}

__global__ void hash_keys_kernel(PartKeys K, int64_t n, uint64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = fib_hash_row(K, i);
}

__global__ void copy_pairs_kernel(const uint64_t* ki, const uint32_t* vi, uint64_t* ko,
                                  uint32_t* vo, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    ko[i] = ki[i];
    vo[i] = vi[i];
  }
}

// ---- small inputs: one CTA, bitonic sort in shared memory -------------------
// Final ORDER BYs and top-k inputs are usually a few hundred rows; the LSD
// radix path would spend 5 launches per 8-bit digit on them.  Stability: ties
// are broken by input position (not by the value payload), so a multi-word
// LSD sort that feeds a previous pass's permutation as values stays stable.
constexpr int kSmallSort = 2048;

__global__ void __launch_bounds__(1024) small_sort_kernel(const uint64_t* kin, const uint32_t* vin,
                                                          uint64_t* kout, uint32_t* vout, int n) {
  __shared__ uint64_t k[kSmallSort];
  __shared__ uint32_t v[kSmallSort];
  __shared__ uint16_t p[kSmallSort];
  for (int i = threadIdx.x; i < kSmallSort; i += blockDim.x) {
    const bool in = i < n;
    k[i] = in ? kin[i] : ~0ull;
    v[i] = in ? vin[i] : 0u;
    p[i] = (uint16_t)i;               // padding sorts last: key max, position >= n
  }
  __syncthreads();
  for (int size = 2; size <= kSmallSort; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < kSmallSort / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const bool gt = k[lo] > k[hi] || (k[lo] == k[hi] && p[lo] > p[hi]);
        if (gt == up) {
          const uint64_t tk = k[lo]; k[lo] = k[hi]; k[hi] = tk;
          const uint32_t tv = v[lo]; v[lo] = v[hi]; v[hi] = tv;
          const uint16_t tp = p[lo]; p[lo] = p[hi]; p[hi] = tp;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    kout[i] = k[i];
    vout[i] = v[i];
  }
}

static int64_t nblocks_for(int64_t n) { return (n + kChunk - 1) / kChunk; }

int scan_u32_excl(const uint32_t* in, uint64_t* out, int64_t m, uint64_t* tmp, cudaStream_t st);
int64_t scan_tmp_words(int64_t m);

// workspace: counts u32[ndig*nb] + offsets u64[ndig*nb + 1] + scan scratch
static int64_t ws_bytes(int64_t n, int ndig) {
  const int64_t nb = nblocks_for(n) > 0 ? nblocks_for(n) : 1;
  const int64_t m = ndig * nb;
  return ((m * 4 + 255) / 256) * 256 + (m + 1) * 8 + 8 * scan_tmp_words(m);
}

static int counting_pass(const DigitSrc& D, int64_t n, int ndig, void* temp, cudaStream_t st,
                         const uint64_t*& offs_out, int& nb_out) {
  const int64_t nb = nblocks_for(n);
  uint32_t* counts = static_cast<uint32_t*>(temp);
  uint64_t* offs = reinterpret_cast<uint64_t*>(static_cast<char*>(temp) + ((nb * ndig * 4 + 255) / 256) * 256);
  uint64_t* tmp = offs + nb * ndig + 1;
  hist_kernel<<<(int)nb, kBlock, 0, st>>>(D, n, ndig, counts, (int)nb);
  SCX_CHECK_LAUNCH("hist_kernel");
  int rc = scan_u32_excl(counts, offs, nb * ndig, tmp, st);
  if (rc) return rc;
  offs_out = offs;
  nb_out = (int)nb;
  return SCX_OK;
}

}  // namespace scx

using namespace scx;

extern "C" int64_t scx_sort_workspace(int64_t n) { return ws_bytes(n, kDigits); }

extern "C" int scx_sort_pairs(const uint64_t* kin, const uint32_t* vin, uint64_t* kout,
                              uint32_t* vout, uint64_t* ktmp, uint32_t* vtmp, int64_t n,
                              int n_bits, void* temp, void* stream) {
  if (n == 0) return SCX_OK;
  if (!kin || !vin || !kout || !vout || n_bits < 0 || n_bits > 64 ||
      (n_bits > 8 && (!ktmp || !vtmp)) || !temp) {
    set_error("sort_pairs: bad arguments");
    return SCX_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int passes = (n_bits + 7) / 8;
  if (passes > 1 && n <= kSmallSort) {
    small_sort_kernel<<<1, 1024, 0, st>>>(kin, vin, kout, vout, (int)n);
    SCX_CHECK_LAUNCH("small_sort_kernel");
    return SCX_OK;
  }
  if (passes == 0) {
    copy_pairs_kernel<<<grid_for(n, 256, 2368), 256, 0, st>>>(kin, vin, kout, vout, n);
    SCX_CHECK_LAUNCH("copy_pairs_kernel");
    return SCX_OK;
  }
  const uint64_t* ks = kin;
  const uint32_t* vs = vin;
  for (int p = 0; p < passes; ++p) {
    // land the final pass in *_out
    const bool to_out = ((passes - 1 - p) % 2) == 0;
    uint64_t* kd = to_out ? kout : ktmp;
    uint32_t* vd = to_out ? vout : vtmp;
    DigitSrc D;
    memset(&D, 0, sizeof(D));
    D.keys = ks;
    D.shift = 8 * p;
    const uint64_t* offs;
    int nb;
    int rc = counting_pass(D, n, kDigits, temp, st, offs, nb);
    if (rc) return rc;
    sort_scatter_kernel<<<nb, kBlock, 0, st>>>(D, n, offs, nb, ks, vs, kd, vd);
    SCX_CHECK_LAUNCH("sort_scatter_kernel");
    ks = kd;
    vs = vd;
  }
  return SCX_OK;
}

extern "C" int scx_hash_keys(const scx_column* keys, int n_keys, int64_t n, uint64_t* out,
                             void* stream) {
  if (n == 0) return SCX_OK;
  if (!keys || n_keys < 1 || n_keys > SCX_MAX_KEYS || !out) {
    set_error("hash_keys: bad arguments");
    return SCX_EINVAL;
  }
  PartKeys K;
  memset(&K, 0, sizeof(K));
  K.n = n_keys;
  for (int i = 0; i < n_keys; ++i) K.k[i] = keys[i];
  hash_keys_kernel<<<grid_for(n, 256, 2368), 256, 0, (cudaStream_t)stream>>>(K, n, out);
  SCX_CHECK_LAUNCH("hash_keys_kernel");
  return SCX_OK;
}

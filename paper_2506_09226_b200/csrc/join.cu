// join.cu -- multi-match inner join expansion (relops.py:59-94, _join_codes
// 32-56): the reference sorts the right side's dense key codes with a stable
// argsort, finds each left key's [lo, hi) run with searchsorted and repeats
// the left index over the run, so the output is in LEFT row order and, per
// left row, in RIGHT row order.
//
// Here the right keys are packed u64 words sorted stably by the radix sort
// (scx_sort_pairs: equal keys keep right row order), then
//   1. scx_join_match_ranges : per left row, lower/upper bound in the sorted
//      right keys (binary search; the sorted keys are read through L2),
//   2. an exclusive scan of the per-row match counts (scan_u32_excl),
//   3. scx_join_expand       : one thread per OUTPUT pair -- a binary search
//      over the scanned offsets finds its left row, so heavy duplicate runs
//      are spread over many threads (no per-left-row loop imbalance).
#include "common.cuh"

namespace scx {

int scan_u32_excl(const uint32_t* in, uint64_t* out, int64_t m, uint64_t* tmp, cudaStream_t st);
int64_t scan_tmp_words(int64_t m);

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* a, int64_t m, uint64_t k) {
  int64_t lo = 0, hi = m;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) < k) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int64_t upper_bound_u64(const uint64_t* a, int64_t lo, int64_t m,
                                                   uint64_t k) {
  int64_t hi = m;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) <= k) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void match_ranges_kernel(const uint64_t* __restrict__ lkeys, int64_t n,
                                    const uint64_t* __restrict__ rsorted, int64_t m,
                                    uint32_t* __restrict__ start, uint32_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = lkeys[i];
    const int64_t a = lower_bound_u64(rsorted, m, k);
    int64_t b = a;
    if (a < m && __ldg(rsorted + a) == k) b = upper_bound_u64(rsorted, a + 1, m, k);
    start[i] = (uint32_t)a;
    cnt[i] = (uint32_t)(b - a);
  }
}

// pair k: left row i = the last row with offs[i] <= k (offs exclusive, n+1
// entries, offs[n] = total), right row = rperm[start[i] + k - offs[i]]
__global__ void expand_kernel(const uint32_t* __restrict__ start, const uint64_t* __restrict__ offs,
                              int64_t n, const uint32_t* __restrict__ rperm, int64_t total,
                              uint32_t* __restrict__ out_l, uint32_t* __restrict__ out_r) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;             // first i with offs[i] > k, minus one
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (__ldg(offs + mid) <= (uint64_t)k) lo = mid + 1; else hi = mid;
    }
    const int64_t i = lo - 1;
    out_l[k] = (uint32_t)i;
    out_r[k] = __ldg(rperm + __ldg(start + i) + (k - (int64_t)__ldg(offs + i)));
  }
}

static int grid_for(int64_t n) {
  int64_t g = (n + kBlock - 1) / kBlock;
  if (g > 148 * 32) g = 148 * 32;       // grid-stride beyond 32 CTAs per SM
  return (int)(g < 1 ? 1 : g);
}

}  // namespace scx

using namespace scx;

extern "C" int64_t scx_join_workspace(int64_t n) {
  // start u32[n] + cnt u32[n] (16-byte padded) + offs u64[n+1] + scan scratch
  const int64_t a = ((n * 4 + 15) / 16) * 16;
  return 2 * a + (n + 1) * 8 + 8 * scan_tmp_words(n) + 16;
}

extern "C" int scx_join_match(const uint64_t* lkeys_dev, int64_t n, const uint64_t* rsorted_dev,
                              int64_t m, void* ws_dev, uint64_t* total_dev, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n < 0 || m < 0 || m > 0xFFFFFFFFll) {
    set_error("scx_join_match: bad sizes n=%lld m=%lld", (long long)n, (long long)m);
    return SCX_EINVAL;
  }
  char* ws = static_cast<char*>(ws_dev);
  const int64_t a = ((n * 4 + 15) / 16) * 16;
  uint32_t* start = reinterpret_cast<uint32_t*>(ws);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(ws + a);
  uint64_t* offs = reinterpret_cast<uint64_t*>(ws + 2 * a);
  uint64_t* tmp = offs + (n + 1);
  if (n > 0) {
    match_ranges_kernel<<<grid_for(n), kBlock, 0, st>>>(lkeys_dev, n, rsorted_dev, m, start, cnt);
    SCX_CHECK_LAUNCH("match_ranges_kernel");
  }
  int rc = scan_u32_excl(cnt, offs, n, tmp, st);
  if (rc != SCX_OK) return rc;
  SCX_CUDA(cudaMemcpyAsync(total_dev, offs + n, 8, cudaMemcpyDeviceToDevice, st));
  return SCX_OK;
}

extern "C" int scx_join_expand(const void* ws_dev, int64_t n, const uint32_t* rperm_dev,
                               int64_t total, uint32_t* out_l_dev, uint32_t* out_r_dev,
                               void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (total <= 0) return SCX_OK;
  if (total > 0xFFFFFFFFll) {
    set_error("scx_join_expand: %lld output pairs exceed u32 row indices", (long long)total);
    return SCX_EUNSUPPORTED;
  }
  const char* ws = static_cast<const char*>(ws_dev);
  const int64_t a = ((n * 4 + 15) / 16) * 16;
  const uint32_t* start = reinterpret_cast<const uint32_t*>(ws);
  const uint64_t* offs = reinterpret_cast<const uint64_t*>(ws + 2 * a);
  expand_kernel<<<grid_for(total), kBlock, 0, st>>>(start, offs, n, rperm_dev, total, out_l_dev,
                                                    out_r_dev);
  SCX_CHECK_LAUNCH("expand_kernel");
  return SCX_OK;
}

// codes.cu -- dictionary code remapping for broadcast_table's dictionary
// reconciliation (exchange.py:177-192, 224-228: when workers' dictionaries
// differ, the union is built in rank order, first seen wins, and every
// worker's codes are rewritten through its remap before the exchange).
#include "common.cuh"

namespace scx {

__global__ void remap_codes_kernel(scx_column in, int64_t n, const int32_t* __restrict__ lut,
                                   int32_t lut_n, scx_column out, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = load_i64(reinterpret_cast<const void*>(in.ptr), in.dtype, i);
    if (c < 0 || c >= lut_n) {
      atomicOr(bad, 1);
      continue;
    }
    store_i64(reinterpret_cast<void*>(out.ptr), out.dtype, i, __ldg(lut + c));
  }
}

}  // namespace scx

using namespace scx;

extern "C" int scx_remap_codes(scx_column in, int64_t n, const int32_t* lut_dev, int32_t lut_n,
                               scx_column out, int* bad_dev, void* stream) {
  if (n < 0 || lut_n < 0 || (n > 0 && (!lut_dev || !bad_dev)) || dtype_size(in.dtype) == 0 ||
      dtype_size(out.dtype) == 0) {
    set_error("scx_remap_codes: bad arguments");
    return SCX_EINVAL;
  }
  if (n == 0) return SCX_OK;
  remap_codes_kernel<<<grid_for(n, 256, 148 * 16), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      in, n, lut_dev, lut_n, out, bad_dev);
  SCX_CHECK_LAUNCH("remap_codes_kernel");
  return SCX_OK;
}

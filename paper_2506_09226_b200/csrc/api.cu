// api.cu -- error plumbing and library info for the libscx C-ABI.
#include <stdarg.h>
#include <stdio.h>
#include "common.cuh"

namespace scx {

static thread_local char g_err[512] = "";
// process-wide count of kernels launched through this library (benchmark
// evidence for "gpu_launches"; an atomic counter, not state any op reads)
static unsigned long long g_launches = 0;

void count_launch() { __atomic_add_fetch(&g_launches, 1ull, __ATOMIC_RELAXED); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  return SCX_ECUDA;
}

}  // namespace scx

extern "C" const char* scx_last_error(void) { return scx::g_err; }

extern "C" int scx_abi_version(void) { return SCX_ABI_VERSION; }

extern "C" uint64_t scx_launch_count(void) {
  return __atomic_load_n(&scx::g_launches, __ATOMIC_RELAXED);
}

extern "C" int64_t scx_sizeof(int which) {
  switch (which) {
    case 0: return sizeof(scx_pipeline);
    case 1: return sizeof(scx_probe);
    case 2: return sizeof(scx_sink);
    case 3: return sizeof(scx_measure);
    case 4: return sizeof(scx_atom);
    case 5: return sizeof(scx_keyspec);
    case 6: return sizeof(scx_lookup);
    case 7: return sizeof(scx_column);
    default: return -1;
  }
}

extern "C" int scx_device_info(int device, int* sm_count, int* smem_optin) {
  if (sm_count) SCX_CUDA(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, device));
  if (smem_optin)
    SCX_CUDA(cudaDeviceGetAttribute(smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
  return SCX_OK;
}

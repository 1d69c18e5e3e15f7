// common.cuh -- shared device helpers for libscx (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/scx.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libscx is written for sm_100a (B200); compile with -gencode arch=compute_100a,code=sm_100a"
#endif

namespace scx {

constexpr int kBlock = 256;            // threads per CTA for the scan kernels
constexpr int kWarps = kBlock / 32;
constexpr uint64_t kFib = 0x9E3779B97F4A7C15ull;   // exchange.py:27

// ---- error reporting (thread-local, scx_last_error) -----------------------
void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

#define SCX_CUDA(call)                                        \
  do {                                                        \
    cudaError_t _e = (call);                                  \
    if (_e != cudaSuccess) return ::scx::cuda_fail(_e, #call); \
  } while (0)

void count_launch();

#define SCX_CHECK_LAUNCH(what)                                 \
  do {                                                         \
    ::scx::count_launch();                                     \
    cudaError_t _e = cudaGetLastError();                       \
    if (_e != cudaSuccess) return ::scx::cuda_fail(_e, what);  \
  } while (0)

inline int dtype_size(int dt) {
  switch (dt) {
    case SCX_I8: case SCX_U8: return 1;
    case SCX_I16: case SCX_U16: return 2;
    case SCX_I32: case SCX_U32: return 4;
    case SCX_I64: case SCX_F64: return 8;
    default: return 0;
  }
}
__host__ __device__ inline int dtype_size_d(int dt) {
  return (dt == SCX_I8 || dt == SCX_U8) ? 1
       : (dt == SCX_I16 || dt == SCX_U16) ? 2
       : (dt == SCX_I32 || dt == SCX_U32) ? 4 : 8;
}

// ---- typed loads/stores; every integer-backed value widens to int64 ----
__device__ __forceinline__ int64_t load_i64(const void* p, int dt, int64_t i) {
  switch (dt) {
    case SCX_I8:  return static_cast<const int8_t*>(p)[i];
    case SCX_I16: return static_cast<const int16_t*>(p)[i];
    case SCX_I32: return static_cast<const int32_t*>(p)[i];
    case SCX_U8:  return static_cast<const uint8_t*>(p)[i];
    case SCX_U16: return static_cast<const uint16_t*>(p)[i];
    case SCX_U32: return static_cast<const uint32_t*>(p)[i];
    default:      return static_cast<const int64_t*>(p)[i];   // I64 (F64 bits)
  }
}

__device__ __forceinline__ void store_i64(void* p, int dt, int64_t i, int64_t v) {
  switch (dt) {
    case SCX_I8:  static_cast<int8_t*>(p)[i] = (int8_t)v; break;
    case SCX_I16: static_cast<int16_t*>(p)[i] = (int16_t)v; break;
    case SCX_I32: static_cast<int32_t*>(p)[i] = (int32_t)v; break;
    case SCX_U8:  static_cast<uint8_t*>(p)[i] = (uint8_t)v; break;
    case SCX_U16: static_cast<uint16_t*>(p)[i] = (uint16_t)v; break;
    case SCX_U32: static_cast<uint32_t*>(p)[i] = (uint32_t)v; break;
    default:      static_cast<int64_t*>(p)[i] = v; break;
  }
}

// ---- hashing -----------------------------------------------------------
// Lookup/group tables: murmur3 fmix64 (independent of the partition hash so
// that a partition's keys still spread over the whole table).
__device__ __forceinline__ uint64_t mix64(uint64_t k) {
  k ^= k >> 33; k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33; k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

// Partition hash step (exchange.py:47-48): acc = (acc ^ (u64(v) * F)) * F
__device__ __forceinline__ uint64_t fib_step(uint64_t acc, int64_t v) {
  return (acc ^ (static_cast<uint64_t>(v) * kFib)) * kFib;
}

// ---- memory-ordering helpers for decoupled look-back ---------------------
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}

// ---- TMA bulk copy (cp.async.bulk) + mbarrier ------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {}
}
// global -> shared bulk copy, completion signalled on `bar` (complete_tx)
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :: "r"(smem_u32(dst_smem)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// ---- 128-bit accumulation into {u64 lo, i64 hi} with two atomics ----------
__device__ __forceinline__ void atomic_add_i128(int64_t* lohi, int64_t v) {
  if (v == 0) return;
  unsigned long long* lo = reinterpret_cast<unsigned long long*>(lohi);
  unsigned long long old = atomicAdd(lo, static_cast<unsigned long long>(v));
  unsigned long long sum = old + static_cast<unsigned long long>(v);
  long long hi_add = (v < 0 ? -1ll : 0ll) + (sum < old ? 1ll : 0ll);
  if (hi_add) atomicAdd(reinterpret_cast<unsigned long long*>(lohi + 1),
                        static_cast<unsigned long long>(hi_add));
}

__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int64_t warp_min_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, (int64_t)__shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int64_t warp_max_i64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, (int64_t)__shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

inline int grid_for(int64_t items, int per_block, int cap) {
  int64_t g = (items + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<int>(g);
}

}  // namespace scx

// Shared host/device helpers for libavion_b200 (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include "../../include/avion_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libavion_b200 targets sm_100a only"
#endif

namespace avb {

// thread-local last-error text, returned by avb_last_error()
void set_error(const char* fmt, ...);

inline int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return AVB_OK;
  set_error("%s: %s", what, cudaGetErrorString(e));
  return AVB_E_CUDA;
}

// Launch status check: peek (does not clear sticky errors of other callers).
inline int launch_status(const char* what) {
  return cuda_status(cudaPeekAtLastError(), what);
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();

// Raise a kernel's dynamic shared-memory limit (and optionally allow non-portable cluster sizes) on
// the CURRENT device, once per (kernel, device).  Kernel attributes are per device, so a process
// that launches on several GPUs needs the call on each; the cache is mutex-protected.
int ensure_kernel_attrs(const void* func, int smem_bytes, const char* what, bool nonportable_cluster = false);

}  // namespace avb

#define AVB_CHECK_ARG(cond, ...)            \
  do {                                      \
    if (!(cond)) {                          \
      avb::set_error(__VA_ARGS__);          \
      return AVB_E_ARG;                     \
    }                                       \
  } while (0)

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// explicit shared-space 16-byte accesses (a pointer that went through integer alignment arithmetic
// loses its address space: plain C++ accesses become generic LD/ST, and a following
// fence.proxy.async then also needs a MEMBAR)
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr)
               : "memory");
  return v;
}

__device__ __forceinline__ int4 ld_nc_v4(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ int floordiv_i64(long long a, long long b) {
  // b > 0
  long long q = a / b;
  if ((a % b != 0) && (a < 0)) --q;
  return static_cast<int>(q);
}

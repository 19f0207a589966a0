// Library-wide C ABI plumbing: error text, version, device info.
#include "common.cuh"

#include <mutex>
#include <set>
#include <utility>
#include <string>

namespace avb {

static thread_local char g_err[1024] = {0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cached[dev] = n;
  }
  return cached[dev];
}

int ensure_kernel_attrs(const void* func, int smem_bytes, const char* what, bool nonportable_cluster) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, what);
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({func, dev})) return AVB_OK;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
  if (e == cudaSuccess && nonportable_cluster)
    e = cudaFuncSetAttribute(func, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
  if (e != cudaSuccess) return cuda_status(e, what);
  done.insert({func, dev});
  return AVB_OK;
}

}  // namespace avb

extern "C" const char* avb_last_error(void) { return avb::g_err; }

extern "C" int avb_version(void) { return 1; }

extern "C" int avb_device_sm_count(void) { return avb::sm_count(); }

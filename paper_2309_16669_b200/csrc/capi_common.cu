// Library-wide C ABI plumbing: error text, version, device info.
#include "common.cuh"

#include <mutex>
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

}  // namespace avb

extern "C" const char* avb_last_error(void) { return avb::g_err; }

extern "C" int avb_version(void) { return 1; }

extern "C" int avb_device_sm_count(void) { return avb::sm_count(); }

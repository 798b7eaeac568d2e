// Library-wide C-ABI entry points: version, last error, device cache.
#include "common.cuh"

#include <mutex>

namespace b2 {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

const DeviceInfo& device_info() {
  // one entry per device ordinal; filled lazily, never freed
  static DeviceInfo cache[64];
  static std::mutex mu;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  DeviceInfo& d = cache[dev];
  if (d.device < 0) {
    std::lock_guard<std::mutex> lock(mu);
    if (d.device < 0) {
      cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, dev);
      cudaDeviceGetAttribute(&d.coop, cudaDevAttrCooperativeLaunch, dev);
      d.device = dev;
    }
  }
  return d;
}

}  // namespace b2

extern "C" const char* b2_version(void) { return "b2ddp 0.1.0 sm_100a"; }

extern "C" const char* b2_last_error(void) { return b2::g_err; }

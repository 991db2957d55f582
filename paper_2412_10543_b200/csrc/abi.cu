// Library-level C ABI entry points: version, error reporting, device checks.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <vector>

#include "rs_common.cuh"

namespace rs {

static thread_local char g_err[1024] = "";
static std::atomic<uint64_t> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

const char* last_error() { return g_err; }

int sm_count(int device) {
  static std::mutex mu;
  static std::vector<int> cache;
  std::lock_guard<std::mutex> lock(mu);
  if (device < 0) return 0;
  if ((int)cache.size() <= device) cache.resize(device + 1, 0);
  if (!cache[device]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
    cache[device] = v;
  }
  return cache[device];
}

}  // namespace rs

extern "C" int rs_abi_version(void) { return RS_ABI_VERSION; }

extern "C" uint64_t rs_launch_count(void) { return rs::g_launches.load(std::memory_order_relaxed); }

extern "C" const char* rs_last_error(void) { return rs::last_error(); }

extern "C" int rs_device_supported(int device) {
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  // compiled for sm_100a only (arch-specific features: tcgen05 / TMEM / TMA)
  return major == 10 && minor == 0;
}

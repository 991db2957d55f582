// Shared host/device helpers for the ragsched_b200 library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "ragsched_b200.h"

namespace rs {

// Thread-local last-error message (rs_last_error).
void set_error(const char* fmt, ...);
const char* last_error();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Count of kernels this library launched (rs_launch_count).
void count_launch();

// Launch-error check used right after every <<<>>> launch.
#define RS_CHECK_LAUNCH(what)                                                     \
  do {                                                                            \
    ::rs::count_launch();                                                         \
    cudaError_t _e = cudaGetLastError();                                          \
    if (_e != cudaSuccess) {                                                      \
      ::rs::set_error("%s: %s", what, cudaGetErrorString(_e));                    \
      return RS_ERR_CUDA;                                                         \
    }                                                                             \
  } while (0)

#define RS_CHECK_CUDA(call, what)                                                 \
  do {                                                                            \
    cudaError_t _e = (call);                                                      \
    if (_e != cudaSuccess) {                                                      \
      ::rs::set_error("%s: %s", what, cudaGetErrorString(_e));                    \
      return _e == cudaErrorMemoryAllocation ? RS_ERR_OOM : RS_ERR_CUDA;          \
    }                                                                             \
  } while (0)

#define RS_REQUIRE(cond, ...)                                                     \
  do {                                                                            \
    if (!(cond)) {                                                                \
      ::rs::set_error(__VA_ARGS__);                                               \
      return RS_ERR_INVALID_ARG;                                                  \
    }                                                                             \
  } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Makes `dev` current for a scope and restores the caller's device after.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// Number of SMs of the current device (cached per device).
int sm_count(int device);

// Packed top-k key: fp32 distance bits (non-negative, so unsigned order ==
// float order) in the high word, uint32 global chunk id in the low word.
// Ascending key order == (distance asc, id asc).
constexpr uint64_t kEmptyKey = ~0ull;

}  // namespace rs

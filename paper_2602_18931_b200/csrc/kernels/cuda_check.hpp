#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <string>

#include "../host/common.hpp"

#define WS_CUDA(expr)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      throw ::wsb::CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_));      \
  } while (0)

namespace wsb {
// Makes `dev` current for a scope and restores the caller's device (the library never leaves a
// caller's thread on another GPU — split placement drives two).
class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    WS_CUDA(cudaGetDevice(&prev_));
    if (dev != prev_) WS_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev_); }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;

 private:
  int prev_ = 0;
};

// Runs fn once per device for a given mask (kernel attributes such as the dynamic shared-memory
// cap are per device: a process may drive the target and the draft model on two GPUs).
template <class F>
void once_per_device(std::atomic<std::uint32_t>& mask, F&& fn) {
  int dev = 0;
  WS_CUDA(cudaGetDevice(&dev));
  const std::uint32_t bit = 1u << (dev & 31);
  if (mask.load(std::memory_order_acquire) & bit) return;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (mask.load(std::memory_order_acquire) & bit) return;
  fn();
  mask.fetch_or(bit, std::memory_order_release);
}
}  // namespace wsb

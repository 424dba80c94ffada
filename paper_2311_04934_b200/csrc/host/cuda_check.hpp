// CUDA status checks and a scoped device buffer for the host layer: every runtime
// call on the hot path and in the store's persistence goes through CK, so a device
// failure surfaces as pcb::Error(CudaError) at the C ABI instead of a silent
// null-pointer kernel argument.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "errors.hpp"

#define CK(x)                                                                                        \
  do {                                                                                               \
    cudaError_t e_ = (x);                                                                            \
    if (e_ != cudaSuccess)                                                                           \
      throw ::pcb::Error(::pcb::ErrorCode::CudaError, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

namespace pcb {

// Device allocation freed on scope exit (exceptions included).
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t bytes) { reset(bytes); }
  ~DeviceBuffer() { release(); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;

  void reset(size_t bytes) {
    release();
    if (bytes) CK(cudaMalloc(&p_, bytes));
    bytes_ = bytes;
  }
  void* get() const { return p_; }
  size_t bytes() const { return bytes_; }
  template <typename T>
  T* as() const { return static_cast<T*>(p_); }

 private:
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    bytes_ = 0;
  }
  void* p_ = nullptr;
  size_t bytes_ = 0;
};

}  // namespace pcb

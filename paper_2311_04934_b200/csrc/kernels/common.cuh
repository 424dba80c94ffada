#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "kernels.cuh"

#define PCB_CUDA(x)                                                                             \
  do {                                                                                          \
    cudaError_t err_ = (x);                                                                     \
    if (err_ != cudaSuccess)                                                                    \
      throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(err_) + " at " + \
                               __FILE__ + ":" + std::to_string(__LINE__));                      \
  } while (0)

namespace pcb::kern {

__device__ __forceinline__ float ld_f(const float* p, int64_t i) { return p[i]; }
__device__ __forceinline__ float ld_f(const __nv_bfloat16* p, int64_t i) { return __bfloat162float(p[i]); }
__device__ __forceinline__ void st_f(float* p, int64_t i, float v) { p[i] = v; }
__device__ __forceinline__ void st_f(__nv_bfloat16* p, int64_t i, float v) { p[i] = __float2bfloat16_rn(v); }

// GELU-tanh exactly as the reference computes it (fp64, model.cpp:176-179),
// with explicit rounding intrinsics so nvcc cannot contract it differently.
__device__ __forceinline__ float gelu_ref(float xf) {
  double x = xf;
  double x3 = __dmul_rn(__dmul_rn(__dmul_rn(0.044715, x), x), x);
  double t = __dmul_rn(0.7978845608028654, __dadd_rn(x, x3));
  return (float)__dmul_rn(__dmul_rn(0.5, x), __dadd_rn(1.0, tanh(t)));
}

__device__ __forceinline__ float gelu_fast(float x) {
  float t = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  return 0.5f * x * (1.0f + tanhf(t));
}

}  // namespace pcb::kern

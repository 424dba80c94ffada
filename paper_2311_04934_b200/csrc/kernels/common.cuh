#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>

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

// ---- programmatic dependent launch (PDL) ----
// Every kernel of the forward chain is launched with programmatic stream
// serialization: it may start (barrier init, TMEM alloc, weight prefetch) while
// its predecessor drains, and calls pdl_wait() before touching memory the
// predecessor produces (or that an earlier kernel still reads).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("PCB_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

// kernel class of the launch in flight (PCB_PDL_MASK bit i enables PDL for class i)
enum PdlCls : int { PDL_OTHER = 0, PDL_GEMM = 1, PDL_ATTN = 2, PDL_LN = 3, PDL_EMBED = 4, PDL_ARGMAX = 5, PDL_ASM = 6 };
inline thread_local int g_pdl_cls = PDL_OTHER;
struct PdlClass {
  int prev;
  explicit PdlClass(int c) : prev(g_pdl_cls) { g_pdl_cls = c; }
  ~PdlClass() { g_pdl_cls = prev; }
};
// Default: every class except attention.  A PDL-launched attention kernel was seen to
// stall its first softmax hand-off under the early-launch overlap with the QKV GEMM
// (reproduced with attention as the only PDL class), so it
// is launched with full stream serialisation until that is understood.
inline int pdl_mask() {
  static const int m = [] {
    const char* v = std::getenv("PCB_PDL_MASK");
    return v ? std::atoi(v) : (0x7f & ~(1 << PDL_ATTN));
  }();
  return m;
}

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cluster_z,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[na].val.programmaticStreamSerializationAllowed = (pdl_enabled() && ((pdl_mask() >> g_pdl_cls) & 1)) ? 1 : 0;
  ++na;
  if (cluster_z > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = 1;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = cluster_z;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  PCB_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

__device__ __forceinline__ float gelu_fast(float x) {
  float t = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  return 0.5f * x * (1.0f + tanhf(t));
}

}  // namespace pcb::kern

// K/V streaming bandwidth of the chain's attention phase access pattern, without the math.
// One persistent launch streams L layers' K/V ([L * rows][4096] bf16, the store's row-major
// layout: per 64-key block two 64x64 TMA boxes of K and two of V, 64 rows x 256 B of a head's
// slice, rows 8 KB apart) through a ring of STAGES x 32 KB per CTA.  The (head, block) space
// of a layer is cut into equal contiguous ranges over the grid (128 CTAs = 32 heads x 4 splits,
// as the chain's attention phase; 148 = every SM).  No barrier between layers: an upper bound.
// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/probe/kvstream tools/probe/kvstream.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0, 1, 0, p;\n}"
                 : "=r"(ok)
                 : "r"(su32(b)), "r"(par)
                 : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* b, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(su32(b)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(su32(b))
               : "memory");
}

template <int STAGES>
__global__ void __launch_bounds__(64, 1) kstream(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
                                                int rows, int layers) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * 32768);
  uint64_t* empty = full + STAGES;
  const int nblk = (rows + 63) / 64, T = 32 * nblk, C = gridDim.x;
  const int u0 = static_cast<int>(static_cast<long long>(T) * blockIdx.x / C);
  const int u1 = static_cast<int>(static_cast<long long>(T) * (blockIdx.x + 1) / C);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nb = (u1 - u0) * layers;
  if (threadIdx.x == 0) {
    for (int it = 0; it < nb; ++it) {
      const int s = it % STAGES;
      wait(&empty[s], ((it / STAGES) & 1) ^ 1);
      expect_tx(&full[s], 32768);
      uint8_t* st = sm + s * 32768;
      const int l = it / (u1 - u0), u = u0 + it % (u1 - u0);
      const int h = u / nblk, b = u % nblk;
      for (int a = 0; a < 2; ++a) {
        tma2d(st + a * 8192, &tk, &full[s], h * 128 + a * 64, l * rows + b * 64);
        tma2d(st + 16384 + a * 8192, &tv, &full[s], h * 128 + a * 64, l * rows + b * 64);
      }
    }
  } else if (threadIdx.x == 32) {
    for (int it = 0; it < nb; ++it) {
      const int s = it % STAGES;
      wait(&full[s], (it / STAGES) & 1);
      arrive(&empty[s]);
    }
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int ST>
float run(const CUtensorMap& tk, const CUtensorMap& tv, int rows, int layers, int ctas) {
  const int smem = ST * 32768 + 1024;
  cudaFuncSetAttribute(kstream<ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kstream<ST><<<ctas, 64, smem>>>(tk, tv, rows, layers);
  cudaEventRecord(e0);
  kstream<ST><<<ctas, 64, smem>>>(tk, tv, rows, layers);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1000.f / layers;
}

int main() {
  const int d = 4096;
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  for (int rows : {4160, 16512}) {
    const int layers = rows == 4160 ? 32 : 8;  // 2.2 GB of K/V per launch (> L2)
    const size_t n = static_cast<size_t>(rows) * layers * d;
    __nv_bfloat16* buf;
    cudaMalloc(&buf, 2 * n * sizeof(__nv_bfloat16));
    cudaMemset(buf, 0, 2 * n * sizeof(__nv_bfloat16));
    auto mk = [&](const void* p) {
      CUtensorMap m;
      cuuint64_t dims[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(rows) * layers};
      cuuint64_t strides[1] = {static_cast<cuuint64_t>(d) * 2};
      cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
      enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      return m;
    };
    const CUtensorMap tk = mk(buf), tv = mk(buf + n);
    const double bytes = 2.0 * rows * d * 2;  // per layer
    for (int ctas : {128, 132, 148})
      for (int st : {4, 5, 6}) {
        const float us = st == 4 ? run<4>(tk, tv, rows, layers, ctas)
                                 : st == 5 ? run<5>(tk, tv, rows, layers, ctas) : run<6>(tk, tv, rows, layers, ctas);
        printf("rows %5d ctas %3d stages %d: %7.2f us/layer  %6.0f GB/s\n", rows, ctas, st, us, bytes / us / 1e3);
      }
    cudaFree(buf);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

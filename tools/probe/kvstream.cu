// K/V streaming bandwidth of the chain's attention phase access pattern, without the math.
// 128 CTAs = 32 heads x 4 key splits, each streaming its keys' K and V in 64-row blocks
// through a ring of STAGES x 32 KB:
//   rowmajor   K/V [rows][4096] bf16, per block two 64x64 TMA boxes of K and two of V
//              (64 rows x 256 B of the head's slice, rows 8 KB apart) -- the store's layout
//   headmajor  K/V [32 heads][rows][128]: a block is 16 KB contiguous per tensor, one bulk copy
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

template <int STAGES, bool HM>
__global__ void __launch_bounds__(64, 1) kstream(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
                                                const __nv_bfloat16* K, const __nv_bfloat16* V, int rows, int splits) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * 32768);
  uint64_t* empty = full + STAGES;
  const int h = blockIdx.x / splits, sp = blockIdx.x % splits;
  const int nblk = (rows + 63) / 64;
  const int b0 = nblk * sp / splits, nb = nblk * (sp + 1) / splits - b0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int it = 0; it < nb; ++it) {
      const int s = it % STAGES;
      wait(&empty[s], ((it / STAGES) & 1) ^ 1);
      expect_tx(&full[s], 32768);
      uint8_t* st = sm + s * 32768;
      const int b = b0 + it;
      if (HM) {
        const size_t off = (static_cast<size_t>(h) * rows + static_cast<size_t>(b) * 64) * 128;
        bulk(st, K + off, 16384, &full[s]);
        bulk(st + 16384, V + off, 16384, &full[s]);
      } else {
        for (int a = 0; a < 2; ++a) {
          tma2d(st + a * 8192, &tk, &full[s], h * 128 + a * 64, b * 64);
          tma2d(st + 16384 + a * 8192, &tv, &full[s], h * 128 + a * 64, b * 64);
        }
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

template <int ST, bool HM>
float run(const std::vector<CUtensorMap>& tk, const std::vector<CUtensorMap>& tv, const std::vector<const __nv_bfloat16*>& K,
          const std::vector<const __nv_bfloat16*>& V, int rows, int splits) {
  const int smem = ST * 32768 + 1024;
  cudaFuncSetAttribute(kstream<ST, HM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int L = static_cast<int>(K.size());
  for (int l = 0; l < L; ++l) kstream<ST, HM><<<32 * splits, 64, smem>>>(tk[l], tv[l], K[l], V[l], rows, splits);
  cudaEventRecord(e0);
  const int reps = 4;
  for (int r = 0; r < reps; ++r)  // a different layer every launch: the working set (12 x 68 MB) exceeds L2
    for (int l = 0; l < L; ++l) kstream<ST, HM><<<32 * splits, 64, smem>>>(tk[l], tv[l], K[l], V[l], rows, splits);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1000.f / (reps * L);
}

int main() {
  const int rows = 4160, d = 4096;
  // 12 K/V layer pairs (> L2) cycled so every launch reads from HBM
  const int L = 12;
  const size_t n = static_cast<size_t>(rows) * d;
  __nv_bfloat16* buf;
  cudaMalloc(&buf, 2 * L * n * sizeof(__nv_bfloat16));
  cudaMemset(buf, 0, 2 * L * n * sizeof(__nv_bfloat16));
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  auto mk = [&](const void* p) {
    CUtensorMap m;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(d) * 2};
    cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims, strides, box, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return m;
  };
  const double bytes = 2.0 * n * 2;
  std::vector<CUtensorMap> tk, tv;
  std::vector<const __nv_bfloat16*> Ks, Vs;
  for (int l = 0; l < L; ++l) {
    Ks.push_back(buf + 2 * l * n);
    Vs.push_back(buf + 2 * l * n + n);
    tk.push_back(mk(Ks.back()));
    tv.push_back(mk(Vs.back()));
  }
  for (int splits : {4, 8}) {
    for (int layout = 0; layout < 2; ++layout) {
      for (int st : {3, 4, 6}) {
        float us;
        if (layout == 0)
          us = st == 3 ? run<3, false>(tk, tv, Ks, Vs, rows, splits)
                       : st == 4 ? run<4, false>(tk, tv, Ks, Vs, rows, splits) : run<6, false>(tk, tv, Ks, Vs, rows, splits);
        else
          us = st == 3 ? run<3, true>(tk, tv, Ks, Vs, rows, splits)
                       : st == 4 ? run<4, true>(tk, tv, Ks, Vs, rows, splits) : run<6, true>(tk, tv, Ks, Vs, rows, splits);
        printf("splits %d %-9s stages %d: %7.1f us  %6.0f GB/s\n", splits, layout ? "headmajor" : "rowmajor", st, us,
               bytes / us / 1e3);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}

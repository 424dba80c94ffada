// Probe: tcgen05.ld cost as the chain's softmax / attention tail sees it.  One CTA per SM,
// W warps (4: one per SM sub-partition, as the chain's epilogue; 8: two per sub-partition),
// each loading its TMEM lane quadrant:
//   serial   ld 32x32b.x16 ; wait::ld ; consume      (latency per round trip)
//   pair     two x16 in flight per wait               (what the chain does)
//   quad     four x16 in flight per wait
//   x64      one 32x32b.x64 per wait
// Cycles per round trip (clock64, median warp) and the TMEM read rate implied per SM.
// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/probe/tmemld tools/probe/tmemld.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int MODE>
__global__ void k_probe(unsigned long long* out, float* sink, int iters) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tslot + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * 64;
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const uint32_t a = tm + (i & 3) * 64 % 256;
    uint32_t r[64];
    if (MODE == 0) {
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                   : "r"(a));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int x = 0; x < 16; ++x) acc += __uint_as_float(r[x]);
    } else if (MODE == 1 || MODE == 2) {
      constexpr int N = MODE == 1 ? 2 : 4;
#pragma unroll
      for (int k = 0; k < N; ++k)
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[16 * k + 0]), "=r"(r[16 * k + 1]), "=r"(r[16 * k + 2]), "=r"(r[16 * k + 3]), "=r"(r[16 * k + 4]),
              "=r"(r[16 * k + 5]), "=r"(r[16 * k + 6]), "=r"(r[16 * k + 7]), "=r"(r[16 * k + 8]), "=r"(r[16 * k + 9]),
              "=r"(r[16 * k + 10]), "=r"(r[16 * k + 11]), "=r"(r[16 * k + 12]), "=r"(r[16 * k + 13]),
              "=r"(r[16 * k + 14]), "=r"(r[16 * k + 15])
            : "r"(a + 16 * k));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int x = 0; x < 16 * N; ++x) acc += __uint_as_float(r[x]);
    } else {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
          "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,"
          "%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
            "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
            "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
            "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]),
            "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]),
            "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),
            "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]),
            "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
          : "r"(a));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int x = 0; x < 64; ++x) acc += __uint_as_float(r[x]);
    }
  }
  const long long t1 = clock64();
  if (lane == 0) out[blockIdx.x * 32 + warp] = t1 - t0;
  if (acc == 1.2345f) sink[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
}

// MUFU.EX2 issue cost: 32 independent ex2 per iteration per thread
__global__ void k_ex2(unsigned long long* out, float* sink, int iters) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float v[32];
#pragma unroll
  for (int x = 0; x < 32; ++x) v[x] = -0.001f * (x + threadIdx.x);
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int x = 0; x < 32; ++x) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[x]));
  const long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int x = 0; x < 32; ++x) acc += v[x];
  if (lane == 0) out[blockIdx.x * 32 + warp] = t1 - t0;
  if (acc == 1.2345f) sink[threadIdx.x] = acc;
}

int main() {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 148 * 32 * 8);
  cudaMalloc(&sink, 1024 * 4);
  const int iters = 4096;
  const char* names[4] = {"serial x16", "pair x16", "quad x16", "x64"};
  const int bytes_per_iter[4] = {16 * 4 * 32, 32 * 4 * 32, 64 * 4 * 32, 64 * 4 * 32};  // per warp
  for (int warps : {4, 8})
    for (int mode = 0; mode < 4; ++mode) {
      auto run = [&] {
        switch (mode) {
          case 0: k_probe<0><<<148, 32 * warps>>>(d, sink, iters); break;
          case 1: k_probe<1><<<148, 32 * warps>>>(d, sink, iters); break;
          case 2: k_probe<2><<<148, 32 * warps>>>(d, sink, iters); break;
          default: k_probe<3><<<148, 32 * warps>>>(d, sink, iters);
        }
      };
      run();
      run();
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      std::vector<unsigned long long> h(148 * 32);
      cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
      std::vector<double> c;
      for (int b = 0; b < 148; ++b)
        for (int w = 0; w < warps; ++w) c.push_back(static_cast<double>(h[b * 32 + w]) / iters);
      std::sort(c.begin(), c.end());
      const double med = c[c.size() / 2];
      printf("warps %d %-10s: %7.1f cycles per wait (median warp)  -> %6.1f B/cycle per SM\n", warps, names[mode], med,
             bytes_per_iter[mode] * warps / med);
    }
  for (int warps : {4, 8}) {
    k_ex2<<<148, 32 * warps>>>(d, sink, 1024);
    k_ex2<<<148, 32 * warps>>>(d, sink, 1024);
    cudaDeviceSynchronize();
    std::vector<unsigned long long> h(148 * 32);
    cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
    std::vector<double> c;
    for (int b = 0; b < 148; ++b)
      for (int w = 0; w < warps; ++w) c.push_back(static_cast<double>(h[b * 32 + w]) / 1024 / 32);
    std::sort(c.begin(), c.end());
    printf("warps %d ex2: %.2f cycles per warp instruction (median warp)\n", warps, c[c.size() / 2]);
  }
  return 0;
}

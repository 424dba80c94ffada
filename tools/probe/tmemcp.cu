// Probe: a packed weight tile (128 rows x 64 bf16, SW128 K-major smem image) copied to TMEM
// with tcgen05.cp and used as the A operand of tcgen05.mma (TS form) must give exactly the
// SS-form result.  Prints max |D_ts - D_ss| and max |D_ss - host fp32|.
// Build: nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/probe/tmemcp tools/probe/tmemcp.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t kdesc(uint32_t a) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((a >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}

__global__ void k_probe(const uint8_t* gA, const uint8_t* gB, float* out_ss, float* out_ts, int mode) {
  __shared__ __align__(1024) uint8_t sA[16384];
  __shared__ __align__(1024) uint8_t sB[8192];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x;
  for (int i = t; i < 16384 / 16; i += 128) reinterpret_cast<uint4*>(sA)[i] = reinterpret_cast<const uint4*>(gA)[i];
  for (int i = t; i < 8192 / 16; i += 128) reinterpret_cast<uint4*>(sB)[i] = reinterpret_cast<const uint4*>(gB)[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (t < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tslot;
  const uint32_t D1 = tm, D2 = tm + 64, TA = tm + 128;
  if (t == 0) {
    const uint32_t a = su32(sA), b = su32(sB);
    constexpr uint32_t id = idesc(128, 64);
    for (int k = 0; k < 4; ++k)
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(D1),
                   "l"(kdesc(a + 32 * k)), "l"(kdesc(b + 32 * k)), "r"(id), "r"(k > 0 ? 1u : 0u));
    for (int k = 0; k < 4; ++k) {
      if (mode == 0)
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(TA + 8 * k), "l"(kdesc(a + 32 * k)));
      else  // two 128x128b halves per K-step
        for (int hh = 0; hh < 2; ++hh)
          asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(TA + 8 * k + 4 * hh), "l"(kdesc(a + 32 * k + 16 * hh)));
    }
    for (int k = 0; k < 4; ++k)
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(D2),
                   "r"(TA + 8 * k), "l"(kdesc(b + 32 * k)), "r"(id), "r"(k > 0 ? 1u : 0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.b32 %0, 1, 0, p;\n}"
                   : "=r"(ok) : "r"(su32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t lane_off = static_cast<uint32_t>((t >> 5) * 32) << 16;
  for (int which = 0; which < 2; ++which)
    for (int c = 0; c < 64; c += 8) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"((which ? D2 : D1) + lane_off + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      float* o = which ? out_ts : out_ss;
      for (int x = 0; x < 8; ++x) o[t * 64 + c + x] = __uint_as_float(r[x]);
    }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

// SW128 K-major image of a [rows][64] bf16 tile: row r at r * 128 B, 16-byte chunk c at (c ^ (r & 7))
static void pack(const std::vector<float>& m, int rows, std::vector<uint8_t>& out) {
  out.assign(rows * 128, 0);
  for (int r = 0; r < rows; ++r)
    for (int k = 0; k < 64; ++k) {
      const __nv_bfloat16 v = __float2bfloat16(m[r * 64 + k]);
      const int chunk = k / 8, within = k % 8;
      std::memcpy(&out[r * 128 + ((chunk ^ (r & 7)) * 16) + within * 2], &v, 2);
    }
}

int main() {
  std::vector<float> A(128 * 64), B(64 * 64);
  uint32_t s = 12345;
  auto rnd = [&] {
    s = s * 1664525u + 1013904223u;
    return ((s >> 8) & 0xFFFF) / 32768.f - 1.f;
  };
  for (auto& x : A) x = __bfloat162float(__float2bfloat16(rnd()));
  for (auto& x : B) x = __bfloat162float(__float2bfloat16(rnd()));
  std::vector<uint8_t> pA, pB;
  pack(A, 128, pA);
  pack(B, 64, pB);
  uint8_t *dA, *dB;
  float *dss, *dts;
  cudaMalloc(&dA, pA.size());
  cudaMalloc(&dB, pB.size());
  cudaMalloc(&dss, 128 * 64 * 4);
  cudaMalloc(&dts, 128 * 64 * 4);
  cudaMemcpy(dA, pA.data(), pA.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, pB.data(), pB.size(), cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dts, 0, 128 * 64 * 4);
    k_probe<<<1, 128>>>(dA, dB, dss, dts, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> ss(128 * 64), ts(128 * 64);
    cudaMemcpy(ss.data(), dss, ss.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(ts.data(), dts, ts.size() * 4, cudaMemcpyDeviceToHost);
    double d_ts = 0, d_ref = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 64; ++n) {
        double ref = 0;
        for (int k = 0; k < 64; ++k) ref += static_cast<double>(A[m * 64 + k]) * B[n * 64 + k];
        d_ref = std::fmax(d_ref, std::fabs(ss[m * 64 + n] - ref));
        d_ts = std::fmax(d_ts, std::fabs(ts[m * 64 + n] - ss[m * 64 + n]));
      }
    printf("mode %s: max|ts - ss| = %.3g   max|ss - host| = %.3g   ss[0]=%f ts[0]=%f\n",
           mode ? "128x128b" : "128x256b", d_ts, d_ref, ss[0], ts[0]);
  }
  return 0;
}

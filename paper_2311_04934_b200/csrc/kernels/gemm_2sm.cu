// tcgen05 CTA-pair GEMM for the tensor-bound shapes (module precompute, full prefill,
// micro-batched suffixes: M >= 256 tokens): C[m][n] = sum_k X[m][k] W[n][k], fused
// epilogue as in gemm_tc.cu.
//
// Why a second kernel: the single-CTA 128 x 256 tile streams 48 KB of operands from L2
// per 512 MMA cycles per SM -- more than the L2 -> SM path delivers chip-wide, which
// caps it near half of the tensor peak (tools/kbench.py: 0.51-0.57 at M = 4160, 0.3-0.4
// at M = 256-512).  Here two CTAs of a cluster (the two SMs of a TPC) run one
// `tcgen05.mma.cta_group::2` 256 x 256 x 16 MMA: each CTA stages ITS 128 weight rows
// (A) and HALF of the 256-token tile (B), 32 KB per 64-deep k-block, and keeps its own
// 128 x 256 fp32 accumulator in TMEM -- 1.5x less operand traffic per FLOP.
//
//   warp 0     TMA producer (both CTAs): packed weight tile + token half-tile per stage,
//              both completing on the LEADER CTA's full barrier (cta_group::2 TMA)
//   warp 1     TMEM allocator (both, cta_group::2); MMA issuer (leader only): waits its
//              full barrier, issues the pair MMA, commits (multicast to both CTAs) the
//              stage-empty and accumulator-full barriers
//   warps 2-5  epilogue (both): TMEM -> registers -> fused op for this CTA's 128
//              weight rows x 256 tokens; then one arrival on the leader's
//              accumulator-empty barrier (remote for the peer)
//
// Tiles (256 weight rows x 256 tokens) are distributed round-robin over the pairs of a
// persistent grid; two TMEM accumulators (2 x 256 columns) let the epilogue of one tile
// overlap the MMAs of the next.
#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <tuple>

#include "gemm_common.cuh"

namespace pcb::kern {

CUtensorMap tmap_bf16_2d(const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows);

namespace {

constexpr int k2Threads = 192;
constexpr int k2Stages = 6;
constexpr int kTileW = 128 * 64 * 2;   // one CTA's weight tile per k-block (16 KB)
constexpr int kTileX = 128 * 64 * 2;   // one CTA's token half-tile per k-block (16 KB)
constexpr int kStage2 = kTileW + kTileX;
constexpr int kBytes2 = k2Stages * kStage2 + 1024 + 1024;

// packed weights viewed as rows of 128 B ([N/128 * K/64 * 128][64] bf16, already in the
// SW128 smem image): a 64 x 128 box is one 16 KB tile copied verbatim
CUtensorMap tmap_packed(const void* ptr, uint64_t rows) {
  static std::mutex mu;
  static std::map<std::pair<const void*, uint64_t>, CUtensorMap> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({ptr, rows});
  if (it != cache.end()) return it->second;
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    PCB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    return reinterpret_cast<EncodeFn>(p);
  }();
  CUtensorMap m;
  cuuint64_t dims[2] = {64, rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (packed weights) failed");
  if (cache.size() > 4096) cache.clear();
  cache.emplace(std::make_pair(ptr, rows), m);
  return m;
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// 2-D TMA load whose bytes complete on the leader CTA's mbarrier (`bar_leader`: a
// shared::cluster address, mapa'd to rank 0)
__device__ __forceinline__ void tma_2sm(void* dst, const CUtensorMap* m, uint32_t bar_leader, int x, int y,
                                        uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_leader), "r"(x), "r"(y), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void umma_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive (once) on the barrier at this smem offset in both CTAs of the pair
__device__ __forceinline__ void commit_2sm_both(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}" ::"r"(
          smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

struct Args2 {
  int64_t M;
  int N, K, kbs, m_tiles, tiles;
};

__global__ void __launch_bounds__(k2Threads, 1)
    k_gemm_2sm(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, Args2 a, Epilogue e) {
  extern __shared__ uint8_t smem_raw[];
  // pointer arithmetic on the __shared__ symbol (not an integer round trip) keeps the
  // shared address space visible to the compiler: LDS/STS instead of generic LD/ST
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + k2Stages * kStage2);
  uint64_t* empty = full + k2Stages;
  uint64_t* acc_full = empty + k2Stages;  // [2]
  uint64_t* acc_empty = acc_full + 2;     // [2] leader: one arrival per CTA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int kbs = a.kbs;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmW);
    tma_prefetch(&tmX);
    for (int s = 0; s < k2Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 2);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs' barriers initialised before any remote signal
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      pdl_wait();
      const uint32_t full_leader = mapa_shared(smem_u32(full), 0);
      const uint64_t pol_w = policy_evict_last();  // re-read by every token tile
      const uint64_t pol_x = policy_evict_last();
      int it = 0;
      for (int t = pair; t < a.tiles; t += npairs) {
        const int n_pair = t / a.m_tiles, m_tile = t - n_pair * a.m_tiles;
        const int wrow0 = ((n_pair * 2 + static_cast<int>(rank)) * kbs) * 128;
        const int xrow = m_tile * 256 + static_cast<int>(rank) * 128;
        for (int kb = 0; kb < kbs; ++kb, ++it) {
          const int s = it % k2Stages;
          mbar_wait(&empty[s], ((it / k2Stages) & 1) ^ 1);
          if (rank == 0) mbar_expect_tx(&full[s], 2 * kStage2);
          uint8_t* st = smem + s * kStage2;
          const uint32_t bar = full_leader + s * 8;
          tma_2sm(st, &tmW, bar, 0, wrow0 + kb * 128, pol_w);
          tma_2sm(st + kTileW, &tmX, bar, kb * 64, xrow, pol_x);
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0 && elect_one()) {
      constexpr uint32_t idesc = idesc_bf16(256, 256);
      int it = 0, tc = 0;
      for (int t = pair; t < a.tiles; t += npairs, ++tc) {
        const int b = tc & 1;
        mbar_wait(&acc_empty[b], ((tc >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t acc = tmem + b * 256;
        for (int kb = 0; kb < kbs; ++kb, ++it) {
          const int s = it % k2Stages;
          mbar_wait(&full[s], (it / k2Stages) & 1);
          tc_fence_after();
          const uint32_t wa = smem_u32(smem + s * kStage2), xb = wa + kTileW;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_2sm(acc, sw128_kmajor_desc(wa + k * 32), sw128_kmajor_desc(xb + k * 32), idesc,
                     (kb > 0 || k > 0) ? 1u : 0u);
          commit_2sm_both(&empty[s]);
        }
        commit_2sm_both(&acc_full[b]);
      }
    }
  } else {
    // ---- epilogue: this CTA's 128 weight rows (TMEM lanes) x 256 tokens (columns) ----
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int et = threadIdx.x - 64;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    const uint32_t acc_empty_leader = mapa_shared(smem_u32(acc_empty), 0);
    pdl_wait();
    float v[16];
    int tc = 0;
    for (int t = pair; t < a.tiles; t += npairs, ++tc) {
      const int n_pair = t / a.m_tiles, m_tile = t - n_pair * a.m_tiles;
      const int n = (n_pair * 2 + static_cast<int>(rank)) * 128 + row;
      const int64_t m_base = static_cast<int64_t>(m_tile) * 256;
      const int b = tc & 1;
      EpiPre cur, nxt;
      epi_prefetch(e, n, a.N, m_base, a.M, cur);
      mbar_wait(&acc_full[b], (tc >> 1) & 1);
      tc_fence_after();
      const uint32_t acc = tmem + b * 256 + lane_off;
#pragma unroll 1
      for (int cc = 0; cc < 256; cc += 16) {
        if (m_base + cc >= a.M) break;  // warp-uniform
        if (cc + 16 < 256 && m_base + cc + 16 < a.M) epi_prefetch(e, n, a.N, m_base + cc + 16, a.M, nxt);
        tmem_ld16(acc + cc, v);
        epi_chunk(e, n, a.N, m_base + cc, a.M, v, cur);
        cur = nxt;
      }
      tc_fence_before();
      named_bar(1, 128);
      if (et == 0) mbar_arrive_remote(acc_empty_leader + b * 8);
    }
  }
  tc_fence_before();
  cluster_sync_all();  // the peer's epilogue is done with its TMEM before the pair frees it
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u) : "memory");
}

}  // namespace

bool gemm_2sm_supported(int64_t M, int N, int K) {
  static const bool on = [] {
    const char* v = std::getenv("PCB_GEMM_2SM");
    return !(v && v[0] == '0');
  }();
  return on && M >= 256 && N % 256 == 0 && K % 64 == 0 && K >= 64;
}

void gemm_2sm(const void* A, const void* Wp, int64_t M, int N, int K, const Epilogue& e, cudaStream_t s) {
  static int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  static bool attr = [] {
    PCB_CUDA(cudaFuncSetAttribute(k_gemm_2sm, cudaFuncAttributeMaxDynamicSharedMemorySize, kBytes2));
    PCB_CUDA(cudaFuncSetAttribute(k_gemm_2sm, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
    return true;
  }();
  (void)attr;
  Args2 a;
  a.M = M;
  a.N = N;
  a.K = K;
  a.kbs = K / 64;
  a.m_tiles = static_cast<int>((M + 255) / 256);
  a.tiles = (N / 256) * a.m_tiles;
  const int pairs = std::max(1, std::min(sms / 2, a.tiles));
  CUtensorMap tw = tmap_packed(Wp, static_cast<uint64_t>(N / 128) * a.kbs * 128);
  CUtensorMap tx = tmap_bf16_2d(A, static_cast<uint64_t>(M), static_cast<uint64_t>(K), 128);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(k2Threads);
  cfg.dynamicSmemBytes = kBytes2;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = (pdl_enabled() && ((pdl_mask() >> PDL_GEMM) & 1)) ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  PCB_CUDA(cudaLaunchKernelEx(&cfg, k_gemm_2sm, tw, tx, a, e));
}

}  // namespace pcb::kern

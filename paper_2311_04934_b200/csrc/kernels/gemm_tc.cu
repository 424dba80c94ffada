// tcgen05 GEMM for the bf16 hot path: C[m][n] = sum_k X[m][k] * W[n][k] with
// the epilogue fused (RoPE + K/V cache write, residual add, GELU, fp32 logits).
//
// Orientation ("swap AB"): the weight tile is the MMA A operand (M = 128 weight
// rows per CTA) and the token tile the B operand (N = BN tokens), so a 64-token
// suffix still issues full-height 128xBNx16 UMMAs and the kernel streams weights
// — the HBM-bound quantity at small token counts.
//   warp 0     TMA producer (one elected lane): W tile [128 x 64] + X tile [BN x 64]
//   warp 1     TMEM allocator + MMA issuer (one elected lane)
//   warps 2-5  epilogue: tcgen05.ld (lane = weight row, column = token) -> fused op
// Split-K over CTAs fills all 148 SMs when (N/128) x token tiles is small; the
// partial sums meet in an L2-resident workspace and the last-arriving CTA of a
// tile adds them in split order (deterministic) before running the epilogue.
#include <cuda.h>

#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "tc_common.cuh"

namespace pcb::kern {

using namespace tc;

// ---------------------------------------------------------------------------
// Host: tensor maps via the driver entry point (no -lcuda link dependency).
// ---------------------------------------------------------------------------
namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    PCB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}
}  // namespace

// 2-D bf16 tensor [rows][cols] (cols contiguous), box [box_rows][64], 128-byte swizzle.
CUtensorMap tmap_bf16_2d(const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, uint64_t, uint64_t, uint32_t>, CUtensorMap> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(ptr, rows, cols, box_rows);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  CUtensorMap m;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, m);
  return m;
}

// ---------------------------------------------------------------------------
// Epilogue on one thread's weight row n for 16 consecutive tokens.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void epi_chunk(const Epilogue& e, int n, int N, int64_t m0, int64_t M, float* v) {
  if (e.kind == EPI_QKV) {
    const int seg = n / e.d, c = n - seg * e.d;
    const bool rot = seg < 2 && e.rope;
    const int half = e.head_dim >> 1, pi = (c % e.head_dim) >> 1;
    const bool odd = c & 1;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float pv = __shfl_xor_sync(0xffffffffu, v[j], 1);  // partner column n^1 lives in lane^1
      int64_t m = m0 + j;
      if (rot && m < M) {
        int64_t p = e.pos[m];
        float cs = e.rope_cos32[p * half + pi], sn = e.rope_sin32[p * half + pi];
        v[j] = odd ? (pv * sn + v[j] * cs) : (v[j] * cs - pv * sn);
      }
    }
    __nv_bfloat16* dst = seg == 0 ? static_cast<__nv_bfloat16*>(e.q_out)
                                  : static_cast<__nv_bfloat16*>(seg == 1 ? e.k_out : e.v_out) + e.kv_row0 * e.d;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (m0 + j < M) dst[(m0 + j) * e.d + c] = __float2bfloat16_rn(v[j]);
    return;
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int64_t m = m0 + j;
    if (m >= M) break;
    if (e.kind == EPI_RESID) {
      e.resid[m * N + n] += v[j];
    } else if (e.kind == EPI_GELU) {
      static_cast<__nv_bfloat16*>(e.out)[m * N + n] = __float2bfloat16_rn(gelu_fast(v[j]));
    } else {
      e.outf[m * e.ldo + n] = v[j];
    }
  }
}

constexpr int kThreads = 192;

template <int BN, int STAGES>
struct GemmSmem {
  static constexpr int kA = 128 * 64 * 2;  // weight tile
  static constexpr int kB = BN * 64 * 2;   // token tile
  static constexpr int kStage = kA + kB;
  static constexpr int kBytes = STAGES * kStage + 1024 /*barriers*/ + 1024 /*align*/;
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, int64_t M, int N,
              int K, int splits, Epilogue e, float* __restrict__ ws, int* __restrict__ counters) {
  using S = GemmSmem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::kStage);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tile = blockIdx.x, m_tile = blockIdx.y, split = blockIdx.z;
  const int n0 = n_tile * 128;
  const int64_t m0 = static_cast<int64_t>(m_tile) * BN;
  const int total_kb = K / 64;
  const int kb0 = static_cast<int>(static_cast<int64_t>(split) * total_kb / splits);
  const int kb1 = static_cast<int>(static_cast<int64_t>(split + 1) * total_kb / splits);
  constexpr uint32_t kCols = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmW);
    tma_prefetch(&tmX);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();  // weights stream once
      const uint64_t pol_x = policy_evict_last();   // activations are re-read by every CTA
      for (int kb = kb0, it = 0; kb < kb1; ++kb, ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * S::kStage;
        mbar_expect_tx(&full[s], S::kStage);
        tma_load_2d_hint(sa, &tmW, &full[s], kb * 64, n0, pol_w);
        tma_load_2d_hint(sa + S::kA, &tmX, &full[s], kb * 64, static_cast<int>(m0), pol_x);
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16(128, BN);
      for (int kb = kb0, it = 0; kb < kb1; ++kb, ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a = smem_u32(smem + s * S::kStage);
        const uint32_t b = a + S::kA;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16(tmem, sw128_kmajor_desc(a + k * 32), sw128_kmajor_desc(b + k * 32), idesc,
                    (kb > kb0 || k > 0) ? 1u : 0u);
        umma_commit(&empty[s]);
      }
      umma_commit(tmem_full);
    }
  } else {
    // ---- epilogue warps 2..5: TMEM lane quadrant = warp % 4 ----
    const int q = warp & 3;
    const int row = q * 32 + lane;  // weight row within the tile
    const int n = n0 + row;
    const int et = threadIdx.x - 64;  // 0..127
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16);
    float v[16];
    if (splits == 1) {
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        tmem_ld16(taddr + c, v);
        if (m0 + c < M) epi_chunk(e, n, N, m0 + c, M, v);
      }
    } else {
      const int tile = m_tile * gridDim.x + n_tile;
      float* mine = ws + (static_cast<int64_t>(tile) * splits + split) * (BN * 128);
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        tmem_ld16(taddr + c, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) mine[(c + j) * 128 + row] = v[j];
      }
      __threadfence();
      named_bar(1, 128);
      if (et == 0) *last_flag = (atomicAdd(&counters[tile], 1) == splits - 1);
      named_bar(1, 128);
      if (*last_flag) {
        __threadfence();
        const float* base = ws + static_cast<int64_t>(tile) * splits * (BN * 128);
#pragma unroll 1
        for (int c = 0; c < BN; c += 16) {
          if (m0 + c >= M) break;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float acc = 0.f;
            for (int s2 = 0; s2 < splits; ++s2) acc += __ldcg(base + s2 * (BN * 128) + (c + j) * 128 + row);
            v[j] = acc;
          }
          epi_chunk(e, n, N, m0 + c, M, v);
        }
        if (et == 0) counters[tile] = 0;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, kCols);
}

bool gemm_tc_supported(int64_t M, int N, int K) { return M >= 1 && N % 128 == 0 && K % 64 == 0 && K >= 64; }

CUtensorMap tmap_bf16_2d(const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows);

template <int BN, int STAGES>
static void launch(const void* A, const void* W, int64_t M, int N, int K, const Epilogue& e, float* ws,
                   size_t ws_bytes, int* counters, cudaStream_t s, int sms) {
  using Sm = GemmSmem<BN, STAGES>;
  static bool attr = [] {
    PCB_CUDA(cudaFuncSetAttribute(k_gemm_tc<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, Sm::kBytes));
    return true;
  }();
  (void)attr;
  const int n_tiles = N / 128;
  const int m_tiles = static_cast<int>((M + BN - 1) / BN);
  const int tiles = n_tiles * m_tiles;
  const int kbs = K / 64;
  // CTAs resident per SM given the shared-memory footprint
  const int per_sm = std::max(1, (227 * 1024) / Sm::kBytes);
  const int slots = sms * per_sm;
  int splits = 1;
  if (tiles < slots) {
    splits = std::min(kbs / 2 > 0 ? kbs / 2 : 1, std::max(1, slots / tiles));
    splits = std::max(1, std::min(splits, 16));
  }
  while (splits > 1 && static_cast<size_t>(tiles) * splits * BN * 128 * sizeof(float) > ws_bytes) --splits;
  CUtensorMap tw = tmap_bf16_2d(W, static_cast<uint64_t>(N), static_cast<uint64_t>(K), 128);
  CUtensorMap tx = tmap_bf16_2d(A, static_cast<uint64_t>(M), static_cast<uint64_t>(K), BN);
  dim3 grid(n_tiles, m_tiles, splits);
  k_gemm_tc<BN, STAGES><<<grid, kThreads, Sm::kBytes, s>>>(tw, tx, M, N, K, splits, e, ws, counters);
  PCB_CUDA(cudaGetLastError());
}

void gemm_tc(const void* A, const void* W, int64_t M, int N, int K, const Epilogue& e, float* ws, size_t ws_bytes,
             int* counters, cudaStream_t s) {
  if (M <= 0) return;
  static int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  if (M <= 16) launch<16, 5>(A, W, M, N, K, e, ws, ws_bytes, counters, s, sms);
  else if (M <= 32) launch<32, 5>(A, W, M, N, K, e, ws, ws_bytes, counters, s, sms);
  else if (M <= 64) launch<64, 4>(A, W, M, N, K, e, ws, ws_bytes, counters, s, sms);
  else if (M <= 128) launch<128, 4>(A, W, M, N, K, e, ws, ws_bytes, counters, s, sms);
  else launch<256, 4>(A, W, M, N, K, e, ws, ws_bytes, counters, s, sms);
}

}  // namespace pcb::kern

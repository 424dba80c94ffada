// tcgen05 GEMM for the bf16 hot path: C[m][n] = sum_k X[m][k] * W[n][k] with
// the epilogue fused (RoPE + K/V cache write, residual add, GELU, fp32 logits).
//
// Design (B200-first):
//  * Weights live in HBM pre-packed as 128x64 bf16 tiles, each tile stored as the
//    exact 128-byte-swizzled shared-memory image the UMMA descriptor expects, tiles
//    of one 128-row block contiguous along K.  A tile is one 16 KB cp.async.bulk:
//    the weight stream is a handful of long sequential reads per SM.
//  * "Swap AB": the weight tile is the MMA A operand (M = 128 weight rows), the
//    token tile the B operand (N = BN tokens), so a 64-token suffix still issues
//    full-height 128xBNx16 UMMAs.
//  * Persistent stream-K: one CTA per SM; the (tile, k-block) units are split into
//    equal contiguous ranges, so every SM streams the same number of weight bytes
//    (the HBM-bound quantity at small token counts).  A tile cut
//    between CTAs is finished by the CTA holding its last k-block, which adds the
//    other CTAs' fp32 partials in CTA order (deterministic) before the epilogue.
//  * Two TMEM accumulators: the epilogue of one tile overlaps the MMAs of the next.
//   warp 0     producer: W tile (bulk copy) + X tile (TMA 2-D) per k-block
//   warp 1     TMEM allocator + MMA issuer (one elected lane)
//   warps 2-5  epilogue: tcgen05.ld (lane = weight row, column = token) -> fused op
#include <cuda.h>

#include <atomic>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "tc_common.cuh"
#include "gemm_common.cuh"

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
// Weight packing: row-major [N][K] bf16 -> tiles [N/128][K/64] of 16 KB, each the
// SW128 K-major smem image (row r at r*128 B, 16-byte chunk c at (c ^ (r & 7))).
// ---------------------------------------------------------------------------
__host__ __device__ inline uint64_t packed_offset_bytes(int n, int k, int K) { return packed_index(n, k, K) * 2; }

__global__ void k_pack(const uint4* __restrict__ src, uint8_t* __restrict__ dst, int N, int K) {
  const int64_t chunks = static_cast<int64_t>(N) * (K / 8);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < chunks; i += (int64_t)gridDim.x * blockDim.x) {
    const int n = static_cast<int>(i / (K / 8)), k = static_cast<int>(i % (K / 8)) * 8;
    *reinterpret_cast<uint4*>(dst + packed_offset_bytes(n, k, K)) = src[i];
  }
}

bool weight_packable(int N, int K) { return N % 128 == 0 && K % 64 == 0 && K >= 64; }

void pack_weight_bf16(const void* src, void* dst, int N, int K, cudaStream_t s) {
  k_pack<<<592, 256, 0, s>>>(static_cast<const uint4*>(src), static_cast<uint8_t*>(dst), N, K);
  PCB_CUDA(cudaGetLastError());
}

constexpr int kThreads = 192;
constexpr int kWTile = 128 * 64 * 2;  // one packed weight tile

template <int BN, int STAGES>
struct SkSmem {
  static constexpr int kStage = kWTile + BN * 128;
  static constexpr int kBytes = STAGES * kStage + 1024 + 1024;
  static constexpr uint32_t kCols = 2 * BN < 32 ? 32 : 2 * BN;  // two accumulators
};

struct SkArgs {
  const uint8_t* w;  // packed weights
  int64_t M;
  int N, K, kbs, m_tiles;
  int64_t units;
  int epoch;
  float* ws;  // [gridDim.x][128][BN] partial tiles
  int* flags; // [gridDim.x] epoch flags
  unsigned long long* tl = nullptr;  // timeline probe: [cta][4] globaltimer ns (PCB_GEMM_PROBE)
};

__device__ __forceinline__ void tl_mark(const SkArgs& a, int ev) {
  if (a.tl) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.tl[blockIdx.x * 4 + ev] = t;
  }
}

template <int BN, int STAGES, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    k_gemm_sk(const __grid_constant__ CUtensorMap tmX, SkArgs a, Epilogue e) {
  using S = SkSmem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  // pointer arithmetic on the __shared__ symbol (not an integer round trip) keeps the
  // shared address space visible to the compiler: LDS/STS instead of generic LD/ST
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::kStage);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = gridDim.x, c = blockIdx.x;
  const int64_t g0 = unit_begin(c, a.units, C), g1 = unit_begin(c + 1, a.units, C);
  const int kbs = a.kbs;
  if (threadIdx.x == 0) tl_mark(a, 0);  // entry

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, S::kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();

  if (warp == 0) {
    if (elect_one()) {
      // one token tile: weights stream through once (evict first); several token tiles
      // (prefill / precompute): each weight tile is re-read per token tile, keep it
      const uint64_t pol_w = a.m_tiles == 1 ? policy_evict_first() : policy_evict_last();
      const uint64_t pol_x = policy_evict_last();  // activations are re-read by every CTA
      auto w_src = [&](int64_t g) {
        const int64_t t = g / kbs;
        const int kb = static_cast<int>(g - t * kbs);
        const int n_tile = static_cast<int>(t / a.m_tiles);
        return a.w + (static_cast<int64_t>(n_tile) * kbs + kb) * kWTile;
      };
      auto x_coords = [&](int64_t g, int& kx, int& my) {
        const int64_t t = g / kbs;
        kx = static_cast<int>(g - t * kbs) * 64;
        my = static_cast<int>(t % a.m_tiles) * BN;
      };
      // Weights do not depend on the previous kernel: start streaming them before
      // waiting on it (programmatic dependent launch), then the activations.
      const int pre = static_cast<int>((g1 - g0) < STAGES ? (g1 - g0) : STAGES);
      for (int it = 0; it < pre; ++it) {
        mbar_expect_tx(&full[it], S::kStage);
        bulk_load(smem + it * S::kStage, w_src(g0 + it), kWTile, &full[it], pol_w);
      }
      pdl_wait();
      for (int it = 0; it < pre; ++it) {
        int kx, my;
        x_coords(g0 + it, kx, my);
        tma_load_2d_hint(smem + it * S::kStage + kWTile, &tmX, &full[it], kx, my, pol_x);
      }
      int it = pre;
      for (int64_t g = g0 + pre; g < g1; ++g, ++it) {
        const int s = it % STAGES;
        mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
        uint8_t* st = smem + s * S::kStage;
        mbar_expect_tx(&full[s], S::kStage);
        bulk_load(st, w_src(g), kWTile, &full[s], pol_w);
        int kx, my;
        x_coords(g, kx, my);
        tma_load_2d_hint(st + kWTile, &tmX, &full[s], kx, my, pol_x);
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16(128, BN);
      int it = 0, seg = 0;
      for (int64_t g = g0; g < g1; ++seg) {
        const int64_t t = g / kbs;
        const int64_t ge = min(g1, (t + 1) * kbs);
        const int buf = seg & 1;
        mbar_wait(&acc_empty[buf], ((seg >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t acc = tmem + buf * BN;
        for (int64_t u = g; u < ge; ++u, ++it) {
          const int s = it % STAGES;
          for (uint32_t sp = 0; !mbar_try(&full[s], (it / STAGES) & 1);)
            if (++sp == (1u << 25)) {
              printf("[pcb] gemm stage timeout: block %d/%d it %d/%lld M %lld N %d K %d BN %d epoch %d\n", blockIdx.x,
                     gridDim.x, it, (long long)(g1 - g0), (long long)a.M, a.N, a.K, BN, a.epoch);
              __trap();
            }
          if (it == 0) tl_mark(a, 1);             // first stage landed
          if (u + 1 == g1) tl_mark(a, 2);         // last stage landed
          tc_fence_after();
          const uint32_t wa = smem_u32(smem + s * S::kStage), xb = wa + kWTile;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(acc, sw128_kmajor_desc(wa + k * 32), sw128_kmajor_desc(xb + k * 32), idesc,
                      (u > g || k > 0) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(&acc_full[buf]);
        g = ge;
      }
    }
  } else {
    // ---- epilogue warps 2..5: TMEM lane quadrant = warp % 4 ----
    const int q = warp & 3;
    const int row = q * 32 + lane;  // weight row within the tile
    const int et = threadIdx.x - 64;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    pdl_wait();  // the epilogue reads / writes activations of earlier kernels
    float v[16];
    int seg = 0;
    for (int64_t g = g0; g < g1; ++seg) {
      const int64_t t = g / kbs;
      const int64_t tb = t * kbs, te = (t + 1) * kbs;
      const int64_t ge = min(g1, te);
      const int n_tile = static_cast<int>(t / a.m_tiles), m_tile = static_cast<int>(t % a.m_tiles);
      const int n = n_tile * 128 + row;
      const int64_t m0 = static_cast<int64_t>(m_tile) * BN;
      const int buf = seg & 1;
      const uint32_t acc = tmem + buf * BN + lane_off;
      EpiPre cur;
      if (g == tb) epi_prefetch(e, n, a.N, m0, a.M, cur);  // before the accumulator is ready
      mbar_wait(&acc_full[buf], (seg >> 1) & 1);
      tc_fence_after();
      if (g > tb) {
        // tile started in an earlier CTA (this is our first segment): park the
        // partial for the owner (the CTA holding the tile's first k-block)
        float* dst = a.ws + (static_cast<int64_t>(c) * 128 + row) * BN;
#pragma unroll 1
        for (int cc = 0; cc < BN; cc += 16) {
          tmem_ld16(acc + cc, v);
#pragma unroll
          for (int j = 0; j < 16; j += 4) *reinterpret_cast<float4*>(dst + cc + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
        tc_fence_before();
        mbar_arrive(&acc_empty[buf]);
        // one gpu-scope release by et 0 (st_release) publishes the CTA's partial: bar.sync
        // orders the other threads' stores before it (cumulativity)
        named_bar(1, 128);
        if (et == 0) st_release(a.flags + c, a.epoch);
      } else {
        // owner (or sole CTA) of tile t: add the later CTAs' partials (their first
        // segments, finished long before this, our last segment) in CTA order
        const int c_last = ge < te ? cta_of(te - 1, a.units, C) : c;
        if (c_last > c) {
          for (int p = c + 1 + et; p <= c_last; p += 128)
            for (uint32_t spins = 0; ld_relaxed(a.flags + p) < a.epoch;) {
              __nanosleep(64);
              if (++spins == (1u << 25)) wait_timeout("stream-K flag", a.flags + p, a.epoch);
            }
          fence_acquire_gpu();
          named_bar(1, 128);
        }
        if (a.m_tiles == 1) {
          owner_finish<BN>(e, acc, n, a.N, a.M, a.ws, c, c_last, a.units, C, row, cur);
        } else {
          // several token tiles (prefill): chunked, the token offset m0 applies
          EpiPre nxt;
#pragma unroll 1
          for (int cc = 0; cc < BN; cc += 16) {
            if (m0 + cc >= a.M) break;  // warp-uniform
            if (cc + 16 < BN && m0 + cc + 16 < a.M) epi_prefetch(e, n, a.N, m0 + cc + 16, a.M, nxt);
            tmem_ld16(acc + cc, v);
            for (int p = c + 1; p <= c_last; ++p) {
              const float* src = a.ws + (static_cast<int64_t>(p) * 128 + row) * BN + cc;
#pragma unroll
              for (int j = 0; j < 16; j += 4) {
                const float4 f = __ldcg(reinterpret_cast<const float4*>(src + j));
                v[j] += f.x;
                v[j + 1] += f.y;
                v[j + 2] += f.z;
                v[j + 3] += f.w;
              }
            }
            epi_chunk(e, n, a.N, m0 + cc, a.M, v, cur);
            cur = nxt;
          }
        }
        tc_fence_before();
        mbar_arrive(&acc_empty[buf]);
      }
      g = ge;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) tl_mark(a, 3);  // epilogue done
  if (warp == 1) tmem_dealloc(tmem, S::kCols);
}

bool gemm_tc_supported(int64_t M, int N, int K) { return M >= 1 && weight_packable(N, K); }

// one launch counter for every instantiation: all of them share a model's flag array
static std::atomic<int> g_sk_epoch{0};

// ---- timeline probe (PCB_GEMM_PROBE=1): per launch, per CTA {entry, first stage landed,
// last stage landed, done} in globaltimer ns, plus the launch shape ----
namespace {
constexpr int kProbeLaunches = 1024, kProbeCtas = 160;
unsigned long long* g_tl = nullptr;
int g_tl_n = 0;
int64_t g_tl_shape[kProbeLaunches][4];
unsigned long long* probe_slot(int64_t M, int N, int K, int C) {
  static const bool on = std::getenv("PCB_GEMM_PROBE") != nullptr;
  if (!on) return nullptr;
  if (!g_tl) {
    PCB_CUDA(cudaMallocManaged(&g_tl, sizeof(unsigned long long) * kProbeLaunches * kProbeCtas * 4));
    std::memset(g_tl, 0, sizeof(unsigned long long) * kProbeLaunches * kProbeCtas * 4);
  }
  if (g_tl_n >= kProbeLaunches) return nullptr;
  g_tl_shape[g_tl_n][0] = M;
  g_tl_shape[g_tl_n][1] = N;
  g_tl_shape[g_tl_n][2] = K;
  g_tl_shape[g_tl_n][3] = C;
  return g_tl + static_cast<size_t>(g_tl_n++) * kProbeCtas * 4;
}
}  // namespace

int gemm_probe_dump(int64_t* shapes, unsigned long long* times, int max_launches) {
  PCB_CUDA(cudaDeviceSynchronize());
  const int n = std::min(g_tl_n, max_launches);
  for (int i = 0; i < n; ++i) {
    std::memcpy(shapes + i * 4, g_tl_shape[i], sizeof(int64_t) * 4);
    std::memcpy(times + static_cast<size_t>(i) * kProbeCtas * 4, g_tl + static_cast<size_t>(i) * kProbeCtas * 4,
                sizeof(unsigned long long) * kProbeCtas * 4);
  }
  g_tl_n = 0;
  return n;
}

template <int BN, int STAGES, int MINB = 1>
static void launch_sk(const void* A, const void* Wp, int64_t M, int N, int K, const Epilogue& e, float* ws,
                      size_t ws_bytes, int* flags, cudaStream_t s, int sms) {
  using Sm = SkSmem<BN, STAGES>;
  static bool attr = [] {
    PCB_CUDA(cudaFuncSetAttribute(k_gemm_sk<BN, STAGES, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, Sm::kBytes));
    return true;
  }();
  (void)attr;
  SkArgs a;
  a.w = static_cast<const uint8_t*>(Wp);
  a.M = M;
  a.N = N;
  a.K = K;
  a.kbs = K / 64;
  a.m_tiles = static_cast<int>((M + BN - 1) / BN);
  a.units = static_cast<int64_t>(N / 128) * a.m_tiles * a.kbs;
  if (!units_fit_u32(a.units, sms)) throw std::runtime_error("gemm: too many work units for the 32-bit split");
  a.ws = ws;
  a.flags = flags;
  a.epoch = ++g_sk_epoch;
  int C = static_cast<int>(std::min<int64_t>(sms, a.units));
  static const int ctas_env = [] {  // tuning override (environment read once)
    const char* v = std::getenv("PCB_GEMM_CTAS");
    return v ? std::max(1, std::atoi(v)) : 0;
  }();
  if (ctas_env) C = std::min(C, ctas_env);
  if (static_cast<size_t>(C) * 128 * BN * sizeof(float) > ws_bytes) throw std::runtime_error("gemm workspace too small");
  a.tl = probe_slot(M, N, K, C);
  CUtensorMap tx = tmap_bf16_2d(A, static_cast<uint64_t>(M), static_cast<uint64_t>(K), BN);
  PdlClass pc(PDL_GEMM);
  launch_k(k_gemm_sk<BN, STAGES, MINB>, dim3(C), dim3(kThreads), Sm::kBytes, s, 1, tx, a, e);
}

void gemm_tc(const void* A, const void* Wp, int64_t M, int N, int K, const Epilogue& e, float* ws, size_t ws_bytes,
             int* flags, cudaStream_t s) {
  if (M <= 0) return;
  static int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  // (Tried: weight-streaming shapes sized for two co-resident CTAs per SM so the next
  // PDL-launched GEMM overlaps this one's drain -- measured slower, 8.1 vs 6.6 ms per 7B
  // request: shallower pipelines and uneven CTA placement.  The few-token path is the
  // persistent chain kernel, chain_tc.cu.)
  if (gemm_2sm_supported(M, N, K)) {
    gemm_2sm(A, Wp, M, N, K, e, s);
    return;
  }
  if (M <= 16) launch_sk<16, 10>(A, Wp, M, N, K, e, ws, ws_bytes, flags, s, sms);
  else if (M <= 32) launch_sk<32, 10>(A, Wp, M, N, K, e, ws, ws_bytes, flags, s, sms);
  else if (M <= 64) launch_sk<64, 8>(A, Wp, M, N, K, e, ws, ws_bytes, flags, s, sms);
  else if (M <= 128) launch_sk<128, 6>(A, Wp, M, N, K, e, ws, ws_bytes, flags, s, sms);
  else launch_sk<256, 4>(A, Wp, M, N, K, e, ws, ws_bytes, flags, s, sms);
}

}  // namespace pcb::kern

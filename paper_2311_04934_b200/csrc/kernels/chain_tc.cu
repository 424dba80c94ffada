// Persistent chain of weight-streaming GEMM and LayerNorm phases for the few-token
// (suffix prefill / decode) regime.  A launch runs the phases of up to 9 transformer layers:
//
//   [LN1_0, QKV_0] then per layer [attention_l, O_l (+resid), W1_l (+GELU), W2_l (+resid), QKV_{l+1}]
//
// with LayerNorm folded into the neighbouring GEMMs (LN phases when the fold is off; the
// last layer ends with the unembedding), reference Model::run, model.cpp:376-436.  An
// attention phase (one request, hd 128) runs the attn_tc.cu pipeline on the ring's shared
// memory -- TMA Q and K/V blocks, QK^T and PV on tcgen05 with S, P and O in TMEM, online
// softmax on the epilogue warps -- over (head, key split) items whose partials merge through
// the cluster's DSMEM; each CTA hands the ring back to the weight stream as soon as its own
// item is done, and the cached modules' K/V blocks load before the grid barrier that
// publishes the phase's Q.  (As a separate kernel, and with one launch per layer, each layer
// paid a launch, a prologue and a cold start.)
// At 64 tokens every GEMM is HBM-bound on its weights, and as separate
// launches each one paid a ramp (launch, prologue, first weight bytes) and a drain
// (stream-K fix-up, epilogue, the slowest CTA) during which HBM idles: the measured
// per-layer time was ~2.6x the weight-streaming time (tools/gemm_timeline.py).
// Here the weight stream never stops at a phase boundary:
//
//   warp 0     W producer: bulk-copies the packed weight tiles of every phase in
//              order; weights depend on nothing, so it runs ahead across phase
//              boundaries, limited only by the shared-memory ring
//   warp 1     TMEM allocator + MMA issuer (swap-AB 128 x BN x 16 UMMAs)
//   warp 2     X producer: TMA-loads the activation tile of each unit, after the
//              grid barrier that publishes the phase's input
//   warps 3-6  epilogue (fused op, stream-K fix-up), LayerNorm rows, grid barrier
//
// Phases are separated by a grid-wide barrier (monotonic 64-bit arrival counter in
// global memory, release/acquire at gpu scope, proxy fences on both sides because the
// consumers read through TMA).  All CTAs are co-resident: the grid is one CTA per SM
// and dependents are released (PDL trigger) only after the first barrier proves it.
// Within a GEMM phase the work is tile-granular: a 128-row weight tile is one item
// (finished straight from TMEM) when there are at least C/2 tiles, else it is split
// along K into S = 2 or 4 items whose CTAs each park a partial and then finish 1/S of
// the token columns from all S partials (one batch of loads, split order: deterministic).
// A stream-K split (equal bytes per SM) was measured first: its owner-side fix-up at
// every phase end cost 8-17 us per phase against ~2-6 us here.  Partials are double-
// buffered by phase parity; flags carry per-phase epochs.
#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstring>
#include <type_traits>

#include "gemm_common.cuh"

namespace pcb::kern {

CUtensorMap tmap_bf16_2d(const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows);
CUtensorMap tmap_bf16_3d(const void* ptr, uint64_t cols, uint64_t rows, uint64_t planes, uint64_t plane_stride,
                         uint32_t box_rows);

namespace {

constexpr int kMaxPhases = kChainMaxPhases;  // [LN1, QKV] + 9 layers x [ATTN, O, W1, W2, QKV] + unembed
constexpr int kMaxAttn = 9;     // attention phases per launch
constexpr int kChainThreads = 224;  // 7 warps
constexpr int kWTileC = 128 * 64 * 2;

struct PhaseDev {
  int kind;  // CHAIN_GEMM / CHAIN_LN
  int N, K, kbs;
  int S;      // k-splits per 128-row weight tile (1: whole tiles; 2 or 4 when tiles are few)
  int items;  // tiles * S work items, item i -> CTA i mod C
  // folded LayerNorm: a residual phase writes per-(tile, token) {sum h, sum h^2} of the new
  // residual; the next GEMM phase turns them into {mean, rstd} per token
  float* stats_out;
  const float* stats_in;
  int stats_tiles, stats_ld, stats_row0, ln_dim;
  int64_t M, units;
  const uint8_t* w;
  const float* ln_src;
  __nv_bfloat16* ln_dst;
  int ln_d;
  Epilogue e;
  // attention phase: item = (head, key split); partials [items][128][128] then (m, l) [items][128]
  int64_t aP;
  int aH, aS, a_d;
  int adup;      // n <= 64: queries duplicated in the Q tile, each half of the lanes takes half the keys
  float ascale;  // log2(e) / sqrt(128)
  float* apart;
  __nv_bfloat16* aout;
  // zero-copy prefix: segment s covers key blocks [a_first[s], a_first[s+1]), rows
  // [a_row0[s], a_row0[s] + a_rows[s]) of its source (tensor map tkv[s], plane 2 layer + w);
  // the last segment is the request's own rows (first a_tail_vis visible to all queries)
  int a_nseg, a_layer, a_tail_vis;
  int a_map;  // index of the phase's K / V maps (contiguous cache)
  const float* a_alibi;   // ALiBi slopes [aH] (null: off); key positions by key block, query positions
  const int32_t* a_kpos;
  const int32_t* a_qpos;
  int a_first[ChainStep::kMaxSeg + 1];
  int a_row0[ChainStep::kMaxSeg];
  int a_rows[ChainStep::kMaxSeg];
};

struct ChainParams {
  CUtensorMap tm[kMaxPhases];  // activation maps of the GEMM phases
  CUtensorMap tma[1];          // attention phases: Q [n][d] (one buffer for every layer)
  CUtensorMap tak[kMaxAttn], tav[kMaxAttn];  // attention phase a_map: K and V planes [P + n][d]
  CUtensorMap tkv[ChainStep::kMaxSeg];  // attention phase, zero-copy: {d, cap, planes} per KV source
  PhaseDev ph[kMaxPhases];
  int n_phases;
  int epoch0;
  float* ws;               // [2][C][128][BN] fp32 partial tiles (phase parity)
  int64_t ws_half;         // floats per parity half
  int* flags;              // [C] partial-ready epochs
  unsigned long long* gbar;  // grid barrier arrival counter (monotonic)
  unsigned long long gbar_base;
  unsigned long long* tl;    // timeline probe [phase][cta][4] (null: off)
  int warm;                  // dry epilogue pass while the weights stream (instruction cache)
  int dsm;                   // launched in clusters of 4: split partials / attention splits meet in DSMEM
};

static_assert(sizeof(ChainParams) <= 32764, "chain kernel parameters exceed the 32 KB parameter space");

// probe events per (phase, CTA): 0 X producer past the phase's barrier, 1 MMA took the
// phase's last stage, 2 epilogue done with the phase, 3 W producer issued the phase's
// last weight tile
__device__ __forceinline__ void ctl(const ChainParams& p, int ph, int ev) {
  if (p.tl) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.tl[(static_cast<size_t>(ph) * 160 + blockIdx.x) * 16 + ev] = t;
  }
}

template <int BN, int STAGES>
struct ChainSmem {
  static constexpr int kStage = kWTileC + BN * 128;
  // cluster exchange buffer (BN <= 64, dsm launches): a split GEMM phase parks its fp32
  // partial (float4 [BN / 4][128]) here, the attention phase its normalised O [64][132] +
  // (m, l)[64];
  // the S CTAs of a tile / head read each other's through DSMEM
  static constexpr int kPbLd = 132;  // floats per parked row (pad 4: conflict-free v4 rows)
  static constexpr int kPbAttn = 64 * kPbLd * 4 + 64 * 8, kPbGemm = 128 * BN * 4;
  static constexpr int kPB = BN <= 64 ? (kPbAttn > kPbGemm ? kPbAttn : kPbGemm) : 0;
  static constexpr int kBytes = STAGES * kStage + kPB + 1024 + 1024 + 1024 + 2 * 16 * 128 * 4;  // + LN-fold scratch
  static constexpr uint32_t kCols = 2 * BN < 32 ? 32 : 2 * BN;
  // attention phase: Q (32 KB) in the cluster exchange buffer when there is one (it is only
  // needed there after the last QK^T), P in TMEM, and the ring re-carved as K/V stages of 32 KB
  // (the phase is bound by K/V arrival: 4 -> 5 stages)
  static constexpr bool kQInPb = kPB >= 32768;
  static constexpr int kAttnFit = (STAGES * kStage - (kQInPb ? 0 : 32768)) / 32768;
  static constexpr int kAttnKV = kAttnFit > 6 ? 6 : kAttnFit;
  static_assert(kAttnKV >= 2, "attention phase needs two K/V stages in the ring");
};

constexpr float kRescaleThreshold = 8.0f;  // log2 domain: stale max tolerated up to 2^8 (as attn_tc.cu)

__device__ __forceinline__ void tmem_st16(uint32_t addr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          addr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tmem_st16u(uint32_t addr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float fast_exp2(float x) {  // MUFU.EX2; exp2(-inf) = +0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// probe slot holding a raw value (cycle counts) instead of a timestamp
__device__ __forceinline__ void ctl_val(const ChainParams& p, int ph, int ev, unsigned long long v) {
  if (p.tl) p.tl[(static_cast<size_t>(ph) * 160 + blockIdx.x) * 16 + ev] = v;
}

// wait until every CTA has finished phases [0, ph)
__device__ __forceinline__ void grid_wait(const ChainParams& p, int ph) {
  const unsigned long long target = p.gbar_base + static_cast<unsigned long long>(ph) * gridDim.x;
  for (uint32_t spins = 0; ld_relaxed_u64(p.gbar) < target;) {
    __nanosleep(32);
    if (++spins == (1u << 24)) {
#ifdef PCB_TIMEOUT_PRINTF
      printf("[pcb] chain grid barrier timeout: block %d thread %d phase %d/%d counter %llu target %llu\n", blockIdx.x,
             threadIdx.x, ph, p.n_phases, ld_acquire_u64(p.gbar), target);
#endif
      __trap();
    }
  }
  fence_acquire_gpu();
}

__device__ __forceinline__ double ln_sum128(double v, double* red, int et) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((et & 31) == 0) red[et >> 5] = v;
  named_bar(1, 128);
  const double t = red[0] + red[1] + red[2] + red[3];
  named_bar(1, 128);
  return t;
}

// One LayerNorm row (model.cpp:156-174: fp64 mean, fp64 centred variance, eps 1e-5,
// gamma 1, beta 0) by the 128 epilogue threads; d % 4 == 0, d <= 8192.
__device__ void ln_row(const PhaseDev& P, int64_t r, double* red, int et) {
  const int d = P.ln_d, nv = d >> 2;
  const float4* src = reinterpret_cast<const float4*>(P.ln_src + r * d);
  float4 x[16];
  double s = 0;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int i = et + u * 128;
    x[u] = i < nv ? __ldcg(src + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    s += (double)x[u].x + (double)x[u].y + (double)x[u].z + (double)x[u].w;
  }
  const double mean = ln_sum128(s, red, et) / d;
  double v = 0;
#pragma unroll
  for (int u = 0; u < 16; ++u)
    if (et + u * 128 < nv) {
      const double a = x[u].x - mean, b = x[u].y - mean, c = x[u].z - mean, e = x[u].w - mean;
      v += a * a + b * b + c * c + e * e;
    }
  const double inv = 1.0 / sqrt(ln_sum128(v, red, et) / d + 1e-5);
  __nv_bfloat16* dst = P.ln_dst + r * d;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int i = et + u * 128;
    if (i < nv) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(static_cast<float>((x[u].x - mean) * inv),
                                                static_cast<float>((x[u].y - mean) * inv));
      __nv_bfloat162 hi = __floats2bfloat162_rn(static_cast<float>((x[u].z - mean) * inv),
                                                static_cast<float>((x[u].w - mean) * inv));
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(dst + 4 * i) = pk;
    }
  }
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kChainThreads, 1) k_chain(const __grid_constant__ ChainParams p) {
  using S = ChainSmem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  // pointer arithmetic on the __shared__ symbol (not an integer round trip) keeps the
  // shared address space visible to the compiler: LDS/STS instead of generic LD/ST
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  float* pb = reinterpret_cast<float*>(smem + STAGES * S::kStage);  // cluster exchange buffer (S::kPB bytes)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::kStage + S::kPB);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  double* red = reinterpret_cast<double*>(acc_empty + 4);  // [4] LayerNorm partial sums
  float2* lnst = reinterpret_cast<float2*>(smem + STAGES * S::kStage + S::kPB + 1024);  // [128] {mean, rstd}
  float* colsum = reinterpret_cast<float*>(lnst + 128);  // [2][16 tokens][128 columns] h, h^2 of a chunk

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = gridDim.x, c = blockIdx.x;
  // launch probes (slot of phase kMaxPhases - 1): 0 entry, 1 prologue done, 2 epilogue past
  // the PDL wait, 3 exit
  if (threadIdx.x == 0) ctl(p, kMaxPhases - 1, 0);
  // attention phase (first phase only): the ring's shared memory is re-carved as Q, P and
  // K/V stages; its barriers sit 512 bytes into the barrier block; S and O live in TMEM
  // columns [256, 512), clear of the GEMM accumulators
  // attention phases: any position (a launch spans several layers); each takes the ring for
  // its K/V stages and needs the previous phase's outputs (Q, the new K/V rows)
  bool has_attn = false;
  for (int ph = 0; ph < p.n_phases; ++ph) has_attn |= p.ph[ph].kind == CHAIN_ATTN;
  constexpr int AKV = S::kAttnKV;
  uint8_t* aQ = S::kQInPb ? reinterpret_cast<uint8_t*>(pb) : smem;
  uint8_t* aKV = S::kQInPb ? smem : smem + 32768;
  uint64_t* a_qfull = full + 64;
  uint64_t* a_kvfull = a_qfull + 1;    // [AKV]
  uint64_t* a_kvempty = a_kvfull + 8;  // [AKV]
  // three score buffers: S(it + 2) is issued right after PV(it), so S(it + 1) is ready when the
  // softmax of block it ends (with two, S(it + 1) waited for PV(it - 1): ~500 cycles per block)
  uint64_t* a_sfull = a_kvempty + 8;   // [3] block it -> buffer it % 3, phase (it / 3) & 1
  uint64_t* a_pfull = a_sfull + 3;     // [3] (one per buffer: a single p_full can deadlock, attn_tc.cu)
  uint64_t* a_pvdone = a_pfull + 3;    // [3]
  uint64_t* a_done = a_pvdone + 3;     // this CTA's attention is off the ring (128 arrivals)
  // exchange-buffer barriers (dsm): pb_ready completes when every CTA of this CTA's group
  // has parked its data (each group member arrives once with count 4 / S, S = group size),
  // pb_free when they have all finished reading this CTA's buffer
  uint64_t* pb_ready = full + 100;
  uint64_t* pb_free = full + 101;
  const bool dsm = S::kPB > 0 && p.dsm;
  // a QKV phase with a per-request RoPE table stages each tile's {cos, sin} operands in TMEM
  // columns [256, 384) and [384, 512) while its weights stream (idle there: attention is
  // phase 0 only; GEMM accumulators use [0, 2 BN) with BN <= 128)
  bool rope_stage_any = false;
  for (int ph = 0; ph < p.n_phases; ++ph)
    rope_stage_any |= p.ph[ph].kind == CHAIN_GEMM && p.ph[ph].e.kind == EPI_QKV && p.ph[ph].e.rope &&
                      p.ph[ph].e.rope_tab != nullptr && p.ph[ph].S == 1;
  const uint32_t tcols = (has_attn || rope_stage_any) ? 512u : S::kCols;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 128);
    }
    if (has_attn) {
      mbar_init(a_qfull, 1);
      for (int s = 0; s < AKV; ++s) {
        mbar_init(&a_kvfull[s], 1);
        mbar_init(&a_kvempty[s], 1);
      }
      for (int b = 0; b < 3; ++b) {
        mbar_init(&a_sfull[b], 1);
        mbar_init(&a_pvdone[b], 1);
        mbar_init(&a_pfull[b], 128);
      }
      mbar_init(a_done, 128);
    }
    if (dsm) {
      mbar_init(pb_ready, 4);
      mbar_init(pb_free, 4);
    }
    fence_barrier_init();
  }
  if (warp == 2 && lane == 0)
    for (int ph = 0; ph < p.n_phases; ++ph)
      if (p.ph[ph].kind == CHAIN_GEMM) tma_prefetch(&p.tm[ph]);
  if (warp == 1) tmem_alloc(tmem_slot, tcols);
  tc_fence_before();
  __syncthreads();
  if (dsm) cluster_sync_all();  // peers' barriers are initialised before any remote arrive
  tc_fence_after();
  if (threadIdx.x == 0) ctl(p, kMaxPhases - 1, 1);
  const uint32_t tmem = *tmem_slot;
  // attention: three 64-column score buffers at [192, 384), O at [384, 512) (the GEMM
  // accumulators [0, 2 BN) are only written by MMAs issued after the last PV)
  const uint32_t aS0 = tmem + 192, aO = tmem + 384;

  // attention item of this CTA: head h, key split sp -> key blocks [b0, b0 + nb) of 64
  auto attn_range = [&](const PhaseDev& A, int& h, int& sp, int& b0, int& nb) {
    h = c / A.aS;
    sp = c - h * A.aS;
    const int64_t nblk = A.a_nseg ? A.a_first[A.a_nseg] : (A.aP + A.M + 63) / 64;
    b0 = static_cast<int>(nblk * sp / A.aS);
    nb = static_cast<int>(nblk * (sp + 1) / A.aS) - b0;
  };

  // Work items of a GEMM phase: item i = (tile i / S, k-split i % S) with k-blocks
  // [j kbs / S, (j+1) kbs / S); CTA c takes items c, c + C, ...  S = 1 (tiles >= C/2):
  // every tile finishes inside one CTA, straight from TMEM.  S = 2 or 4 (few tiles: Wo,
  // W2): the S CTAs of a tile each park a partial and then finish 1/S of its token
  // columns from all S partials (one batch of loads, summed in split order).
  auto item_kb = [](const PhaseDev& P, int i, int& tile, int& kb0, int& kb1) {
    tile = i / P.S;
    const int j = i - tile * P.S;
    kb0 = j * P.kbs / P.S;
    kb1 = (j + 1) * P.kbs / P.S;
  };
  if (warp == 0) {
    // ---- W producer: never waits for a phase boundary ----
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();
      int it = 0, ab = 0, an = 0;  // weight stages issued; attention blocks / phases so far
      for (int ph = 0; ph < p.n_phases; ++ph) {
        const PhaseDev& P = p.ph[ph];
        if (P.kind == CHAIN_ATTN) {
          // attention loads (Q once, then the K/V blocks of this CTA's split) through the ring;
          // the weight stream resumes once this CTA's softmax no longer uses it
          if (c < P.items) {
            int h, sp, b0, nb;
            attn_range(P, h, sp, b0, nb);
            const CUtensorMap* tk = &p.tak[P.a_map];
            const CUtensorMap* tv = &p.tav[P.a_map];
            tma_prefetch(&p.tma[0]);
            if (P.a_nseg) {
              for (int sgi = 0; sgi < P.a_nseg; ++sgi) tma_prefetch(&p.tkv[sgi]);
            } else {
              tma_prefetch(tk);
              tma_prefetch(tv);
            }
            auto load_kv = [&](int j, int& sg) {
              const int g = ab + j;  // block sequence over the launch's attention phases
              const int s = g % AKV;
              mbar_wait(&a_kvempty[s], ((g / AKV) & 1) ^ 1);
              uint8_t* st = aKV + s * 32768;
              const int b = b0 + j;
              mbar_expect_tx(&a_kvfull[s], P.a_alibi ? 32768 + 256 : 32768);
              if (P.a_alibi)  // the block's 64 key positions into the (idle) LN-fold scratch
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(reinterpret_cast<int32_t*>(colsum) + s * 64)),
                    "l"(P.a_kpos + static_cast<int64_t>(b) * 64), "r"(256), "r"(smem_u32(&a_kvfull[s]))
                    : "memory");
              if (P.a_nseg) {
                while (b >= P.a_first[sg + 1]) ++sg;
                const int row = P.a_row0[sg] + (b - P.a_first[sg]) * 64;
                for (int a = 0; a < 2; ++a) {
                  tma_load_3d(st + a * 8192, &p.tkv[sg], &a_kvfull[s], h * 128 + a * 64, row, 2 * P.a_layer);
                  tma_load_3d(st + 16384 + a * 8192, &p.tkv[sg], &a_kvfull[s], h * 128 + a * 64, row,
                              2 * P.a_layer + 1);
                }
              } else {
                for (int a = 0; a < 2; ++a) {
                  tma_load_2d(st + a * 8192, tk, &a_kvfull[s], h * 128 + a * 64, b * 64);
                  tma_load_2d(st + 16384 + a * 8192, tv, &a_kvfull[s], h * 128 + a * 64, b * 64);
                }
              }
            };
            if (ph > 0)  // the K/V stages overwrite the ring: every weight stage issued so far consumed
              for (int k = 0; k < STAGES; ++k) mbar_wait(&empty[(it + k) % STAGES], (((it + k) / STAGES) & 1) ^ 1);
            // Blocks whose keys the phase before does not write -- cached-module segments read in
            // place, or cache rows below P -- are loaded before waiting for it (no ALiBi: its key
            // positions go through the LN scratch the phase before may still use)
            int pre = 0, sg = 0;
            if (!P.a_alibi) {
              const int indep = P.a_nseg ? P.a_first[P.a_nseg - 1] : static_cast<int>(P.aP / 64);
              pre = max(0, min(min(indep - b0, nb), AKV));
            }
            for (int j = 0; j < pre; ++j) load_kv(j, sg);
            if (ph == 0) {
              pdl_wait();  // Q and the new K/V rows come from the previous chain's QKV phase
            } else {
              grid_wait(p, ph);  // ... or from this launch's QKV phase
              fence_proxy_async_global();
            }
            mbar_expect_tx(a_qfull, 32768);
            for (int a = 0; a < 2; ++a)  // 64-row boxes: rows [0, 64) twice (dup) or [0, 128)
              for (int hh = 0; hh < 2; ++hh)
                tma_load_2d(aQ + a * 16384 + hh * 8192, &p.tma[0], a_qfull, h * 128 + a * 64, P.adup ? 0 : 64 * hh);
            for (int j = pre; j < nb; ++j) load_kv(j, sg);
            ab += nb;
            mbar_wait(a_done, an & 1);
          }
          ++an;
          ctl(p, ph, 3);
          continue;
        }
        if (P.kind != CHAIN_GEMM) continue;
        for (int i = c; i < P.items; i += C) {
          int tile, kb0, kb1;
          item_kb(P, i, tile, kb0, kb1);
          for (int kb = kb0; kb < kb1; ++kb, ++it) {
            const int s = it % STAGES;
            mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
            mbar_expect_tx(&full[s], S::kStage);
            // packed tiles of one 128-row block are contiguous along K
            bulk_load(smem + s * S::kStage, P.w + (static_cast<int64_t>(tile) * P.kbs + kb) * kWTileC, kWTileC,
                      &full[s], pol_w);
          }
        }
        ctl(p, ph, 3);
      }
    }
  } else if (warp == 2) {
    // ---- X producer: activation tiles, after the phase's inputs are published ----
    if (elect_one()) {
      const uint64_t pol_x = policy_evict_last();  // re-read by every CTA
      int it = 0;
      for (int ph = 0; ph < p.n_phases; ++ph) {
        const PhaseDev& P = p.ph[ph];
        if (P.kind != CHAIN_GEMM || c >= P.items) continue;
        ctl(p, ph, 6);
        if (ph == 0) pdl_wait();
        else grid_wait(p, ph);
        ctl(p, ph, 7);
        fence_proxy_async_global();  // generic-proxy stores of other CTAs -> our TMA reads
        ctl(p, ph, 0);
        for (int i = c; i < P.items; i += C) {
          int tile, kb0, kb1;
          item_kb(P, i, tile, kb0, kb1);
          for (int kb = kb0; kb < kb1; ++kb, ++it) {
            const int s = it % STAGES;
            mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
            tma_load_2d_hint(smem + s * S::kStage + kWTileC, &p.tm[ph], &full[s], kb * 64, 0, pol_x);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: one accumulator per item ----
    if (elect_one()) {
      // attention phase: S_j = Q K_j^T (M=128, N=64, K=128) into one of three score buffers,
      // O += P_j V_j (P from TMEM, V MN-major) accumulated in TMEM
      int ab = 0, aw = 0;  // attention blocks / phases with work so far (barrier phases)
      auto attn_mma = [&](const PhaseDev& A, int ph) {
        int h, sp, b0, nb;
        attn_range(A, h, sp, b0, nb);
        constexpr uint32_t idS = idesc_bf16(128, 64);
        constexpr uint32_t idO = idesc_bf16(128, 128, false, true);
        const uint32_t q_addr = smem_u32(aQ);
        mbar_wait(a_qfull, aw & 1);
        ++aw;
        long long kv_wait = 0, p_wait = 0;
        auto issue_qk = [&](int j) {
          const int g = ab + j, s = g % AKV;
          const long long t0 = p.tl ? clock64() : 0;
          mbar_wait(&a_kvfull[s], (g / AKV) & 1);
          if (p.tl) kv_wait += clock64() - t0;
          tc_fence_after();
          const uint32_t k_addr = smem_u32(aKV + s * 32768);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            umma_bf16(aS0 + (g % 3) * 64, sw128_kmajor_desc(q_addr + (k >> 2) * 16384 + (k & 3) * 32),
                      sw128_kmajor_desc(k_addr + (k >> 2) * 8192 + (k & 3) * 32), idS, k > 0 ? 1u : 0u);
          umma_commit(&a_sfull[g % 3]);
        };
        issue_qk(0);
        if (nb > 1) issue_qk(1);
        for (int j = 0; j < nb; ++j) {
          const int g = ab + j;
          const long long t1 = p.tl ? clock64() : 0;
          mbar_wait(&a_pfull[g % 3], (g / 3) & 1);
          if (p.tl) p_wait += clock64() - t1;
          tc_fence_after();
          const uint32_t v_addr = smem_u32(aKV + (g % AKV) * 32768 + 16384);
          // P(j) is the A operand straight from TMEM: packed bf16 over the first 32 columns of
          // its score buffer (S(j + 3) reuses the buffer; it is issued after this PV)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16_ts(aO, aS0 + (g % 3) * 64 + k * 8, sw128_mnmajor_desc(v_addr + k * 2048, 8192, 1024), idO,
                         (j > 0 || k > 0) ? 1u : 0u);
          umma_commit(&a_pvdone[g % 3]);
          umma_commit(&a_kvempty[g % AKV]);
          // S(j + 2) into the buffer of P(j - 1), whose PV was issued an iteration ago
          if (j + 2 < nb) issue_qk(j + 2);
        }
        ab += nb;
        ctl(p, ph, 1);
        ctl_val(p, ph, 14, kv_wait);  // MMA thread: cycles waiting for K/V blocks, for P
        ctl_val(p, ph, 15, p_wait);
      };
      constexpr uint32_t idesc = idesc_bf16(128, BN);
      int it = 0, seg = 0;
      for (int ph = 0; ph < p.n_phases; ++ph) {
        const PhaseDev& P = p.ph[ph];
        if (P.kind == CHAIN_ATTN && c < P.items) attn_mma(P, ph);
        if (P.kind != CHAIN_GEMM) continue;
        for (int i = c; i < P.items; i += C, ++seg) {
          int tile, kb0, kb1;
          item_kb(P, i, tile, kb0, kb1);
          const int buf = seg & 1;
          mbar_wait(&acc_empty[buf], ((seg >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t acc = tmem + buf * BN;
          for (int kb = kb0; kb < kb1; ++kb, ++it) {
            const int s = it % STAGES;
            mbar_wait(&full[s], (it / STAGES) & 1);
            tc_fence_after();
            const uint32_t wa = smem_u32(smem + s * S::kStage), xb = wa + kWTileC;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(acc, sw128_kmajor_desc(wa + k * 32), sw128_kmajor_desc(xb + k * 32), idesc,
                        (kb > kb0 || k > 0) ? 1u : 0u);
            umma_commit(&empty[s]);
          }
          umma_commit(&acc_full[buf]);
        }
        ctl(p, ph, 1);
      }
    }
  } else {
    // ---- epilogue warps 3..6 (TMEM lane quadrant = warp % 4) ----
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int et = threadIdx.x - 96;
    const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
    float v[16];
    int seg = 0;
    int ab = 0;            // attention blocks so far (buffer / barrier phases)
    uint32_t pb_uses = 0;  // dsm: completed uses of this CTA's exchange buffer
    // dsm helpers: the S CTAs [g0, g0 + S) of a group sit in one cluster of 4 (C % 4 == 0,
    // S in {1, 2, 4}, groups aligned), so a member's cluster rank is its index & 3
    // One remote arrive per (CTA, member): bar.sync orders the 128 epilogue threads' buffer
    // writes / reads before thread u's cluster-scope release (128 remote arrivals per barrier,
    // one per thread, serialised on the barrier word: +2 us per exchange).  The wait is one
    // acquiring thread followed by bar.sync.
    auto pb_signal = [&](uint64_t* bar, int g0, int S_) {
      named_bar(1, 128);
      if (et < S_) mbar_arrive_cluster(mapa_shared(smem_u32(bar), (g0 + et) & 3), 4 / S_);
    };
    auto pb_wait = [&](uint64_t* bar, uint32_t parity) {
      if (et == 0) mbar_wait_cluster(bar, parity);
      named_bar(1, 128);
    };
    for (int ph = 0; ph < p.n_phases; ++ph) {
      const PhaseDev& P = p.ph[ph];
      if (ph == 0) {
        pdl_wait();
        if (et == 0) ctl(p, kMaxPhases - 1, 2);
      } else {
        if (et == 0) grid_wait(p, ph);
        named_bar(1, 128);
        if (ph == 1) pdl_trigger();  // every CTA is resident: dependents may launch
      }
      if (P.kind == CHAIN_LN) {
        for (int64_t r = c; r < P.M; r += C) ln_row(P, r, red, et);
      } else if (P.kind == CHAIN_ATTN) {
        // ---- softmax: one thread per TMEM lane (reference model.cpp:401-427, causal by
        // sequence order: query i sees keys j <= P + i).  n <= 64 ("dup"): the Q tile holds
        // the n queries twice, lanes [0, 64) take keys [0, 32) of every block and lanes
        // [64, 128) keys [32, 64) -- all four warps work, each on half the columns, and the
        // two halves of a query merge like two more key splits ----
        const int epoch = p.epoch0 + ph;
        int h = 0, sp = 0, b0 = 0, nb = 0;
        if (c < P.items) attn_range(P, h, sp, b0, nb);
        const int64_t n_ = P.M;
        const bool dup = P.adup;
        const int qi = dup ? (row & 63) : row;  // query of this lane
        float m = -INFINITY, l = 0.f;
        const bool live = (dup ? ((q & 1) * 32) : (q * 32)) < n_;  // else the warp keeps the protocol only
        if (et == 0) ctl(p, ph, 0);
        // ALiBi in raw score units (the exponent scale is log2(e)/sqrt(128)):
        //   s + slope sqrt(128) (pos_key - pos_query)
        const bool alibi = P.a_alibi != nullptr;
        const int32_t qpos = alibi && c < P.items && qi < n_ ? P.a_qpos[qi] : 0;
        const float slope_raw = alibi && c < P.items ? P.a_alibi[h] * 11.313708498984761f : 0.f;
        long long sfull_wait = 0;
        const long long tsm0 = p.tl ? clock64() : 0;
        auto blocks = [&](auto ncols) {
          constexpr int NC = decltype(ncols)::value;  // score columns per lane: 64, or 32 (dup)
          const int hi = NC == 32 ? (row >> 6) : 0;     // dup: which half of each block's keys
          const int c0 = hi * 32;
          const float ascale = P.ascale, thr = kRescaleThreshold / ascale;
          // key-block visibility in 32-bit arithmetic (positions < 2^31, checked on the host):
          // lim = last visible key of the block relative to this lane's first column
          //     = vis - 64 b, vis re-derived only when the block enters a new segment
          // contiguous: key j visible iff j <= P + qi; zero-copy: a prefix segment's rows are
          // all visible (its padding is not), the tail is visible up to tail_vis + qi
          int sg = -1, seg_next = P.a_nseg ? 0 : 0x7fffffff;
          int vis = static_cast<int>(P.aP) + qi - c0;
          for (int it = 0; it < nb; ++it) {
            const int b = b0 + it;
            const int g = ab + it;  // block sequence over the launch's attention phases
            if (b >= seg_next) {
              do ++sg;
              while (b >= P.a_first[sg + 1]);
              const int seg_first = P.a_first[sg];
              seg_next = P.a_first[sg + 1];
              vis = (sg == P.a_nseg - 1 ? P.a_tail_vis + qi : P.a_rows[sg] - 1) + seg_first * 64 - c0;
            }
            const int lim = vis - b * 64;
            if (!live) {
              // S(it) was issued after p_full(it - 2) completed: arriving after it keeps this
              // warp's arrival out of block it - 3's phase of the same barrier
              mbar_wait(&a_sfull[g % 3], (g / 3) & 1);
              mbar_arrive(&a_pfull[g % 3]);
              continue;
            }
            const long long tw0 = p.tl ? clock64() : 0;
            mbar_wait(&a_sfull[g % 3], (g / 3) & 1);
            if (p.tl) sfull_wait += clock64() - tw0;
            tc_fence_after();
            float sv[NC];
            {
              uint32_t raw[NC];
#pragma unroll
              for (int x = 0; x < NC; x += 16) tmem_ld16_nowait(aS0 + (g % 3) * 64 + lane_off + c0 + x, raw + x);
              tmem_wait_ld();
#pragma unroll
              for (int x = 0; x < NC; ++x) sv[x] = __uint_as_float(raw[x]);
            }
            if (alibi) {
              mbar_wait(&a_kvfull[g % AKV], (g / AKV) & 1);  // the positions' bulk copy (complete)
              const int4* kp = reinterpret_cast<const int4*>(reinterpret_cast<const int32_t*>(colsum) +
                                                             (g % AKV) * 64 + c0);
#pragma unroll
              for (int x = 0; x < NC; x += 4) {
                const int4 k4 = kp[x >> 2];
                sv[x] = fmaf(slope_raw, static_cast<float>(k4.x - qpos), sv[x]);
                sv[x + 1] = fmaf(slope_raw, static_cast<float>(k4.y - qpos), sv[x + 1]);
                sv[x + 2] = fmaf(slope_raw, static_cast<float>(k4.z - qpos), sv[x + 2]);
                sv[x + 3] = fmaf(slope_raw, static_cast<float>(k4.w - qpos), sv[x + 3]);
              }
            }
            if (NC - 1 > lim) {
#pragma unroll
              for (int x = 0; x < NC; ++x)
                if (x > lim) sv[x] = -INFINITY;
            }
            // exponentials against the running max, computed alongside the block max (they do
            // not wait for it); only when some lane's max grows past the lazy-rescale threshold
            // (the first block, rarely later) are they recomputed against the new max
            float bs[4];
            uint32_t packed[NC / 2];
            auto expo = [&](float mb) {
#pragma unroll
              for (int x = 0; x < 4; ++x) bs[x] = 0.f;
#pragma unroll
              for (int x = 0; x < NC; x += 2) {
                const float p0 = fast_exp2(fmaf(sv[x], ascale, -mb));
                const float p1 = fast_exp2(fmaf(sv[x + 1], ascale, -mb));
                bs[(x >> 1) & 3] += p0 + p1;
                __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
                packed[x >> 1] = *reinterpret_cast<uint32_t*>(&b2);
              }
            };
            expo(m == -INFINITY ? 0.f : m * ascale);
            float mx[8];
#pragma unroll
            for (int x = 0; x < 8; ++x) mx[x] = sv[x];
#pragma unroll
            for (int x = 8; x < NC; ++x) mx[x & 7] = fmaxf(mx[x & 7], sv[x]);
#pragma unroll
            for (int w = 4; w; w >>= 1)
#pragma unroll
              for (int x = 0; x < w; ++x) mx[x] = fmaxf(mx[x], mx[x + w]);
            const float bm = mx[0];
            const bool grow = bm > m + thr || (m == -INFINITY && bm > -INFINITY);
            if (__any_sync(0xffffffffu, grow)) {
              if (it > 0) {
                mbar_wait(&a_pvdone[(g - 1) % 3], ((g - 1) / 3) & 1);
                tc_fence_after();
                const float f = grow ? fast_exp2((m - bm) * ascale) : 1.f;
#pragma unroll 1
                for (int x = 0; x < 128; x += 16) {
                  float ov[16];
                  tmem_ld16(aO + lane_off + x, ov);
#pragma unroll
                  for (int y = 0; y < 16; ++y) ov[y] *= f;
                  tmem_st16(aO + lane_off + x, ov);
                }
                tmem_st_wait();
              }
              if (grow) {
                l *= fast_exp2((m - bm) * ascale);
                m = bm;
              }
              expo(m == -INFINITY ? 0.f : m * ascale);
            }
            l += (bs[0] + bs[1]) + (bs[2] + bs[3]);
            // P row into TMEM over the first 32 columns of the score buffer (64 bf16 keys; dup:
            // this lane's half of the keys, zeros in the other half)
            {
              const uint32_t pa = aS0 + (g % 3) * 64 + lane_off;
              if constexpr (NC == 64) {
                tmem_st16u(pa, packed);
                tmem_st16u(pa + 16, packed + 16);
              } else {
                const uint32_t z[16] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
                tmem_st16u(pa + 16 * hi, packed);
                tmem_st16u(pa + 16 * (1 - hi), z);
              }
              tmem_st_wait();
            }
            tc_fence_before();
            mbar_arrive(&a_pfull[g % 3]);  // after block it-3's phase: S(it) needed p_full(it-2)
          }
        };
        if (dup) blocks(std::integral_constant<int, 32>{});
        else blocks(std::integral_constant<int, 64>{});
        if (et == 0) {  // softmax loop: total cycles, cycles waiting for S
          ctl_val(p, ph, 12, p.tl ? clock64() - tsm0 : 0);
          ctl_val(p, ph, 13, sfull_wait);
        }
        // one partial per (query, split): the dup halves combine first through shared memory
        // (the K/V stages are idle once the last PV completed); a single split writes O
        const int nparts = P.aS;
        const bool out_lane = dup ? row < 64 : true;  // lanes that own a query's result
        // dsm (n <= 64): the split partials meet in the cluster's exchange buffers -- one
        // DSMEM round trip instead of global partials + release flags + L2 polls (~7 us of
        // the phase tail under a saturated memory system)
        const bool adsm = dsm && dup && nparts > 1 && c < P.items;
        float2* pbml = reinterpret_cast<float2*>(pb + 64 * S::kPbLd);
        float* part = P.apart + (static_cast<int64_t>(c) * 128 + qi) * 128;
        float2* ml = reinterpret_cast<float2*>(P.apart + static_cast<int64_t>(P.items) * 128 * 128);
        // a_done hands the ring to the W producer (the next phase's weights).  It is free once
        // the last PV completed -- the dup halves combine in the exchange buffer (Q, parked
        // there, is dead) -- except on the global-partials path, where a split CTA publishes
        // its partial first (with the weight prefetch in flight its flag became visible ~2 us
        // later, tools/chain_ab.py per-CTA attention events)
        const bool merge = c < P.items && nparts > 1;
        const bool early = (!merge || adsm) && (S::kPB > 0 || !dup);
        if (nb > 0) {
          mbar_wait(&a_pvdone[(ab + nb - 1) % 3], ((ab + nb - 1) / 3) & 1);
          tc_fence_after();
          ab += nb;
        }
        if (early) mbar_arrive(a_done);
        long long tpk0 = 0, tld = 0;
        if (nb > 0) {
          constexpr int kXld = 132;  // padded fp32 row (= S::kPbLd: a lane reads its dup partner's
                                     // row, then parks its own result over it, in order)
          float* xo = S::kPB > 0 ? pb : reinterpret_cast<float*>(aKV);
          float2* xml = reinterpret_cast<float2*>(xo + 64 * kXld);
          float w0 = 1.f, w1 = 0.f;
          // tcgen05.ld is warp-collective: lane conditions only guard the memory operations
          if (dup) {
            if (row >= 64) {
#pragma unroll 1
              for (int x = 0; x < 128; x += 32) {
                uint32_t ov[32];
                tmem_ld16_nowait(aO + lane_off + x, ov);
                tmem_ld16_nowait(aO + lane_off + x + 16, ov + 16);
                tmem_wait_ld();
                if (qi < n_)
#pragma unroll
                  for (int y = 0; y < 32; y += 4)
                    *reinterpret_cast<float4*>(xo + qi * kXld + x + y) =
                        make_float4(__uint_as_float(ov[y]), __uint_as_float(ov[y + 1]), __uint_as_float(ov[y + 2]),
                                    __uint_as_float(ov[y + 3]));
              }
              if (qi < n_) xml[qi] = make_float2(m, l);
            }
            named_bar(1, 128);
            if (row < 64 && qi < n_) {
              const float2 o = xml[qi];
              const float M = l > 0.f && o.y > 0.f ? fmaxf(m, o.x) : (l > 0.f ? m : o.x);
              w0 = l > 0.f ? fast_exp2((m - M) * P.ascale) : 0.f;
              w1 = o.y > 0.f ? fast_exp2((o.x - M) * P.ascale) : 0.f;
              l = w0 * l + w1 * o.y;
              m = M;
            }
          }
          if (et == 32) ctl(p, ph, 9);  // a result lane (warp quadrant 0): dup halves combined
          tpk0 = p.tl ? clock64() : 0;
          if (out_lane) {
            const float inv = nparts == 1 ? 1.f / l : 1.f;
            __nv_bfloat16* dst = P.aout + qi * P.a_d + h * 128;
            // two 16-column TMEM loads in flight per wait
#pragma unroll 1
            for (int x2 = 0; x2 < 128; x2 += 32) {
              float ov2[32];
              {
                uint32_t raw[32];
                if (p.tl && x2 == 32) tld = clock64() - tpk0;  // first iteration (cold code)
                tmem_ld16_nowait(aO + lane_off + x2, raw);
                tmem_ld16_nowait(aO + lane_off + x2 + 16, raw + 16);
                tmem_wait_ld();
#pragma unroll
                for (int y = 0; y < 32; ++y) ov2[y] = __uint_as_float(raw[y]);
              }
              if (qi >= n_) continue;
#pragma unroll
              for (int hx = 0; hx < 2; ++hx) {
                const int x = x2 + 16 * hx;
                float* ov = ov2 + 16 * hx;
                if (dup) {
#pragma unroll
                  for (int y = 0; y < 16; y += 4) {
                    const float4 o4 = *reinterpret_cast<const float4*>(xo + qi * kXld + x + y);
                    ov[y] = w0 * ov[y] + w1 * o4.x;
                    ov[y + 1] = w0 * ov[y + 1] + w1 * o4.y;
                    ov[y + 2] = w0 * ov[y + 2] + w1 * o4.z;
                    ov[y + 3] = w0 * ov[y + 3] + w1 * o4.w;
                  }
                }
                if (nparts == 1) {
                  uint4 w2[2];
                  __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(w2);
#pragma unroll
                  for (int y = 0; y < 8; ++y) b[y] = __floats2bfloat162_rn(ov[2 * y] * inv, ov[2 * y + 1] * inv);
                  *reinterpret_cast<uint4*>(dst + x) = w2[0];
                  *reinterpret_cast<uint4*>(dst + x + 8) = w2[1];
                } else if (adsm) {  // park O / l (fp32) in this CTA's exchange buffer
                  const float il = l > 0.f ? 1.f / l : 0.f;
                  float* pr = pb + qi * S::kPbLd + x;
#pragma unroll
                  for (int y = 0; y < 16; y += 4)
                    *reinterpret_cast<float4*>(pr + y) =
                        make_float4(ov[y] * il, ov[y + 1] * il, ov[y + 2] * il, ov[y + 3] * il);
                } else {  // park the normalised O row in fp16 (O / l: |values| <= max |V|) for the merge
                  const float il = l > 0.f ? 1.f / l : 0.f;
                  uint32_t hw[8];
#pragma unroll
                  for (int y = 0; y < 8; ++y) {
                    const __half2 t = __floats2half2_rn(ov[2 * y] * il, ov[2 * y + 1] * il);
                    hw[y] = *reinterpret_cast<const uint32_t*>(&t);
                  }
                  __half* ph = reinterpret_cast<__half*>(part) + x;  // row stride stays 128 floats
                  __stcg(reinterpret_cast<uint4*>(ph), make_uint4(hw[0], hw[1], hw[2], hw[3]));
                  __stcg(reinterpret_cast<uint4*>(ph + 8), make_uint4(hw[4], hw[5], hw[6], hw[7]));
                }
              }
            }
            if (nparts > 1 && qi < n_) {
              if (adsm) pbml[qi] = make_float2(m, l);
              else __stcg(ml + static_cast<int64_t>(c) * 128 + qi, make_float2(m, l));
            }
          }
        }
        if (et == 32) {
          ctl(p, ph, 10);
          ctl_val(p, ph, 6, p.tl ? clock64() - tpk0 : 0);  // cycles of the output / park loop
          ctl_val(p, ph, 7, tld);
        }
        tc_fence_before();
        if (et == 0) ctl(p, ph, 4);
        if (!early && !merge) mbar_arrive(a_done);
        if (adsm) {
          // every epilogue thread releases its parked rows to the head's S CTAs, then the CTA
          // merges queries {sp, sp + S, ...} reading all S buffers (split order: deterministic)
          const int base = h * P.aS;
          pb_signal(pb_ready, base, nparts);
          if (!early) mbar_arrive(a_done);
          if (et == 0) ctl(p, ph, 8);
          pb_wait(pb_ready, pb_uses & 1);
          if (et == 0) ctl(p, ph, 5);
          const long long tmg0 = p.tl ? clock64() : 0;
          const int x0 = (et & 7) * 4;  // dims x0 + 32 y + [0, 4): 8 threads read 128 contiguous bytes
          for (int64_t r2 = sp + static_cast<int64_t>(et >> 3) * P.aS; r2 < n_; r2 += 16 * P.aS) {
            // every remote load issued before the first use (member indices past S re-read
            // member 0 and get weight 0)
            float ms[4], ls[4], f[4][16];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int rk = (base + (u < nparts ? u : 0)) & 3;
              const uint32_t a = mapa_shared(smem_u32(pbml + r2), rk);
              asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(ms[u]), "=f"(ls[u]) : "r"(a) : "memory");
              const uint32_t b = mapa_shared(smem_u32(pb + r2 * S::kPbLd + x0), rk);
#pragma unroll
              for (int y = 0; y < 4; ++y) ld_dsmem_v4(b + 128 * y, f[u] + 4 * y);
            }
            float M = -INFINITY;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (u < nparts && ls[u] > 0.f) M = fmaxf(M, ms[u]);
            float den = 0.f, acc[16];
#pragma unroll
            for (int x = 0; x < 16; ++x) acc[x] = 0.f;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float wl = (u < nparts && ls[u] > 0.f) ? fast_exp2((ms[u] - M) * P.ascale) * ls[u] : 0.f;
              den += wl;
#pragma unroll
              for (int x = 0; x < 16; ++x) acc[x] = fmaf(wl, f[u][x], acc[x]);
            }
            const float inv = 1.f / den;
            __nv_bfloat16* dst = P.aout + r2 * P.a_d + h * 128 + x0;
#pragma unroll
            for (int y = 0; y < 4; ++y) {
              const __nv_bfloat162 lo = __floats2bfloat162_rn(acc[4 * y] * inv, acc[4 * y + 1] * inv);
              const __nv_bfloat162 hi = __floats2bfloat162_rn(acc[4 * y + 2] * inv, acc[4 * y + 3] * inv);
              *reinterpret_cast<uint2*>(dst + 32 * y) =
                  make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
            }
          }
          if (et == 0) {
            ctl(p, ph, 11);
            (void)tmg0;
          }
          pb_signal(pb_free, base, nparts);
          ++pb_uses;
        } else if (merge) {
          // the S split CTAs of head h each merge queries {sp, sp + S, ...} of all S partials
          // in split order (deterministic):
          //   O = sum_s w_s O_s / sum_s w_s l_s,  w_s = 2^((m_s - M) scale),  M = max_s m_s
          named_bar(1, 128);
          if (et == 0) {
            st_release(p.flags + c, epoch);
            ctl(p, ph, 8);
          }
          mbar_arrive(a_done);
          const int base = h * P.aS;
          if (et < P.aS)
            for (uint32_t spins = 0; ld_relaxed(p.flags + base + et) < epoch;) {
              __nanosleep(32);
              if (++spins == (1u << 25)) wait_timeout("chain attention split flag", p.flags + base + et, epoch);
            }
          fence_acquire_gpu();
          named_bar(1, 128);
          if (et == 0) ctl(p, ph, 5);
          const int x0 = (et & 7) * 16;
          auto prow_of = [&](int u, int64_t r2) { return static_cast<int64_t>(base + u) * 128 + r2; };
          for (int64_t r2 = sp + static_cast<int64_t>(et >> 3) * P.aS; r2 < n_; r2 += 16 * P.aS) {
            float ms[16], ls[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              float2 v2 = make_float2(-INFINITY, 0.f);
              if (u < nparts) v2 = __ldcg(ml + prow_of(u, r2));
              ms[u] = v2.x;
              ls[u] = v2.y;
            }
            float M = -INFINITY;
#pragma unroll
            for (int u = 0; u < 16; ++u)
              if (u < nparts && ls[u] > 0.f) M = fmaxf(M, ms[u]);
            float den = 0.f, acc[16];
#pragma unroll
            for (int x = 0; x < 16; ++x) acc[x] = 0.f;
#pragma unroll
            for (int g = 0; g < 16; g += 4) {
              if (g >= nparts) break;
              uint4 f[4][2];  // 16 fp16 values of O / l per partial
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (g + u < nparts) {
                  const uint4* src =
                      reinterpret_cast<const uint4*>(reinterpret_cast<const __half*>(P.apart + prow_of(g + u, r2) * 128) + x0);
                  f[u][0] = __ldcg(src);
                  f[u][1] = __ldcg(src + 1);
                }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int uu = g + u;
                if (uu >= nparts || !(ls[uu] > 0.f)) continue;
                const float wl = fast_exp2((ms[uu] - M) * P.ascale) * ls[uu];  // weight of O_s / l_s
                den += wl;
                const __half2* hv = reinterpret_cast<const __half2*>(&f[u][0]);
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                  const float2 t = __half22float2(hv[x]);
                  acc[2 * x] += wl * t.x;
                  acc[2 * x + 1] += wl * t.y;
                }
              }
            }
            const float inv = 1.f / den;
            __nv_bfloat16* dst = P.aout + r2 * P.a_d + h * 128 + x0;
            uint4 w2[2];
            __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(w2);
#pragma unroll
            for (int y = 0; y < 8; ++y) b[y] = __floats2bfloat162_rn(acc[2 * y] * inv, acc[2 * y + 1] * inv);
            *reinterpret_cast<uint4*>(dst) = w2[0];
            *reinterpret_cast<uint4*>(dst + 8) = w2[1];
          }
        }
      } else {
        const Epilogue& e = P.e;
        const int64_t M = P.M;
        const int Mc = static_cast<int>(M < BN ? M : BN);
        const float2* ln = nullptr;
        if (P.stats_in) {
          // {mean, rstd} per token from the residual phase's per-tile partial sums (fp64, tile order)
          if (et < Mc) {
            double s1 = 0, s2 = 0;
            const float2* src = reinterpret_cast<const float2*>(P.stats_in) + P.stats_row0 + et;
#pragma unroll 1
            for (int t0 = 0; t0 < P.stats_tiles; t0 += 8) {  // 8 independent loads per round trip
              float2 st[8];
#pragma unroll
              for (int u = 0; u < 8; ++u)
                st[u] = t0 + u < P.stats_tiles ? __ldcg(src + static_cast<int64_t>(t0 + u) * P.stats_ld)
                                               : make_float2(0.f, 0.f);
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                s1 += st[u].x;
                s2 += st[u].y;
              }
            }
            const double mean = s1 / P.ln_dim, var = fmax(s2 / P.ln_dim - mean * mean, 0.0);
            lnst[et] = make_float2(static_cast<float>(mean), static_cast<float>(1.0 / sqrt(var + 1e-5)));
          }
          named_bar(1, 128);
          ln = lnst;
        }
        // column sums of the new residual of one 16-token chunk -> stats_out[tile][m]
        // (transposed through smem: each thread parks its 16 values, then 8 threads per
        // token sum 16 columns each and combine with 3 shuffles)
        auto stats_chunk = [&](int tile, int64_t m0, int64_t lim, bool nost = false) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            colsum[j * 128 + row] = v[j];
            colsum[2048 + j * 128 + row] = v[j] * v[j];
          }
          named_bar(1, 128);
          const int j = et >> 3, g = (et & 7) * 16;
          float a = 0.f, b = 0.f;
#pragma unroll
          for (int x = 0; x < 16; ++x) {
            a += colsum[j * 128 + g + x];
            b += colsum[2048 + j * 128 + g + x];
          }
#pragma unroll
          for (int o = 4; o; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
          }
          if ((et & 7) == 0 && m0 + j < lim && !nost)
            reinterpret_cast<float2*>(P.stats_out)[static_cast<int64_t>(tile) * P.stats_ld + m0 + j] = make_float2(a, b);
          named_bar(1, 128);
        };
        const int epoch = p.epoch0 + ph;
        // [items][128][BN] fp16 partials (a K-split partial of 1024-4096 products; fp16's
        // 2^-11 is 8x finer than the bf16 operands' rounding, and half the bytes shorten the
        // publish -> flag -> reload round trip at every split phase end)
        __half* ws = reinterpret_cast<__half*>(p.ws + (ph & 1) * p.ws_half);
        const bool rope_stage = e.kind == EPI_QKV && e.rope && e.rope_tab != nullptr && P.S == 1;
        for (int i = c; i < P.items; i += C, ++seg) {
          const int tile = i / P.S, j = i - tile * P.S;
          const int n = tile * 128 + row;
          const int buf = seg & 1;
          const uint32_t acc = tmem + buf * BN + lane_off;
          EpiPre cur, nxt;
          // RoPE rows of every chunk into TMEM while the weights stream (per-chunk loads at
          // epilogue time each cost a loaded-L2 round trip, ~1 us: 4 of them per QKV tile)
          const bool rot = rope_stage && (tile * 128) / e.d < 2;  // Q and K tiles (warp-uniform)
          if (rot) {
            const float4* src = reinterpret_cast<const float4*>(e.rope_tab + (((n % e.d) % e.head_dim) >> 1) * e.rope_ld);
            const int Mr = (Mc + 15) & ~15;  // rope_ld leaves >= 16 tokens of slack
#pragma unroll 1
            for (int cc = 0; cc < Mc; cc += 32) {
              float4 t[16];
#pragma unroll
              for (int u = 0; u < 16; ++u) t[u] = cc + 2 * u < Mr ? __ldg(src + (cc >> 1) + u) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
              for (int h2 = 0; h2 < 2; ++h2) {
                if (cc + 16 * h2 >= Mc) break;  // warp-uniform
                float cs[16], sn[16];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                  cs[2 * u] = t[8 * h2 + u].x;
                  sn[2 * u] = t[8 * h2 + u].y;
                  cs[2 * u + 1] = t[8 * h2 + u].z;
                  sn[2 * u + 1] = t[8 * h2 + u].w;
                }
                tmem_st16(tmem + 256 + lane_off + cc + 16 * h2, cs);
                tmem_st16(tmem + 384 + lane_off + cc + 16 * h2, sn);
              }
            }
            tmem_st_wait();
          }
          // bf16 outputs (QKV, GELU) of <= 64 tokens: stage the 128 x Mc tile in shared memory
          // (the LN-fold scratch, idle in these phases) and store whole 256-byte token rows --
          // 8 16-byte stores per thread instead of 64 scattered 2-byte ones
          const bool tstore = P.S == 1 && (e.kind == EPI_QKV || e.kind == EPI_GELU) && Mc <= 64 && !P.stats_out;
          __nv_bfloat16* T = reinterpret_cast<__nv_bfloat16*>(colsum);  // [64 tokens][128 rows]
          // the lean path stages <= 64 tokens at a time in T: 65-128 tokens (configs[2]'s 128-token
          // suffix) take two rounds
          const bool tlean = P.S == 1 && (e.kind == EPI_QKV || e.kind == EPI_GELU) && Mc <= 128 && !P.stats_out &&
                             (e.kind == EPI_GELU || !e.rope || rope_stage);
          if (tlean) {
            // Lean path: every per-row choice (GELU / RoPE / LN fold, the RoPE sign of an odd
            // column) is made once, outside the element loops, so the 16-token chunk is
            // straight-line code.  One epilogue warp per scheduler has no latency hiding: the
            // generic epi_chunk's per-element branches and divergence checks cost ~1 us per
            // chunk (QKV), this path a fraction of that.
            const bool gelu = e.kind == EPI_GELU;
            const float lnw = (ln && e.ln_wsum) ? __ldg(e.ln_wsum + n) : 0.f;
            const float sg = (n & 1) ? 1.f : -1.f;  // partner column n ^ 1 in lane ^ 1 (d even)
            __nv_bfloat16* base;
            int64_t ld;
            const int64_t* off = nullptr;
            if (gelu) {
              base = static_cast<__nv_bfloat16*>(e.out) + static_cast<int64_t>(tile) * 128;
              ld = P.N;
            } else {
              const int sq = (tile * 128) / e.d, c0 = tile * 128 - sq * e.d;
              ld = e.d;
              if (sq == 0) {
                base = static_cast<__nv_bfloat16*>(e.q_out) + c0;
              } else {
                base = static_cast<__nv_bfloat16*>(sq == 1 ? e.k_out : e.v_out) + c0;
                if (e.kv_off) off = e.kv_off;
                else base += e.kv_row0 * e.d;
              }
            }
            // pass 0 ("dry", while the weights stream): the same code on whatever the
            // accumulator holds, no waits, arrivals or global stores -- it pulls the
            // epilogue's instructions into the instruction cache, so the real pass does not
            // fetch them from a saturated L2 once the accumulator is ready (W1: 4.3 -> 2.4 us)
#pragma unroll 1
            for (int pass = p.warm ? 0 : 1; pass < 2; ++pass) {
              const bool dry = pass == 0;
              if (!dry) {
                mbar_wait(&acc_full[buf], (seg >> 1) & 1);
                tc_fence_after();
                if (et == 0) ctl(p, ph, 4);
              }
#pragma unroll 1
              for (int h0 = 0; h0 < Mc; h0 += 64) {  // rounds of <= 64 tokens through T
                const int hn = Mc - h0 < 64 ? Mc - h0 : 64;
#pragma unroll 1
              for (int cc = h0; cc < h0 + hn; cc += 16) {
                uint32_t ra[16], rc[16], rs[16];
                tmem_ld16_nowait(acc + cc, ra);
                if (rot) {
                  tmem_ld16_nowait(tmem + 256 + lane_off + cc, rc);
                  tmem_ld16_nowait(tmem + 384 + lane_off + cc, rs);
                }
                tmem_wait_ld();
                float x[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) x[j] = __uint_as_float(ra[j]);
                if (et == 0 && !dry && cc < 32) ctl(p, ph, 12 + 2 * (cc >> 4));
                if (ln) {  // folded LayerNorm: rstd (acc - mean sum_k W); rows past M are never stored
#pragma unroll
                  for (int j = 0; j < 16; ++j) {
                    const float2 st = lnst[cc + j];
                    x[j] = st.y * fmaf(-st.x, lnw, x[j]);
                  }
                }
                if (gelu) {
#pragma unroll
                  for (int j = 0; j < 16; ++j) x[j] = gelu_bf16path(x[j]);
                } else if (rot) {
#pragma unroll
                  for (int j = 0; j < 16; ++j) {
                    const float pv = __shfl_xor_sync(0xffffffffu, x[j], 1);
                    x[j] = fmaf(sg * pv, __uint_as_float(rs[j]), x[j] * __uint_as_float(rc[j]));
                  }
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) T[(cc - h0 + j) * 128 + row] = __float2bfloat16_rn(x[j]);
                if (et == 0 && !dry && cc < 32) ctl(p, ph, 13 + 2 * (cc >> 4));
              }
              if (!dry && h0 + hn >= Mc) {  // the accumulator is fully read
                tc_fence_before();
                mbar_arrive(&acc_empty[buf]);
                if (et == 0) ctl(p, ph, 9);
              }
              named_bar(1, 128);
#pragma unroll
              for (int u = 0; u < 8; ++u) {  // hn * 16 <= 1024 16-byte pieces, 128 threads
                const int i = et + u * 128;
                if (i < hn * 16) {
                  const int m = i >> 4, q16 = i & 15;
                  const uint4 val = *reinterpret_cast<const uint4*>(T + m * 128 + q16 * 8);
                  __nv_bfloat16* dst = off ? base + off[h0 + m] + q16 * 8 : base + (h0 + m) * ld + q16 * 8;
                  if (!dry) *reinterpret_cast<uint4*>(dst) = val;
                }
              }
              if (h0 + hn < Mc) named_bar(1, 128);  // T is reused by the next round
              }
              if (et == 0 && !dry) ctl(p, ph, 10);
              named_bar(1, 128);  // T is reused by this CTA's next item
            }
            if (et == 0) ctl(p, ph, 5);
            continue;
          }
          if (P.S == 1) {
            epi_prefetch(e, n, P.N, 0, M, cur, !rope_stage);  // before the accumulator is ready
            mbar_wait(&acc_full[buf], (seg >> 1) & 1);
            tc_fence_after();
            if (et == 0) ctl(p, ph, 4);
#pragma unroll 1
            for (int cc = 0; cc < Mc; cc += 16) {
              if (rope_stage) {  // operands staged in TMEM; the LN-fold weight sum is per row
                if (rot) {
                  tmem_ld16(tmem + 256 + lane_off + cc, cur.a);
                  tmem_ld16(tmem + 384 + lane_off + cc, cur.b);
                }
              } else if (cc + 16 < Mc) {
                epi_prefetch(e, n, P.N, cc + 16, M, nxt, true, false);
                nxt.lnw = cur.lnw;
              }
              tmem_ld16(acc + cc, v);
              if (tstore) {
                epi_values(e, n, cc, M, v, cur, ln);
#pragma unroll
                for (int j = 0; j < 16; ++j) T[(cc + j) * 128 + row] = __float2bfloat16_rn(v[j]);
              } else {
                epi_chunk(e, n, P.N, cc, M, v, cur, ln);
                if (P.stats_out) stats_chunk(tile, cc, M);
              }
              if (!rope_stage) cur = nxt;
            }
            tc_fence_before();
            mbar_arrive(&acc_empty[buf]);
            if (et == 0) ctl(p, ph, 9);
            if (tstore) {
              named_bar(1, 128);
              __nv_bfloat16* base;
              int64_t ld;
              const int64_t* off = nullptr;
              if (e.kind == EPI_GELU) {
                base = static_cast<__nv_bfloat16*>(e.out) + static_cast<int64_t>(tile) * 128;
                ld = P.N;
              } else {
                const int sq = (tile * 128) / e.d, c0 = tile * 128 - sq * e.d;
                ld = e.d;
                if (sq == 0) {
                  base = static_cast<__nv_bfloat16*>(e.q_out) + c0;
                } else {
                  base = static_cast<__nv_bfloat16*>(sq == 1 ? e.k_out : e.v_out) + c0;
                  if (e.kv_off) off = e.kv_off;
                  else base += e.kv_row0 * e.d;
                }
              }
              for (int i = et; i < Mc * 16; i += 128) {
                const int m = i >> 4, q16 = i & 15;
                const uint4 val = *reinterpret_cast<const uint4*>(T + m * 128 + q16 * 8);
                __nv_bfloat16* dst = off ? base + off[m] + q16 * 8 : base + m * ld + q16 * 8;
                *reinterpret_cast<uint4*>(dst) = val;
              }
              if (et == 0) ctl(p, ph, 10);
              named_bar(1, 128);  // T is reused by this CTA's next item
            }
            if (et == 0) ctl(p, ph, 5);
            continue;
          }
          if (dsm) {
            // split tile, cluster path: park the fp32 partial in this CTA's exchange buffer,
            // release it to the tile's S CTAs (one cluster), then finish a 1/S slice of the
            // token columns reading all S buffers through DSMEM (split order: deterministic).
            // Pass 0 is a dry run while the weights stream (no waits, arrivals or stores): it
            // only warms the instruction cache, as for the S = 1 epilogue.
            // partial layout float4 [BN / 4][128 rows]: a warp's v4 access to one 4-token group
            // of 32 rows is 512 contiguous bytes (DSMEM reads coalesce into whole lines; a
            // row-per-thread layout made every 16-byte read its own remote transaction)
            const int g0 = tile * P.S;
            float4* pb4 = reinterpret_cast<float4*>(pb);
            const int Mr = (Mc + 3) & ~3;
            const int sw = ((Mr + P.S - 1) / P.S + 3) & ~3;
            const int s0 = j * sw, s1 = min(Mr, s0 + sw);
            const int64_t lim = min(static_cast<int64_t>(s1), M);
            // (only where the item streams long enough to hide it: Wo's 256 KB items are done
            // before a cold dry pass is, which then delayed the real one by ~5 us)
#pragma unroll 1
            for (int pass = (p.warm && P.kbs / P.S >= 32) ? 0 : 1; pass < 2; ++pass) {
              const bool dry = pass == 0;
              if (!dry) {
                // the residual slice (written a phase or a launch ago: an HBM / loaded-L2 round
                // trip of ~2 us) is read while the accumulator is still being filled
                if (s0 < lim) epi_prefetch(e, n, P.N, s0, lim, cur);
                mbar_wait(&acc_full[buf], (seg >> 1) & 1);
                tc_fence_after();
                if (et == 0) ctl(p, ph, 4);
                if (pb_uses > 0) pb_wait(pb_free, (pb_uses - 1) & 1);  // peers done with the last use
              }
#pragma unroll 1
              for (int cc = 0; cc < Mc; cc += 16) {
                tmem_ld16(acc + cc, v);
                if (!dry)
#pragma unroll
                  for (int x = 0; x < 16; x += 4) pb4[((cc + x) >> 2) * 128 + row] = make_float4(v[x], v[x + 1], v[x + 2], v[x + 3]);
              }
              if (!dry) {
                tc_fence_before();
                mbar_arrive(&acc_empty[buf]);
                pb_signal(pb_ready, g0, P.S);
              }
              if (dry && s0 < lim) epi_prefetch(e, n, P.N, s0, lim, cur);
              if (!dry) {
                pb_wait(pb_ready, pb_uses & 1);
                if (et == 0) ctl(p, ph, 5);
              }
#pragma unroll 1
              for (int m0 = s0; m0 < lim; m0 += 16) {
                // all 16 DSMEM loads in flight at once (a member index past S re-reads
                // member 0 and is not summed): a data-dependent loop bound serialised one
                // remote round trip per member
                float f[4][16];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const uint32_t a = mapa_shared(smem_u32(pb4 + (m0 >> 2) * 128 + row), (g0 + (u < P.S ? u : 0)) & 3);
#pragma unroll
                  for (int y = 0; y < 4; ++y) ld_dsmem_v4(a + y * 128 * 16, f[u] + 4 * y);
                }
#pragma unroll
                for (int x = 0; x < 16; ++x) v[x] = f[0][x];
#pragma unroll
                for (int u = 1; u < 4; ++u)
                  if (u < P.S)
#pragma unroll
                    for (int x = 0; x < 16; ++x) v[x] += f[u][x];
                if (et == 0 && m0 == s0 && !dry) ctl(p, ph, 9);
                if (m0 + 16 < lim) epi_prefetch(e, n, P.N, m0 + 16, lim, nxt);
                epi_chunk(e, n, P.N, m0, lim, v, cur, ln, dry);
                if (et == 0 && m0 == s0 && !dry) ctl(p, ph, 10);
                if (P.stats_out) stats_chunk(tile, m0, lim, dry);
                if (et == 0 && m0 == s0 && !dry) ctl(p, ph, 11);
                cur = nxt;
              }
              if (!dry) {
                pb_signal(pb_free, g0, P.S);
                ++pb_uses;
              }
            }
            continue;
          }
          mbar_wait(&acc_full[buf], (seg >> 1) & 1);
          tc_fence_after();
          if (et == 0) ctl(p, ph, 4);
          // split tile: park this k-split's partial, then finish a 1/S slice of the
          // token columns from all S partials of the tile
          {
            __half* dst = ws + (static_cast<int64_t>(i) * 128 + row) * BN;
#pragma unroll 1
            for (int cc = 0; cc < Mc; cc += 16) {
              tmem_ld16(acc + cc, v);
#pragma unroll
              for (int x = 0; x < 16; x += 8) {
                const __half2 h0 = __floats2half2_rn(v[x], v[x + 1]), h1 = __floats2half2_rn(v[x + 2], v[x + 3]);
                const __half2 h2 = __floats2half2_rn(v[x + 4], v[x + 5]), h3 = __floats2half2_rn(v[x + 6], v[x + 7]);
                *reinterpret_cast<uint4*>(dst + cc + x) =
                    make_uint4(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1),
                               *reinterpret_cast<const uint32_t*>(&h2), *reinterpret_cast<const uint32_t*>(&h3));
              }
            }
          }
          tc_fence_before();
          mbar_arrive(&acc_empty[buf]);
          // one gpu-scope release by et 0 publishes the partial: bar.sync orders the other
          // threads' stores before it (cumulativity)
          named_bar(1, 128);
          if (et == 0) st_release(p.flags + i, epoch);
          const int Mr = (Mc + 3) & ~3;
          const int sw = ((Mr + P.S - 1) / P.S + 3) & ~3;
          const int s0 = j * sw, s1 = min(Mr, s0 + sw);
          const int64_t lim = min(static_cast<int64_t>(s1), M);
          if (s0 < lim) epi_prefetch(e, n, P.N, s0, lim, cur);
          const int base = tile * P.S;
          if (et < P.S)
            for (uint32_t spins = 0; ld_relaxed(p.flags + base + et) < epoch;) {
              __nanosleep(32);
              if (++spins == (1u << 25)) wait_timeout("chain split flag", p.flags + base + et, epoch);
            }
          fence_acquire_gpu();
          named_bar(1, 128);
          if (et == 0) ctl(p, ph, 5);
#pragma unroll 1
          for (int m0 = s0; m0 < lim; m0 += 16) {
            // all S partials of these 16 columns in one batch of independent loads
            uint2 f[4][4];  // 4 halves each (m0 is a multiple of 4)
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
              if (jj < P.S) {
                const uint2* src =
                    reinterpret_cast<const uint2*>(ws + (static_cast<int64_t>(base + jj) * 128 + row) * BN + m0);
#pragma unroll
                for (int x = 0; x < 4; ++x) f[jj][x] = __ldcg(src + x);
              }
#pragma unroll
            for (int x = 0; x < 16; ++x) v[x] = 0.f;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)  // split order: deterministic
              if (jj < P.S) {
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&f[jj][x].x));
                  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&f[jj][x].y));
                  v[4 * x] += a.x;
                  v[4 * x + 1] += a.y;
                  v[4 * x + 2] += b.x;
                  v[4 * x + 3] += b.y;
                }
              }
            if (et == 0 && m0 == s0) ctl(p, ph, 9);
            if (m0 + 16 < lim) epi_prefetch(e, n, P.N, m0 + 16, lim, nxt);
            epi_chunk(e, n, P.N, m0, lim, v, cur, ln);
            if (et == 0 && m0 == s0) ctl(p, ph, 10);
            if (P.stats_out) stats_chunk(tile, m0, lim);
            if (et == 0 && m0 == s0) ctl(p, ph, 11);
            cur = nxt;
          }
        }
      }
      if (et == 0) ctl(p, ph, 2);
      if (ph + 1 < p.n_phases) {
        // publish this CTA's phase outputs: all epilogue stores -> one release arrival
        named_bar(1, 128);
        // (bar.sync orders the other epilogue threads' stores before et 0's gpu-scope release,
        // as for the split flags; a __threadfence in front of it cost 0.3 us per barrier)
        if (et == 0) {
          fence_proxy_async_global();
          red_release_add_u64(p.gbar, 1ull);
        }
      }
    }
    if (p.n_phases == 1) pdl_trigger();
  }
  tc_fence_before();
  __syncthreads();
  if (dsm) cluster_sync_all();  // no CTA leaves while a peer may still read its buffer
  if (warp == 1) tmem_dealloc(tmem, tcols);
  if (threadIdx.x == 0) ctl(p, kMaxPhases - 1, 3);
}

std::atomic<int> g_chain_epoch{0};


constexpr int kProbeMax = 64;
unsigned long long* g_ctl = nullptr;
int g_ctl_n = 0;
int g_ctl_ph[kProbeMax];
// the probe buffer is made resident on the device before kernels write it: a first GPU touch
// of a host-resident managed page faults (tens of us inside the timed chain per 64 KB page)
void probe_to_device() {
  int dev = 0;
  PCB_CUDA(cudaGetDevice(&dev));
  cudaMemLocation loc{};
  loc.type = cudaMemLocationTypeDevice;
  loc.id = dev;
  PCB_CUDA(cudaMemPrefetchAsync(g_ctl, sizeof(unsigned long long) * kMaxPhases * 160 * 16 * kProbeMax, loc, 0, 0));
  PCB_CUDA(cudaDeviceSynchronize());
}
unsigned long long* chain_probe_slot(int n_phases) {
  static const bool on = std::getenv("PCB_CHAIN_PROBE") != nullptr;
  if (!on || g_ctl_n >= kProbeMax) return nullptr;
  const size_t per = static_cast<size_t>(kMaxPhases) * 160 * 16;
  if (!g_ctl) {
    PCB_CUDA(cudaMallocManaged(&g_ctl, sizeof(unsigned long long) * per * kProbeMax));
    std::memset(g_ctl, 0, sizeof(unsigned long long) * per * kProbeMax);
    probe_to_device();
  }
  g_ctl_ph[g_ctl_n] = n_phases;
  return g_ctl + per * g_ctl_n++;
}

// per device: the stream that launched the last chain (cross-stream chain ordering)
struct ChainOrder {
  std::mutex mu;
  cudaStream_t last = nullptr;
  cudaEvent_t ev = nullptr;
};
ChainOrder& chain_order(int dev) {
  static ChainOrder orders[64];
  return orders[dev & 63];
}

template <int BN, int STAGES>
void launch_chain(const ChainStep* steps, int n, float* ws, size_t ws_bytes, int* flags, unsigned long long* gbar,
                  unsigned long long& gbar_count, cudaStream_t s, int sms) {
  using Sm = ChainSmem<BN, STAGES>;
  static bool attr = [] {
    PCB_CUDA(cudaFuncSetAttribute(k_chain<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, Sm::kBytes));
    return true;
  }();
  (void)attr;
  ChainParams p;
  std::memset(&p, 0, sizeof(p));
  p.n_phases = n;
  // Cluster launch (BN <= 64): 4-CTA clusters so the S CTAs of a split tile / attention head
  // exchange partials through DSMEM.  Clusters of 4 with this kernel's footprint fit fewer
  // than all SMs (132 of 148 on B200); every phase of the layer chain has <= 128 work items,
  // so the grid is the co-resident cluster count x 4 (the grid barrier needs co-residency).
  static const int dsm_grid = [&] {
    const char* v = std::getenv("PCB_CHAIN_DSM");
    if (Sm::kPB == 0 || (v && v[0] == '0')) return 0;
    PCB_CUDA(cudaFuncSetAttribute(k_chain<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, Sm::kBytes));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((sms / 4) * 4);
    cfg.blockDim = dim3(kChainThreads);
    cfg.dynamicSmemBytes = Sm::kBytes;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 4;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, k_chain<BN, STAGES>, &cfg) != cudaSuccess) {
      cudaGetLastError();
      return 0;
    }
    return std::min(nc, sms / 4) * 4;
  }();
  const bool dsm = dsm_grid >= 128;
  const int C = dsm ? dsm_grid : sms;
  p.dsm = dsm ? 1 : 0;
  int n_attn = 0;
  const ChainStep* attn0 = nullptr;
  for (int i = 0; i < n; ++i) {
    const ChainStep& st = steps[i];
    PhaseDev& d = p.ph[i];
    d.kind = st.kind;
    d.M = st.M;
    if (st.kind == CHAIN_GEMM) {
      d.N = st.N;
      d.K = st.K;
      d.kbs = st.K / 64;
      d.units = static_cast<int64_t>(st.N / 128) * d.kbs;
      const int tiles = st.N / 128;
      d.S = 2 * tiles > C ? 1 : std::min({4, C / tiles, d.kbs});  // dsm: a tile's splits share a cluster
      if (d.S == 3) d.S = 2;  // slices of 1/S of the columns: S in {1, 2, 4}
      d.items = tiles * d.S;
      d.w = static_cast<const uint8_t*>(st.w);
      d.e = st.e;
      d.stats_out = st.stats_out;
      d.stats_in = st.stats_in;
      d.stats_tiles = st.stats_tiles;
      d.stats_ld = st.stats_ld;
      d.stats_row0 = st.stats_row0;
      d.ln_dim = st.ln_dim;
      p.tm[i] = tmap_bf16_2d(st.x, static_cast<uint64_t>(st.M), static_cast<uint64_t>(st.K), BN);
    } else if (st.kind == CHAIN_ATTN) {
      // every attention phase of a launch serves the same request (one Q buffer, one segment
      // table); a contiguous cache has K / V maps per layer
      if (n_attn == kMaxAttn) throw std::runtime_error("chain: too many attention phases");
      if (n_attn > 0 && (st.aq != attn0->aq || st.M != attn0->M || st.a_d != attn0->a_d || st.aP != attn0->aP ||
                         st.a_nseg != attn0->a_nseg || st.aH != attn0->aH))
        throw std::runtime_error("chain: attention phases of one launch must serve one request");
      if (n_attn == 0) attn0 = &st;
      d.a_map = n_attn++;
      d.aP = st.aP;
      d.aH = st.aH;
      d.a_d = st.a_d;
      d.a_alibi = st.a_alibi;
      d.a_kpos = st.a_kpos;
      d.a_qpos = st.a_qpos;
      if (st.a_alibi && (!st.a_kpos || !st.a_qpos)) throw std::runtime_error("chain: ALiBi needs key and query positions");
      int64_t nblk = (st.aP + st.M + 63) / 64;
      if (st.a_nseg) {
        nblk = 0;
        for (int sgi = 0; sgi < st.a_nseg; ++sgi) nblk += (st.a_seg[sgi].rows + 63) / 64;
      }
      d.aS = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>({C / st.aH, nblk, dsm ? 4 : 8})));
      if (dsm && d.aS == 3) d.aS = 2;  // a head's splits share one cluster of 4
      d.items = st.aH * d.aS;
      d.ascale = 1.4426950408889634f / sqrtf(128.f);
      d.apart = st.a_scratch;
      d.aout = static_cast<__nv_bfloat16*>(st.aout);
      if (static_cast<size_t>(d.items) * 128 * 130 * sizeof(float) > st.a_scratch_bytes)
        throw std::runtime_error("chain: attention scratch too small");
      static const bool nodup = std::getenv("PCB_CHAIN_ATTN_NODUP") != nullptr;  // A/B switch
      d.adup = st.M <= 64 && !nodup;
      if (d.a_map == 0) p.tma[0] = tmap_bf16_2d(st.aq, static_cast<uint64_t>(st.M), static_cast<uint64_t>(st.a_d), 64);
      d.a_nseg = st.a_nseg;
      if (st.a_nseg) {
        if (st.a_nseg > ChainStep::kMaxSeg) throw std::runtime_error("chain: too many KV segments");
        d.a_layer = st.a_layer;
        d.a_tail_vis = static_cast<int>(st.a_tail_vis);
        int64_t keys = 0;
        d.a_first[0] = 0;
        for (int sgi = 0; sgi < st.a_nseg; ++sgi) {
          const ChainStep::KVSeg& g = st.a_seg[sgi];
          if (g.rows <= 0 || g.row0 + g.rows > g.cap) throw std::runtime_error("chain: bad KV segment");
          // rows end at the segment's last valid row: the rest of a 64-row block is TMA
          // zero fill, never stale memory (a masked key has P = 0, but 0 * NaN in PV is NaN)
          const ChainStep::KVSeg& g0 = attn0->a_seg[sgi];
          if (g.base != g0.base || g.row0 != g0.row0 || g.rows != g0.rows)
            throw std::runtime_error("chain: attention phases of one launch must share the KV segments");
          if (d.a_map == 0)
            p.tkv[sgi] = tmap_bf16_3d(g.base, static_cast<uint64_t>(st.a_d), static_cast<uint64_t>(g.row0 + g.rows),
                                      static_cast<uint64_t>(st.a_planes), g.plane_bytes, 64);
          d.a_row0[sgi] = static_cast<int>(g.row0);
          d.a_rows[sgi] = static_cast<int>(g.rows);
          d.a_first[sgi + 1] = d.a_first[sgi] + static_cast<int>((g.rows + 63) / 64);
          keys += g.rows;
        }
        if (keys != st.aP + st.M) throw std::runtime_error("chain: KV segments do not cover the keys");
      } else {
        p.tak[d.a_map] = tmap_bf16_2d(st.ak, static_cast<uint64_t>(st.aP + st.M), static_cast<uint64_t>(st.a_d), 64);
        p.tav[d.a_map] = tmap_bf16_2d(st.av, static_cast<uint64_t>(st.aP + st.M), static_cast<uint64_t>(st.a_d), 64);
      }
    } else {
      d.ln_src = st.ln_src;
      d.ln_dst = static_cast<__nv_bfloat16*>(st.ln_dst);
      d.ln_d = st.ln_d;
    }
  }
  p.ws = ws;
  p.ws_half = static_cast<int64_t>(C) * 128 * BN;
  if (C > 160) throw std::runtime_error("chain: grid exceeds the timeline probe layout");
  if (static_cast<size_t>(2 * p.ws_half) * sizeof(float) > ws_bytes) throw std::runtime_error("chain workspace too small");
  p.flags = flags;
  p.epoch0 = g_chain_epoch.fetch_add(n) + 1;
  p.gbar = gbar;
  p.gbar_base = gbar_count;
  p.tl = chain_probe_slot(n);
  if (p.tl)  // phase kinds for the timeline tools, in a slot no CTA writes (CTA 159, event 15)
    for (int i = 0; i < n; ++i) p.tl[(static_cast<size_t>(i) * 160 + 159) * 16 + 15] = 1 + p.ph[i].kind;
  static const int warm = [] {  // A/B switch: PCB_CHAIN_WARM=0 turns the dry epilogue pass off
    const char* v = std::getenv("PCB_CHAIN_WARM");
    return v ? std::atoi(v) : 1;
  }();
  p.warm = warm;
  gbar_count += static_cast<unsigned long long>(n - 1) * C;  // one arrival per CTA per phase boundary
  // The grid barrier needs all C CTAs resident at once: one per SM must fit (checked once
  // per instantiation), and two chains may never run concurrently on one device (each
  // could hold part of the SMs while waiting for the rest).  Chains of one stream are
  // ordered by the stream; a chain on another stream of the same device first waits for
  // everything submitted to the stream that launched the previous chain.
  static const int fit = [] {
    int nb = 0;
    PCB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_chain<BN, STAGES>, kChainThreads, Sm::kBytes));
    return nb;
  }();
  if (fit < 1) throw std::runtime_error("chain: one CTA per SM does not fit (shared memory or register limits)");
  int dev = 0;
  PCB_CUDA(cudaGetDevice(&dev));
  ChainOrder& o = chain_order(dev);
  std::lock_guard<std::mutex> lk(o.mu);
  if (o.last && o.last != s) {
    if (!o.ev) PCB_CUDA(cudaEventCreateWithFlags(&o.ev, cudaEventDisableTiming));
    PCB_CUDA(cudaEventRecord(o.ev, o.last));
    PCB_CUDA(cudaStreamWaitEvent(s, o.ev, 0));
  }
  o.last = s;
  PdlClass pc(PDL_GEMM);
  // cooperative launch attribute (default on; PCB_CHAIN_COOP=0: off): the driver guarantees every
  // CTA of the grid-barrier kernel co-resident or fails the launch, instead of a partly resident
  // grid spinning into the watchdog (same-box A/B neutral: tools/runs/gpu_r5d.sh)
  static const bool coop = [] {
    const char* v = std::getenv("PCB_CHAIN_COOP");
    return v == nullptr || v[0] != '0';
  }();
  if (dsm) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(kChainThreads);
    cfg.dynamicSmemBytes = Sm::kBytes;
    cfg.stream = s;
    cudaLaunchAttribute at[3];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 4;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = (pdl_enabled() && ((pdl_mask() >> PDL_GEMM) & 1)) ? 1 : 0;
    at[2].id = cudaLaunchAttributeCooperative;  // co-residency guaranteed by the launch (grid barrier)
    at[2].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = coop ? 3 : 2;
    PCB_CUDA(cudaLaunchKernelEx(&cfg, k_chain<BN, STAGES>, p));
  } else if (coop) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(kChainThreads);
    cfg.dynamicSmemBytes = Sm::kBytes;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PCB_CUDA(cudaLaunchKernelEx(&cfg, k_chain<BN, STAGES>, p));
  } else {
    launch_k(k_chain<BN, STAGES>, dim3(C), dim3(kChainThreads), Sm::kBytes, s, 1, p);
  }
}

}  // namespace

void chain_forget_stream(cudaStream_t s) {
  for (int dev = 0; dev < 64; ++dev) {
    ChainOrder& o = chain_order(dev);
    std::lock_guard<std::mutex> lk(o.mu);
    if (o.last == s) o.last = nullptr;
  }
}

bool chain_tc_supported(int64_t M, int N, int K) { return M >= 1 && M <= 128 && weight_packable(N, K); }
bool chain_ln_supported(int d) { return d % 4 == 0 && d <= 8192; }
bool chain_attn_supported(int64_t n, int64_t P, int H, int hd) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return hd == 128 && n >= 1 && n <= 128 && H >= 1 && H <= sms && P >= 0 && P + n < (1LL << 31);
}

int chain_probe_dump(unsigned long long* times, int max_launches, int* phases) {
  PCB_CUDA(cudaDeviceSynchronize());
  const int n = std::min(g_ctl_n, max_launches);
  const size_t per = static_cast<size_t>(kMaxPhases) * 160 * 16;
  if (n > 0) std::memcpy(times, g_ctl, sizeof(unsigned long long) * per * n);
  for (int i = 0; i < n; ++i) phases[i] = g_ctl_ph[i];
  if (g_ctl) {
    std::memset(g_ctl, 0, sizeof(unsigned long long) * per * kProbeMax);
    probe_to_device();
  }
  g_ctl_n = 0;
  return n;
}

void chain_tc(const ChainStep* steps, int n_steps, float* ws, size_t ws_bytes, int* flags,
              unsigned long long* gbar, unsigned long long& gbar_count, cudaStream_t s) {
  if (n_steps <= 0) return;
  if (n_steps > kMaxPhases) throw std::runtime_error("chain: too many phases");
  static int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  int64_t M = 1;
  for (int i = 0; i < n_steps; ++i) {
    const ChainStep& st = steps[i];
    if (st.kind == CHAIN_GEMM && !chain_tc_supported(st.M, st.N, st.K))
      throw std::runtime_error("chain: unsupported GEMM shape");
    if (st.kind == CHAIN_LN && !chain_ln_supported(st.ln_d)) throw std::runtime_error("chain: unsupported LN width");
    if (st.kind == CHAIN_ATTN && !chain_attn_supported(st.M, st.aP, st.aH, st.a_d / std::max(1, st.aH)))
      throw std::runtime_error("chain: unsupported attention phase");
    M = std::max<int64_t>(M, st.M);
  }
  // ring depth: what is left of 227 KB after the cluster exchange buffer (BN <= 64) and the
  // barrier / LayerNorm scratch
  if (M <= 16) launch_chain<16, 9>(steps, n_steps, ws, ws_bytes, flags, gbar, gbar_count, s, sms);
  else if (M <= 32) launch_chain<32, 8>(steps, n_steps, ws, ws_bytes, flags, gbar, gbar_count, s, sms);
  else if (M <= 64) launch_chain<64, 7>(steps, n_steps, ws, ws_bytes, flags, gbar, gbar_count, s, sms);
  else launch_chain<128, 6>(steps, n_steps, ws, ws_bytes, flags, gbar, gbar_count, s, sms);
}

}  // namespace pcb::kern

// Causal prefill attention on tcgen05 for long query ranges (module precompute, full
// prefill, long suffixes): reference Model::run attention, model.cpp:401-427 -- query i
// sees keys j <= P + i in sequence order, scores in fp32, softmax, P V.
//
// One CTA = one head x a PAIR of 128-query tiles (A = rows [q0, q0 + 128), B = the next
// 128) sharing one K/V stream of 128-key blocks; the MMA issuer alternates between the
// tiles so that one tile's softmax runs while the tensor core works on the other's:
//
//   tensor pipe:  ... PV_A(j-1) S_A(j) PV_B(j-1) S_B(j) PV_A(j) S_A(j+1) PV_B(j) S_B(j+1) ...
//   softmax A:                  [---- block j ----]         [---- block j+1 ...
//   softmax B:                                    [---- block j ----]
//
// so each softmax has two MMA slots (~1000 clk at 128x128x128) to turn S into P.
//
//   warp 0      TMA: both Q tiles once, then K_0 V_0 K_1 V_1 ... through a 5-slot ring of
//               32 KB (released in the same order the MMAs finish with them)
//   warp 1      TMEM (512 columns) + MMA issue: S_t = Q_t K_j^T (M=N=K=128) into tile t's
//               S columns; O_t += P_t V_j with P read from TMEM (the .kind::f16 TS form:
//               A operand in tensor memory), V an MN-major smem operand
//   warps 2-5   softmax of tile A, warps 6-9 of tile B: one thread per query row (TMEM
//               lane); the 128 scores of a block in registers, exponentials against a
//               lazily-updated running max (O in TMEM rescaled only when a row's max grows
//               by more than 2^8), P written back as packed bf16 over the first 64 S columns
//
// TMEM columns: tile t's S (then P) at [256 t, 256 t + 128), O at [256 t + 128, 256 t + 256).
// In-order execution of one thread's tcgen05.mma makes the S/P aliasing safe: S_t(j+1) is
// issued after PV_t(j) has been issued (and PV_t(j) reads P_t(j) first), and the commit that
// publishes S_t(j+1) also covers PV_t(j), so O_t is quiescent while the softmax rescales it.
// (attn_tc.cu keeps the single-tile kernel for few-query suffixes, split-KV, batched
// micro-batches, zero-copy segments and ALiBi.)
#include <cuda.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace pcb::kern {

using namespace tc;
CUtensorMap tmap_bf16_2d(const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows);

namespace {

constexpr int HD = 128, BQ = 128, BK = 128;
constexpr int kThreads = 320;
constexpr int kSlots = 5;
constexpr int kQBytes = BQ * HD * 2;     // one Q tile: two 64-column atoms of [128][128 B]
constexpr int kSlotBytes = BK * HD * 2;  // one K or V block: two atoms of [128 keys][128 B]
constexpr int kAtom = 128 * 128;         // bytes of one [128 rows][64 bf16] atom
constexpr int kSmem = 2 * kQBytes + kSlots * kSlotBytes + 1024 + 1024;
static_assert(kSmem <= 232448, "prefill attention shared memory");
constexpr float kThr = 8.0f;  // log2 domain: stale running max tolerated up to 2^8

struct PrefillParams {
  int n;            // query rows
  int H;            // heads
  int P;            // past rows before the queries (keys = P + n)
  int d;            // hidden (row stride of q / out in elements)
  float scale_log2; // log2(e) / sqrt(hd)
  __nv_bfloat16* out;
};

__device__ __forceinline__ void tmem_ld32_nowait(uint32_t addr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
}
__device__ __forceinline__ void tmem_st16u(uint32_t addr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st8u(uint32_t addr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float ex2(float x) {  // MUFU.EX2; ex2(-inf) = +0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (for part of the exponentials: MUFU.EX2 issues at a quarter of the
// FMA rate and bounds the softmax): round-to-nearest split x = k + f, f in [-1/2, 1/2],
// a degree-3 fit of 2^f (max rel. error 7.5e-5, far below the bf16 rounding of P), and k
// added to the exponent field -- (bits(x + 1.5 2^23) << 23) is exactly k << 23.
__device__ __forceinline__ float ex2_fma(float x) {
  x = fmaxf(x, -126.f);  // -inf (masked keys) -> 2^-126, i.e. 0 after the bf16 rounding of P
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  const float q = fmaf(fmaf(fmaf(0.05517084f, f, 0.24260935f), f, 0.69326097f), f, 0.99992818f);
  return __int_as_float(__float_as_int(q) + (__float_as_int(t) << 23));
}

// EMU: of every 8 key pairs, how many take ex2_fma instead of MUFU.EX2.  Measured (4160 /
// 16512 tokens, 32 heads): EMU 0 151 / 1947 us, 2 160 / 2037, 3 169 / 2137, 4 175 / 2196 --
// the softmax is not MUFU-bound here, so the default is 0 (PCB_PREFILL_EMU=3 for A/B).
template <int EMU>
__global__ void __launch_bounds__(kThreads, 1)
    k_attn_prefill(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, PrefillParams p) {
  extern __shared__ uint8_t smem_raw[];
  // pointer arithmetic on the __shared__ symbol (not an integer round trip) keeps the
  // shared address space visible to the compiler: LDS/STS instead of generic LD/ST
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  uint8_t* sQ = smem;                 // [2 tiles][32 KB]
  uint8_t* sKV = smem + 2 * kQBytes;  // [kSlots][32 KB]: K_0, V_0, K_1, V_1, ... (across units)
  uint64_t* q_full = reinterpret_cast<uint64_t*>(sKV + kSlots * kSlotBytes);  // Q tiles of a unit landed
  uint64_t* q_empty = q_full + 1;         // every MMA of the unit that reads Q is done
  uint64_t* kv_full = q_empty + 1;        // [kSlots]
  uint64_t* kv_empty = kv_full + kSlots;  // [kSlots]
  uint64_t* s_full = kv_empty + kSlots;   // [2] S_t(j) in TMEM
  uint64_t* p_full = s_full + 2;          // [2] P_t(j) in TMEM (128 arrivals)
  uint64_t* o_full = p_full + 2;          // [2] last PV_t of a unit complete
  uint64_t* o_empty = o_full + 2;         // [2] O_t read out by the softmax warps (128 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t total = static_cast<int64_t>(p.P) + p.n;
  const int T = (p.n + BQ - 1) / BQ;  // query tiles
  const int units = ((T + 1) >> 1) * p.H;
  // Unit u = (pair u / H, head u % H), heaviest pair first; a pair is the tiles
  // (hi - 1, hi) with hi = T - 1 - 2 (u / H), so a lone tile (T odd) is the lightest, tile 0.
  // CTA c takes its k-th unit in snake order (k C + c, then k C + C - 1 - c, ...): with
  // heaviest-first units that balances the per-CTA sums to within a few % of the mean.
  struct Unit {
    int h, qA, qB, nbA, nbB;
  };
  auto unit_of = [&](int k, Unit& U) -> bool {
    const int C = gridDim.x, c = blockIdx.x;
    const int u = k * C + ((k & 1) ? C - 1 - c : c);
    if (u >= units) return false;
    const int hi = T - 1 - 2 * (u / p.H), lo = hi - 1;
    U.h = u % p.H;
    U.qB = hi * BQ;
    U.qA = lo * BQ;
    auto nblocks = [&](int qt) {  // keys [0, min(total, P + qt + 128)) in blocks of 128
      const int64_t e = min(total, static_cast<int64_t>(p.P) + qt + BQ);
      return static_cast<int>((e + BK - 1) / BK);
    };
    U.nbA = lo >= 0 ? nblocks(U.qA) : 0;
    U.nbB = nblocks(U.qB);
    return true;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&s_full[t], 1);
      mbar_init(&p_full[t], 128);
      mbar_init(&o_full[t], 1);
      mbar_init(&o_empty[t], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // q / k / v come from the QKV GEMM just before

  if (warp == 0) {
    if (elect_one()) {
      Unit U;
      int i = 0;  // K/V ring sequence, continuous across units
      for (int k = 0; unit_of(k, U); ++k) {
        mbar_wait(q_empty, (k & 1) ^ 1);  // the previous unit's S MMAs are done with Q
        const int t0 = U.nbA > 0 ? 0 : 1;
        mbar_expect_tx(q_full, (2 - t0) * kQBytes);
        for (int t = t0; t < 2; ++t)
          for (int a = 0; a < 2; ++a)
            tma_load_2d(sQ + t * kQBytes + a * kAtom, &tmQ, q_full, U.h * HD + a * 64, t ? U.qB : U.qA);
        for (int b = 0; b < 2 * U.nbB; ++b, ++i) {
          const int s = i % kSlots;
          mbar_wait(&kv_empty[s], ((i / kSlots) & 1) ^ 1);
          mbar_expect_tx(&kv_full[s], kSlotBytes);
          const CUtensorMap* m = (b & 1) ? &tmV : &tmK;
          for (int a = 0; a < 2; ++a)
            tma_load_2d(sKV + s * kSlotBytes + a * kAtom, m, &kv_full[s], U.h * HD + a * 64, (b >> 1) * BK);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idS = idesc_bf16(BQ, BK);
      constexpr uint32_t idO = idesc_bf16(BQ, HD, false, true);  // V: MN-major
      int i0 = 0;                // ring index of this unit's K_0
      int js[2] = {0, 0};        // blocks issued per tile (s_full / p_full phases)
      int ou[2] = {0, 0};        // units per tile (o_full / o_empty phases)
      Unit U;
      for (int k = 0; unit_of(k, U); ++k) {
        mbar_wait(q_full, k & 1);
        auto issue_s = [&](int t, int j) {  // S_t = Q_t K_j^T
          const int i = i0 + 2 * j, s = i % kSlots;
          mbar_wait(&kv_full[s], (i / kSlots) & 1);
          tc_fence_after();
          const uint32_t qa = smem_u32(sQ + t * kQBytes), ka = smem_u32(sKV + s * kSlotBytes);
#pragma unroll
          for (int x = 0; x < HD / 16; ++x)
            umma_bf16(tmem + 256 * t, sw128_kmajor_desc(qa + (x >> 2) * kAtom + (x & 3) * 32),
                      sw128_kmajor_desc(ka + (x >> 2) * kAtom + (x & 3) * 32), idS, x > 0 ? 1u : 0u);
          umma_commit(&s_full[t]);
        };
        auto issue_pv = [&](int t, int j) {  // O_t += P_t V_j, P_t from TMEM
          const int i = i0 + 2 * j + 1, s = i % kSlots;
          if (j == 0) {  // O_t of the previous unit read out
            mbar_wait(&o_empty[t], (ou[t] & 1) ^ 1);
            ++ou[t];
          }
          mbar_wait(&kv_full[s], (i / kSlots) & 1);
          mbar_wait(&p_full[t], js[t] & 1);
          ++js[t];
          tc_fence_after();
          const uint32_t va = smem_u32(sKV + s * kSlotBytes);
#pragma unroll
          for (int x = 0; x < BK / 16; ++x)
            umma_bf16_ts(tmem + 256 * t + 128, tmem + 256 * t + x * 8,
                         sw128_mnmajor_desc(va + x * 2048, kAtom, 1024), idO, (j > 0 || x > 0) ? 1u : 0u);
        };
        if (U.nbA > 0) issue_s(0, 0);
        issue_s(1, 0);
        umma_commit(&kv_empty[i0 % kSlots]);  // K_0
        for (int j = 0; j < U.nbB; ++j) {
          if (j < U.nbA) {
            issue_pv(0, j);
            if (j + 1 < U.nbA) issue_s(0, j + 1);
            else umma_commit(&o_full[0]);
          }
          issue_pv(1, j);
          if (j + 1 < U.nbB) issue_s(1, j + 1);
          else umma_commit(&o_full[1]);
          umma_commit(&kv_empty[(i0 + 2 * j + 1) % kSlots]);                      // V_j
          if (j + 1 < U.nbB) umma_commit(&kv_empty[(i0 + 2 * j + 2) % kSlots]);  // K_{j+1}
        }
        umma_commit(q_empty);
        i0 += 2 * U.nbB;
      }
    }
  } else {
    // ---- softmax: tile t, query row r = TMEM lane ----
    const int t = (warp - 2) >> 2;
    const int qd = warp & 3;
    const int r = qd * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(qd * 32) << 16;
    const uint32_t tS = tmem + 256 * t + lane_off, tO = tS + 128;
    const float sc = p.scale_log2, thr = kThr / sc;
    int js = 0, ou = 0;  // s_full / o_full phases of this tile
    Unit U;
    for (int k = 0; unit_of(k, U); ++k) {
      const int nb = t ? U.nbB : U.nbA;
      if (nb == 0) continue;
      const int qi = (t ? U.qB : U.qA) + r;
      const int limit = p.P + qi;  // last visible key (sequence order)
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < nb; ++j, ++js) {
        mbar_wait(&s_full[t], js & 1);
        tc_fence_after();
        float sv[BK];
        {
          uint32_t raw[BK];
#pragma unroll
          for (int c = 0; c < BK; c += 32) tmem_ld32_nowait(tS + c, raw + c);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < BK; ++c) sv[c] = __uint_as_float(raw[c]);
        }
        const int lim = limit - j * BK;  // key c of the block visible iff c <= lim
        if (lim < BK - 1) {
#pragma unroll
          for (int c = 0; c < BK; ++c)
            if (c > lim) sv[c] = -INFINITY;
        }
        float mx[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) mx[c] = sv[c];
#pragma unroll
        for (int c = 8; c < BK; ++c) mx[c & 7] = fmaxf(mx[c & 7], sv[c]);
#pragma unroll
        for (int w = 4; w; w >>= 1)
#pragma unroll
          for (int c = 0; c < w; ++c) mx[c] = fmaxf(mx[c], mx[c + w]);
        const float bm = mx[0];
        const bool grow = bm > m + thr || (m == -INFINITY && bm > -INFINITY);
        if (__any_sync(0xffffffffu, grow) && j > 0) {
          // O_t holds blocks < j and is quiescent (its last PV completed before S_t(j))
          const float f = grow ? ex2((m - bm) * sc) : 1.f;
#pragma unroll 1
          for (int c = 0; c < HD; c += 32) {
            uint32_t o[32];
            tmem_ld32_nowait(tO + c, o);
            tmem_wait_ld();
#pragma unroll
            for (int x = 0; x < 32; ++x) o[x] = __float_as_uint(__uint_as_float(o[x]) * f);
            tmem_st16u(tO + c, o);
            tmem_st16u(tO + c + 16, o + 16);
          }
          tmem_st_wait();
        }
        if (grow) {
          l *= ex2((m - bm) * sc);
          m = bm;
        }
        const float mb = m == -INFINITY ? 0.f : m * sc;
        float bs0 = 0.f, bs1 = 0.f;
#pragma unroll
        for (int c = 0; c < BK; c += 16) {  // 16 keys -> 8 packed bf16 pairs -> P columns [c/2, c/2 + 8)
          uint32_t pk[8];
#pragma unroll
          for (int x = 0; x < 16; x += 2) {
            const bool emu = (x >> 1) >= 8 - EMU;
            const float a0 = fmaf(sv[c + x], sc, -mb), a1 = fmaf(sv[c + x + 1], sc, -mb);
            const float p0 = emu ? ex2_fma(a0) : ex2(a0);
            const float p1 = emu ? ex2_fma(a1) : ex2(a1);
            if (x & 2) bs1 += p0 + p1;
            else bs0 += p0 + p1;
            __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
            pk[x >> 1] = *reinterpret_cast<uint32_t*>(&b2);
          }
          tmem_st8u(tS + (c >> 1), pk);
        }
        l += bs0 + bs1;
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[t]);
      }
      mbar_wait(&o_full[t], ou & 1);
      ++ou;
      tc_fence_after();
      const float inv = 1.f / l;
      __nv_bfloat16* dst = p.out + static_cast<int64_t>(qi) * p.d + U.h * HD;
#pragma unroll 1
      for (int c = 0; c < HD; c += 32) {
        uint32_t o[32];
        tmem_ld32_nowait(tO + c, o);
        tmem_wait_ld();
        if (qi < p.n) {
#pragma unroll
          for (int x = 0; x < 32; x += 8) {
            uint4 w;
            __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
            for (int y = 0; y < 4; ++y)
              b[y] = __floats2bfloat162_rn(__uint_as_float(o[x + 2 * y]) * inv, __uint_as_float(o[x + 2 * y + 1]) * inv);
            *reinterpret_cast<uint4*>(dst + c + x) = w;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&o_empty[t]);  // the next unit's first PV_t may overwrite O_t
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

}  // namespace

bool attention_prefill_supported(const AttnArgs& a, int sms) {
  const int64_t pairs = (a.n + 2 * BQ - 1) / (2 * BQ);
  return a.hd == HD && !a.alibi && !a.mask && !a.block_id && !a.segs && !a.req && a.n_req == 0 && a.i0 == 0 &&
         a.nq < 0 && a.n > BQ && a.d % 64 == 0 && a.P + a.n < (1LL << 31) &&
         (a.pair == 2 || (a.pair == 1 && pairs * a.H >= sms));
}

void attention_prefill(const AttnArgs& a, cudaStream_t s) {
  static const int emu = [] {  // tuning override: exponentials on the FMA pipe per 8 pairs
    const char* v = std::getenv("PCB_PREFILL_EMU");
    return v ? std::atoi(v) : 0;
  }();
  static bool attr = [] {
    PCB_CUDA(cudaFuncSetAttribute(k_attn_prefill<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    PCB_CUDA(cudaFuncSetAttribute(k_attn_prefill<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    return true;
  }();
  (void)attr;
  PrefillParams p;
  p.n = static_cast<int>(a.n);
  p.P = static_cast<int>(a.P);
  p.d = a.d;
  p.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(HD));
  p.out = static_cast<__nv_bfloat16*>(a.out);
  const uint64_t total = static_cast<uint64_t>(a.P + a.n);
  CUtensorMap tq = tmap_bf16_2d(a.q, static_cast<uint64_t>(a.n), static_cast<uint64_t>(a.d), BQ);
  CUtensorMap tk = tmap_bf16_2d(a.k, total, static_cast<uint64_t>(a.d), BK);
  CUtensorMap tv = tmap_bf16_2d(a.v, total, static_cast<uint64_t>(a.d), BK);
  static const int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  p.H = a.H;
  const int64_t units = (a.n + 2 * BQ - 1) / (2 * BQ) * a.H;
  PdlClass pc(PDL_ATTN);
  const dim3 grid(static_cast<unsigned>(std::min<int64_t>(units, sms)));
  auto* kern = emu ? k_attn_prefill<3> : k_attn_prefill<0>;
  launch_k(kern, grid, dim3(kThreads), kSmem, s, 1, tq, tk, tv, p);
}

}  // namespace pcb::kern

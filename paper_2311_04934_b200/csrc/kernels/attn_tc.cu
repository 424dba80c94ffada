// tcgen05 flash attention for the bf16 hot path: a 128-query tile of one head
// against a range of key rows of the assembled cache (reference model.cpp:401-427:
// causal by sequence order, query i sees keys j <= P + i).
//
//   warp 0     TMA: Q tile once, then K/V blocks of 64 keys (2-stage ring)
//   warp 1     TMEM alloc + MMA issue: S = Q K^T (M=128, N=64, K=hd) into TMEM,
//              then O_blk = P V (M=128, N=hd, K=64; V as an MN-major operand)
//   warps 2-5  softmax: one thread per query row (TMEM lane), online max/sum in
//              fp32, P -> swizzled smem (bf16), O accumulated in registers
// Suffix prefill (few queries, long cache) splits the key range across CTAs so
// all SMs stream the KV; a combine kernel merges the (O, m, l) partials in split
// order (deterministic).  Prefill (P = 0) tiles queries and skips key blocks above
// the causal diagonal.
#include <cuda.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace pcb::kern {

using namespace tc;
CUtensorMap tmap_bf16_2d(const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows);

namespace {

constexpr int BQ = 128, BKV = 64, kAttnThreads = 192;

template <int HD>
struct AttnSmem {
  static constexpr int kAtoms = HD / 64;
  static constexpr int kQ = BQ * HD * 2;        // Q tile
  static constexpr int kKV = BKV * HD * 2;      // one K (or V) block
  static constexpr int kStage = 2 * kKV;        // K + V
  static constexpr int kP = BQ * BKV * 2;       // probabilities (bf16)
  static constexpr int kBytes = kQ + 2 * kStage + kP + 1024 + 1024;
  static constexpr uint32_t kTmemCols = HD + BKV <= 256 ? 256 : 512;
};

struct AttnParams {
  int64_t n, P, total;
  int H, d;
  int splits;
  int64_t blocks_total;  // key blocks for the whole (causal) range of tile 0
  float scale_log2;      // log2(e) / sqrt(hd)
  __nv_bfloat16* out;
  float* part_o;  // [H][splits][BQ][HD]
  float* part_ml; // [H][splits][BQ][2]
};

template <int HD>
__global__ void __launch_bounds__(kAttnThreads, 1)
    k_attn_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, AttnParams p) {
  using S = AttnSmem<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + S::kQ;
  uint8_t* sP = sKV + 2 * S::kStage;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sP + S::kP);
  uint64_t* q_full = bar;
  uint64_t* kv_full = bar + 1;   // [2]
  uint64_t* kv_empty = bar + 3;  // [2]
  uint64_t* s_full = bar + 5;
  uint64_t* p_full = bar + 6;
  uint64_t* o_full = bar + 7;
  uint64_t* o_free = bar + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 9);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q_tile = gridDim.x - 1 - blockIdx.x, h = blockIdx.y, split = blockIdx.z;  // heaviest tiles first
  const int64_t q0 = static_cast<int64_t>(q_tile) * BQ;
  // causal key range of this tile: keys [0, min(total, P + q0 + BQ))
  const int64_t key_end = min(p.total, p.P + q0 + BQ);
  const int64_t nblk = (key_end + BKV - 1) / BKV;
  const int64_t b0 = nblk * split / p.splits, b1 = nblk * (split + 1) / p.splits;
  const int nb = static_cast<int>(b1 - b0);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 128);
    mbar_init(o_full, 1);
    mbar_init(o_free, 128);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, S::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + BKV;
  pdl_trigger();
  pdl_wait();  // Q/K/V come from the QKV GEMM (and assembly) just before

  if (warp == 0) {
    if (elect_one() && nb > 0) {
      mbar_expect_tx(q_full, S::kQ);
      for (int a = 0; a < S::kAtoms; ++a)
        tma_load_2d(sQ + a * (BQ * 128), &tmQ, q_full, h * HD + a * 64, static_cast<int>(q0));
      for (int it = 0; it < nb; ++it) {
        const int s = it & 1;
        mbar_wait(&kv_empty[s], ((it >> 1) & 1) ^ 1);
        uint8_t* st = sKV + s * S::kStage;
        const int j0 = static_cast<int>((b0 + it) * BKV);
        mbar_expect_tx(&kv_full[s], S::kStage);
        for (int a = 0; a < S::kAtoms; ++a) {
          tma_load_2d(st + a * (BKV * 128), &tmK, &kv_full[s], h * HD + a * 64, j0);
          tma_load_2d(st + S::kKV + a * (BKV * 128), &tmV, &kv_full[s], h * HD + a * 64, j0);
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one() && nb > 0) {
      constexpr uint32_t idS = idesc_bf16(BQ, BKV);
      constexpr uint32_t idO = idesc_bf16(BQ, HD, false, true);  // V is MN-major
      const uint32_t q_addr = smem_u32(sQ), p_addr = smem_u32(sP);
      mbar_wait(q_full, 0);
      auto issue_qk = [&](int it) {
        const int s = it & 1;
        mbar_wait(&kv_full[s], (it >> 1) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sKV + s * S::kStage);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const int a = k >> 2, kk = k & 3;
          umma_bf16(tS, sw128_kmajor_desc(q_addr + a * (BQ * 128) + kk * 32),
                    sw128_kmajor_desc(k_addr + a * (BKV * 128) + kk * 32), idS, k > 0 ? 1u : 0u);
        }
        umma_commit(s_full);
      };
      issue_qk(0);
      for (int it = 0; it < nb; ++it) {
        const int s = it & 1;
        mbar_wait(p_full, it & 1);  // P(it) in smem, S(it) consumed
        tc_fence_after();
        if (it + 1 < nb) issue_qk(it + 1);
        if (it > 0) mbar_wait(o_free, (it - 1) & 1);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sKV + s * S::kStage + S::kKV);
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k)
          umma_bf16(tO, sw128_kmajor_desc(p_addr + k * 32), sw128_mnmajor_desc(v_addr + k * 2048, BKV * 128, 1024),
                    idO, k > 0 ? 1u : 0u);
        umma_commit(o_full);
        umma_commit(&kv_empty[s]);
      }
    }
  } else {
    // ---- softmax warps: query row = TMEM lane ----
    const int qd = warp & 3;
    const int r = qd * 32 + lane;
    const int64_t qi = q0 + r;             // query index within the n new rows
    const int64_t limit = p.P + qi;        // last visible key (sequence order)
    const uint32_t lane_off = static_cast<uint32_t>(qd * 32) << 16;
    float o[HD];
#pragma unroll
    for (int x = 0; x < HD; ++x) o[x] = 0.f;
    float m = -INFINITY, l = 0.f;
    for (int it = 0; it < nb; ++it) {
      const int64_t j0 = (b0 + it) * BKV;
      mbar_wait(s_full, it & 1);
      tc_fence_after();
      float sv[BKV];
#pragma unroll
      for (int c = 0; c < BKV; c += 16) tmem_ld16(tS + lane_off + c, sv + c);
      float bm = -INFINITY;
#pragma unroll
      for (int c = 0; c < BKV; ++c) {
        sv[c] = (j0 + c <= limit) ? sv[c] * p.scale_log2 : -INFINITY;
        bm = fmaxf(bm, sv[c]);
      }
      const float mn = fmaxf(m, bm);
      const float alpha = (mn == -INFINITY) ? 1.f : exp2f(m - mn);
      float bsum = 0.f;
      uint32_t packed[BKV / 2];
#pragma unroll
      for (int c = 0; c < BKV; c += 2) {
        float p0 = (mn == -INFINITY) ? 0.f : exp2f(sv[c] - mn);
        float p1 = (mn == -INFINITY) ? 0.f : exp2f(sv[c + 1] - mn);
        __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
        // the denominator sums the bf16-rounded weights actually fed to the MMA
        float2 f2 = __bfloat1622float2(b2);
        bsum += f2.x + f2.y;
        packed[c >> 1] = *reinterpret_cast<uint32_t*>(&b2);
      }
      l = l * alpha + bsum;
      m = mn;
      // P row r -> 128-byte swizzled smem row (16-byte chunk c at c ^ (r & 7))
      uint8_t* prow = sP + r * 128;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint4 v = make_uint4(packed[4 * c], packed[4 * c + 1], packed[4 * c + 2], packed[4 * c + 3]);
        *reinterpret_cast<uint4*>(prow + ((c ^ (r & 7)) << 4)) = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      mbar_arrive(p_full);
#pragma unroll
      for (int x = 0; x < HD; ++x) o[x] *= alpha;
      mbar_wait(o_full, it & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < HD; c += 16) {
        float ob[16];
        tmem_ld16(tO + lane_off + c, ob);
#pragma unroll
        for (int x = 0; x < 16; ++x) o[c + x] += ob[x];
      }
      tc_fence_before();
      mbar_arrive(o_free);
    }
    if (qi < p.n && nb > 0) {
      if (p.splits == 1) {
        const float inv = 1.f / l;
        __nv_bfloat16* dst = p.out + qi * p.d + h * HD;
#pragma unroll
        for (int x = 0; x < HD; x += 8) {
          uint4 v;
          __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
          for (int y = 0; y < 4; ++y) b[y] = __floats2bfloat162_rn(o[x + 2 * y] * inv, o[x + 2 * y + 1] * inv);
          *reinterpret_cast<uint4*>(dst + x) = v;
        }
      } else {
        const int64_t slot = (static_cast<int64_t>(h) * p.splits + split) * BQ + r;
        float* po = p.part_o + slot * HD;
#pragma unroll
        for (int x = 0; x < HD; x += 4) *reinterpret_cast<float4*>(po + x) = make_float4(o[x], o[x + 1], o[x + 2], o[x + 3]);
        p.part_ml[slot * 2] = m;
        p.part_ml[slot * 2 + 1] = l;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, S::kTmemCols);
}

// Merge split partials in split order: O = sum_s 2^(m_s - M) O_s / sum_s 2^(m_s - M) l_s.
template <int HD>
__global__ void k_attn_combine(AttnParams p) {
  pdl_trigger();
  pdl_wait();
  const int64_t qi = blockIdx.x;
  const int h = blockIdx.y, x = threadIdx.x;
  float M = -INFINITY;
  for (int s = 0; s < p.splits; ++s) {
    const int64_t slot = (static_cast<int64_t>(h) * p.splits + s) * BQ + qi;
    if (p.part_ml[slot * 2 + 1] > 0.f) M = fmaxf(M, p.part_ml[slot * 2]);
  }
  float num = 0.f, den = 0.f;
  for (int s = 0; s < p.splits; ++s) {
    const int64_t slot = (static_cast<int64_t>(h) * p.splits + s) * BQ + qi;
    const float ls = p.part_ml[slot * 2 + 1];
    if (!(ls > 0.f)) continue;
    const float w = exp2f(p.part_ml[slot * 2] - M);
    num += w * p.part_o[slot * HD + x];
    den += w * ls;
  }
  p.out[qi * p.d + h * HD + x] = __float2bfloat16_rn(num / den);
}

template <int HD>
void launch_attn(const AttnArgs& a, float* scratch, size_t scratch_bytes, cudaStream_t s) {
  using Sm = AttnSmem<HD>;
  static bool attr = [] {
    PCB_CUDA(cudaFuncSetAttribute(k_attn_tc<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, Sm::kBytes));
    return true;
  }();
  (void)attr;
  static int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  AttnParams p;
  p.n = a.n;
  p.P = a.P;
  p.total = a.P + a.n;
  p.H = a.H;
  p.d = a.d;
  p.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(HD));
  p.out = static_cast<__nv_bfloat16*>(a.out);
  const int q_tiles = static_cast<int>((a.n + BQ - 1) / BQ);
  const int64_t nblk0 = (std::min<int64_t>(p.total, a.P + BQ) + BKV - 1) / BKV;  // tile 0 key blocks
  // one CTA per SM (the fp32 O row lives in registers); pick the split count that
  // minimises (waves x blocks per CTA) for single-tile (suffix) launches
  const int base = q_tiles * a.H;
  int splits = 1;
  if (q_tiles == 1 && base < 2 * sms) {
    int64_t best = -1;
    for (int s2 = 1; s2 <= std::max<int64_t>(1, std::min<int64_t>(nblk0 / 2, 32)); ++s2) {
      const size_t need = static_cast<size_t>(a.H) * s2 * BQ * (HD + 2) * sizeof(float);
      if (s2 > 1 && need > scratch_bytes) break;
      const int64_t cost = ((static_cast<int64_t>(base) * s2 + sms - 1) / sms) * ((nblk0 + s2 - 1) / s2) * 16 + s2;
      if (best < 0 || cost < best) {
        best = cost;
        splits = s2;
      }
    }
  }
  p.splits = splits;
  p.part_o = scratch;
  p.part_ml = scratch + static_cast<size_t>(a.H) * splits * BQ * HD;
  CUtensorMap tq = tmap_bf16_2d(a.q, static_cast<uint64_t>(a.n), static_cast<uint64_t>(a.d), BQ);
  CUtensorMap tk = tmap_bf16_2d(a.k, static_cast<uint64_t>(p.total), static_cast<uint64_t>(a.d), BKV);
  CUtensorMap tv = tmap_bf16_2d(a.v, static_cast<uint64_t>(p.total), static_cast<uint64_t>(a.d), BKV);
  dim3 grid(q_tiles, a.H, splits);
  launch_k(k_attn_tc<HD>, grid, dim3(kAttnThreads), Sm::kBytes, s, 1, tq, tk, tv, p);
  if (splits > 1) {
    launch_k(k_attn_combine<HD>, dim3(static_cast<unsigned>(a.n), a.H), dim3(HD), 0, s, 1, p);
  }
}

}  // namespace

bool attention_tc_supported(const AttnArgs& a) {
  return (a.hd == 128 || a.hd == 64) && !a.mask && !a.block_id && !a.alibi && a.n >= 1 && a.d % 64 == 0 &&
         (a.P + a.n) < (1LL << 31);
}

void attention_tc(const AttnArgs& a, float* scratch, size_t scratch_bytes, cudaStream_t s) {
  if (a.hd == 128) launch_attn<128>(a, scratch, scratch_bytes, s);
  else launch_attn<64>(a, scratch, scratch_bytes, s);
}

}  // namespace pcb::kern

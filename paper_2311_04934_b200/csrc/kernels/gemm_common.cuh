// Shared pieces of the tcgen05 weight-streaming GEMMs (gemm_tc.cu: one GEMM per
// launch; chain_tc.cu: a persistent chain of GEMM / LayerNorm phases): the fused
// epilogue, bulk copies, release/acquire flags and the stream-K unit split.
#pragma once
#include <cuda.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace pcb::kern {

using namespace tc;

// ---------------------------------------------------------------------------
// Epilogue on one thread's weight row n for 16 consecutive tokens [m0, m0+16),
// split into a prefetch (global loads that do not depend on the accumulator:
// residual rows, RoPE cos/sin) and the apply step, so the loads of the next
// chunk are in flight while the current one is processed.
// ---------------------------------------------------------------------------
struct EpiPre {
  float a[16], b[16];
  float lnw;  // LN fold: sum_k W[n][k] (prefetched with the chunk's other operands)
};

// rope = false: the RoPE operands come from elsewhere (staged in TMEM by the chain)
__device__ __forceinline__ void epi_prefetch(const Epilogue& ep, int n, int N, int64_t m0, int64_t M, EpiPre& p,
                                             bool rope = true, bool lnw = true) {
  const int kind = ep.kind;
  // an L2 round trip under a saturated memory system is ~1 us: issued before the
  // accumulator is ready instead of inside the first chunk (tools/chain_ab.py c0_values)
  if (ep.ln_wsum && lnw) p.lnw = __ldg(ep.ln_wsum + n);
  if (kind == EPI_QKV && !rope) return;
  if (kind == EPI_RESID) {
    const float* src = ep.resid + m0 * N + n;
#pragma unroll
    for (int j = 0; j < 16; ++j) p.a[j] = (m0 + j < M) ? __ldcg(src + j * N) : 0.f;  // L2: written by other SMs
  } else if (kind == EPI_QKV) {
    const int d = ep.d, hd = ep.head_dim;
    const int seg = n / d, c = n - seg * d;
    if (seg < 2 && ep.rope && ep.rope_tab) {
      const float4* src = reinterpret_cast<const float4*>(ep.rope_tab + ((c % hd) >> 1) * ep.rope_ld + m0);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float4 t = src[u];
        p.a[2 * u] = t.x;
        p.b[2 * u] = t.y;
        p.a[2 * u + 1] = t.z;
        p.b[2 * u + 1] = t.w;
      }
    } else if (seg < 2 && ep.rope) {
      const int half = hd >> 1, pi = (c % hd) >> 1;
      const int32_t* pos = ep.pos + m0;
      const float* cs = ep.rope_cos32 + pi;
      const float* sn = ep.rope_sin32 + pi;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int64_t q = (m0 + j < M) ? static_cast<int64_t>(pos[j]) * half : 0;
        p.a[j] = cs[q];
        p.b[j] = sn[q];
      }
    }
  }
}

__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// tanh-GELU for the bf16 path (the result is rounded to bf16, 2^-8, so the MUFU tanh's
// ~2^-11 relative error is below the output precision; the fp32 path uses gelu_ref)
__device__ __forceinline__ float gelu_bf16path(float x) {
  const float t = 0.7978845608028654f * fmaf(0.044715f * x, x * x, x);
  const float hx = 0.5f * x;
  return fmaf(hx, tanh_approx(t), hx);
}

// The epilogue warps are one per scheduler, so the per-element cost is latency, not
// throughput: fields are read once into registers, full chunks take an unguarded,
// fully unrolled path, and only a ragged last chunk is guarded.
// nost: compute everything but store nothing (the chain's instruction-cache warm-up pass)
__device__ __forceinline__ void epi_chunk(const Epilogue& ep, int n, int N, int64_t m0, int64_t M, float* v,
                                          const EpiPre& pre, const float2* lnst = nullptr, bool nost = false) {
  const int kind = ep.kind;
  const int jn = M - m0 >= 16 ? 16 : static_cast<int>(M - m0);
  if (lnst) {  // folded LayerNorm: {mean, rstd} of token m0 + j
    const float ws = pre.lnw;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float2 st = lnst[j < jn ? m0 + j : m0];
      v[j] = st.y * fmaf(-st.x, ws, v[j]);
    }
  }
  if (kind != EPI_RESID && nost) return;  // the warm-up pass only runs residual (split) phases
  if (kind == EPI_QKV) {
    const int d = ep.d;
    const int seg = n / d, c = n - seg * d;
    const bool rot = seg < 2 && ep.rope;
    const bool odd = c & 1;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float pv = __shfl_xor_sync(0xffffffffu, v[j], 1);  // partner column n^1 lives in lane^1
      if (rot) v[j] = odd ? fmaf(pv, pre.b[j], v[j] * pre.a[j]) : fmaf(v[j], pre.a[j], -pv * pre.b[j]);
    }
    if (seg > 0 && ep.kv_off) {  // batched requests: each token's row lives in its own cache
      __nv_bfloat16* base = static_cast<__nv_bfloat16*>(seg == 1 ? ep.k_out : ep.v_out) + c;
      const int64_t* off = ep.kv_off + m0;
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < jn) base[off[j]] = __float2bfloat16_rn(v[j]);
      return;
    }
    __nv_bfloat16* dst = (seg == 0 ? static_cast<__nv_bfloat16*>(ep.q_out)
                                   : static_cast<__nv_bfloat16*>(seg == 1 ? ep.k_out : ep.v_out) + ep.kv_row0 * d) +
                         m0 * d + c;
    if (jn == 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j) dst[j * d] = __float2bfloat16_rn(v[j]);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < jn) dst[j * d] = __float2bfloat16_rn(v[j]);
    }
    return;
  }
  if (kind == EPI_RESID) {
    float* dst = ep.resid + m0 * N + n;
    if (ep.x_out) {  // LN fold: the new residual also as the next GEMM's bf16 input; v <- new residual
      __nv_bfloat16* xo = static_cast<__nv_bfloat16*>(ep.x_out) + m0 * N + n;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        v[j] = pre.a[j] + v[j];
        if (j < jn) {
          if (!nost) {
            dst[j * N] = v[j];
            xo[j * N] = __float2bfloat16_rn(v[j]);
          }
        } else {
          v[j] = 0.f;
        }
      }
      return;
    }
    if (nost) return;
    if (jn == 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j) dst[j * N] = pre.a[j] + v[j];
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < jn) dst[j * N] = pre.a[j] + v[j];
    }
  } else if (kind == EPI_GELU) {
    __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(ep.out) + m0 * N + n;
    if (jn == 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j) dst[j * N] = __float2bfloat16_rn(gelu_bf16path(v[j]));
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < jn) dst[j * N] = __float2bfloat16_rn(gelu_bf16path(v[j]));
    }
  } else if (kind == EPI_F32) {
    float* dst = ep.outf + m0 * ep.ldo + n;
    const int64_t ldo = ep.ldo;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (j < jn) dst[j * ldo] = v[j];
  }
}

// The value part of epi_chunk for the bf16-output kinds (QKV, GELU): folded-LN
// correction, RoPE (partner column in lane^1) or GELU applied in place, no stores -- for
// epilogues that stage the tile in shared memory and store whole rows.
__device__ __forceinline__ void epi_values(const Epilogue& ep, int n, int64_t m0, int64_t M, float* v,
                                           const EpiPre& pre, const float2* lnst) {
  const int jn = M - m0 >= 16 ? 16 : static_cast<int>(M - m0);
  if (lnst) {
    const float ws = pre.lnw;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float2 st = lnst[j < jn ? m0 + j : m0];
      v[j] = st.y * fmaf(-st.x, ws, v[j]);
    }
  }
  if (ep.kind == EPI_QKV) {
    const int d = ep.d;
    const int seg = n / d, c = n - seg * d;
    const bool rot = seg < 2 && ep.rope;
    const bool odd = c & 1;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float pv = __shfl_xor_sync(0xffffffffu, v[j], 1);
      if (rot) v[j] = odd ? fmaf(pv, pre.b[j], v[j] * pre.a[j]) : fmaf(v[j], pre.a[j], -pv * pre.b[j]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = gelu_bf16path(v[j]);
  }
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Spin-wait reads are relaxed (an acquire load invalidates the SM's whole L1 -- CCTL.IVALL
// -- on every poll); the waiter issues one acquire fence after the condition holds.
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}



// First unit of CTA c when U units are split evenly over C CTAs.  c * U < 2^32 for every
// launch (checked on the host: units_fit_u32), so the split uses 32-bit division (a 64-bit
// divide is a ~100-instruction software routine, and these sit on the phase-end path).
__device__ __forceinline__ int64_t unit_begin(int c, int64_t U, int C) {
  return static_cast<int64_t>(static_cast<uint32_t>(c) * static_cast<uint32_t>(U) / static_cast<uint32_t>(C));
}
inline bool units_fit_u32(int64_t U, int C) { return U >= 0 && (static_cast<uint64_t>(U) * (C + 1)) < (1ull << 32); }

__device__ __forceinline__ bool has_units(int cc, int64_t U, int C) {
  return unit_begin(cc, U, C) < unit_begin(cc + 1, U, C);
}

// CTA whose unit range contains unit g
__device__ __forceinline__ int cta_of(int64_t g, int64_t U, int C) {
  int c = static_cast<int>((g * C) / U);
  while (c + 1 < C && unit_begin(c + 1, U, C) <= g) ++c;
  while (c > 0 && unit_begin(c, U, C) > g) --c;
  return c;
}


// Owner of a stream-K tile: its TMEM accumulator (lane = weight row n, column =
// token) plus the fp32 partials parked by CTAs (c, c_last] in CTA order
// (deterministic), then the fused epilogue.  The end of a phase is L2-latency-bound
// (~1 us per dependent round trip while the weight stream saturates the memory
// system), so each partial is fetched as one batch of independent loads and the
// epilogue inputs of the next two chunks are in flight meanwhile.  `cur` holds the
// prefetched inputs of chunk 0.
template <int BN>
__device__ __forceinline__ void owner_finish(const Epilogue& e, uint32_t acc, int n, int N, int64_t M, const float* ws,
                                             int c, int c_last, int64_t U, int C, int row, EpiPre& cur,
                                             unsigned long long* tp = nullptr) {
  auto mark = [&](int i) {
    if (tp) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      tp[i] = t;
    }
  };
  constexpr int G = BN < 64 ? BN : 64;  // columns (tokens) per register group
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += G) {
    if (c0 >= M) break;  // warp-uniform
    float a[G];
    {
      uint32_t r[G];
#pragma unroll
      for (int j = 0; j < G; j += 16) tmem_ld16_nowait(acc + c0 + j, r + j);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < G; ++j) a[j] = __uint_as_float(r[j]);
    }
    if (c0 == 0) mark(0);
    EpiPre nxt;
    if (c0 > 0) epi_prefetch(e, n, N, c0, M, cur);
    if (16 < G && c0 + 16 < M) epi_prefetch(e, n, N, c0 + 16, M, nxt);
#pragma unroll 1
    for (int pp = c + 1; pp <= c_last; ++pp) {
      if (!has_units(pp, U, C)) continue;  // more CTAs than units: empty ranges
      const float4* src = reinterpret_cast<const float4*>(ws + (static_cast<int64_t>(pp) * 128 + row) * BN + c0);
      float4 f[G / 4];
#pragma unroll
      for (int j = 0; j < G / 4; ++j) f[j] = __ldcg(src + j);
#pragma unroll
      for (int j = 0; j < G / 4; ++j) {
        a[4 * j] += f[j].x;
        a[4 * j + 1] += f[j].y;
        a[4 * j + 2] += f[j].z;
        a[4 * j + 3] += f[j].w;
      }
    }
    if (c0 == 0) mark(1);
#pragma unroll
    for (int cc = 0; cc < G; cc += 16) {
      if (c0 + cc >= M) break;
      EpiPre nn;
      if (cc + 32 < G && c0 + cc + 32 < M) epi_prefetch(e, n, N, c0 + cc + 32, M, nn);
      epi_chunk(e, n, N, c0 + cc, M, a + cc, cur);
      cur = nxt;
      nxt = nn;
    }
    if (c0 == 0) mark(2);
  }
  mark(3);
}

}  // namespace pcb::kern

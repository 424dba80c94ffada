// SIMT kernels: weight generation, embed, LayerNorm, argmax, the fp32-parity
// GEMM / attention (fp64 accumulation in the reference's order), the KV
// assembly copy engine and row gather.  The bf16 hot-path GEMM and attention
// live in gemm_tc.cu / attn_tc.cu.
#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace pcb::kern {

// ---------------------------------------------------------------------------
// Weights: PCG32 (XSH-RR) with LCG jump-ahead.  The reference's fill_uniform
// (model.cpp:122-127) constructs Pcg32(seed) (state = seed + inc, one output
// discarded) and writes element i from output i+1; element i therefore comes
// from the state reached after i+1 LCG steps.  Each thread jumps straight to its
// chunk: bit-identical fp32 values, then RNE to bf16 for the bf16 model.
// ---------------------------------------------------------------------------

constexpr uint64_t kMul = 6364136223846793005ULL;
constexpr uint64_t kInc = 1442695040888963407ULL;

__device__ __forceinline__ uint64_t lcg_advance(uint64_t state, uint64_t delta) {
  uint64_t acc_mult = 1, acc_plus = 0, cur_mult = kMul, cur_plus = kInc;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__device__ __forceinline__ uint32_t pcg_out(uint64_t old) {
  uint32_t xs = static_cast<uint32_t>(((old >> 18u) ^ old) >> 27u);
  uint32_t rot = static_cast<uint32_t>(old >> 59u);
  return (xs >> rot) | (xs << ((-rot) & 31u));
}

template <typename T>
__global__ void k_init_uniform(T* dst, uint64_t count, uint64_t seed, float scale, uint64_t chunk) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t begin = t * chunk;
  if (begin >= count) return;
  uint64_t end = min(begin + chunk, count);
  uint64_t state = lcg_advance(seed + kInc, begin + 1);
  for (uint64_t i = begin; i < end; ++i) {
    uint32_t x = pcg_out(state);
    state = state * kMul + kInc;
    float u = __fmul_rn(static_cast<float>(x >> 8), 1.0f / 16777216.0f);
    float w = __fmul_rn(__fsub_rn(__fmul_rn(2.0f, u), 1.0f), scale);
    st_f(dst, static_cast<int64_t>(i), w);
  }
}

void init_uniform(int dtype, void* dst, uint64_t count, uint64_t seed, float scale, cudaStream_t s) {
  const uint64_t chunk = 256;
  uint64_t threads = (count + chunk - 1) / chunk;
  unsigned blocks = static_cast<unsigned>((threads + 255) / 256);
  if (dtype == F32)
    k_init_uniform<float><<<blocks, 256, 0, s>>>(static_cast<float*>(dst), count, seed, scale, chunk);
  else
    k_init_uniform<__nv_bfloat16><<<blocks, 256, 0, s>>>(static_cast<__nv_bfloat16*>(dst), count, seed, scale, chunk);
  PCB_CUDA(cudaGetLastError());
}

// Block of a larger stream-backed [*][full_cols] tensor: dst[i][j] = element
// (row0 + i) * full_cols + col0 + j of the stream (tensor-parallel shards: row ranges of
// column-parallel weights, column ranges of row-parallel ones), one jump per row chunk.
template <typename T>
__global__ void k_init_uniform_block(T* dst, int64_t rows, int64_t cols, uint64_t seed, float scale, int64_t row0,
                                     int64_t col0, int64_t full_cols, int64_t chunk) {
  const int64_t chunks_per_row = (cols + chunk - 1) / chunk;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= rows * chunks_per_row) return;
  const int64_t i = t / chunks_per_row, j0 = (t % chunks_per_row) * chunk;
  const int64_t j1 = min(j0 + chunk, cols);
  uint64_t state = lcg_advance(seed + kInc, static_cast<uint64_t>((row0 + i) * full_cols + col0 + j0) + 1);
  for (int64_t j = j0; j < j1; ++j) {
    uint32_t x = pcg_out(state);
    state = state * kMul + kInc;
    float u = __fmul_rn(static_cast<float>(x >> 8), 1.0f / 16777216.0f);
    float w = __fmul_rn(__fsub_rn(__fmul_rn(2.0f, u), 1.0f), scale);
    st_f(dst, i * cols + j, w);
  }
}
void init_uniform_block(int dtype, void* dst, int64_t rows, int64_t cols, uint64_t seed, float scale, int64_t row0,
                        int64_t col0, int64_t full_cols, cudaStream_t s) {
  const int64_t chunk = 256;
  const int64_t threads = rows * ((cols + chunk - 1) / chunk);
  const unsigned blocks = static_cast<unsigned>((threads + 255) / 256);
  if (dtype == F32)
    k_init_uniform_block<float><<<blocks, 256, 0, s>>>(static_cast<float*>(dst), rows, cols, seed, scale, row0, col0,
                                                        full_cols, chunk);
  else
    k_init_uniform_block<__nv_bfloat16><<<blocks, 256, 0, s>>>(static_cast<__nv_bfloat16*>(dst), rows, cols, seed,
                                                                scale, row0, col0, full_cols, chunk);
  PCB_CUDA(cudaGetLastError());
}

// out[n] = sum_k W[n][k] (bf16 row-major; one warp per row, fp64 accumulation)
__global__ void k_row_sums_bf16(const __nv_bfloat16* W, int N, int K, float* out) {
  const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
  if (row >= N) return;
  double acc = 0;
  for (int k = lane; k < K; k += 32) acc += static_cast<double>(__bfloat162float(W[static_cast<int64_t>(row) * K + k]));
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[row] = static_cast<float>(acc);
}
void row_sums_bf16(const void* W, int N, int K, float* out, cudaStream_t s) {
  k_row_sums_bf16<<<(N + 7) / 8, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(W), N, K, out);
  PCB_CUDA(cudaGetLastError());
}

// h += part (tensor-parallel: the all-reduced partial sums of a row-parallel GEMM)
__global__ void k_add_inplace(float* __restrict__ h, const float* __restrict__ part, int64_t n) {
  pdl_trigger();
  pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    h[i] = __fadd_rn(h[i], part[i]);
}
void add_inplace(float* h, const float* part, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 1184));
  launch_k(k_add_inplace, dim3(blocks), dim3(256), 0, s, 1, h, part, n);
  PCB_CUDA(cudaGetLastError());
}

// vocab shards gathered rank-major [T][rows][Vl] -> logits rows [rows][T*Vl]
__global__ void k_interleave_shards(const float* __restrict__ in, int T, int64_t rows, int64_t Vl, float* __restrict__ out) {
  const int64_t n = T * rows * Vl;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (T * Vl), rem = i % (T * Vl), t = rem / Vl, v = rem % Vl;
    out[i] = in[(t * rows + r) * Vl + v];
  }
}
void interleave_shards(const float* in, int T, int64_t rows, int64_t Vl, float* out, cudaStream_t s) {
  const int64_t n = T * rows * Vl;
  if (n <= 0) return;
  k_interleave_shards<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 1184)), 256, 0, s>>>(in, T, rows, Vl,
                                                                                                      out);
  PCB_CUDA(cudaGetLastError());
}

__global__ void k_fill(float* d, uint64_t n, float v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    d[i] = v;
}
void fill_const(float* d, uint64_t n, float v, cudaStream_t s) {
  k_fill<<<592, 256, 0, s>>>(d, n, v);
  PCB_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// embed (model.cpp:354-362): h[i] = embed[tok[i]] (+ abs_table[pos[i]])
// ---------------------------------------------------------------------------
__global__ void k_embed(const int32_t* tok, const int32_t* pos, const float* table, const float* abs_table, int d,
                        float* h, const float* cos32, const float* sin32, int half, float2* rope_tab, int64_t rope_ld) {
  pdl_trigger();
  pdl_wait();
  int64_t i = blockIdx.x;
  const float* e = table + static_cast<int64_t>(tok[i]) * d;
  if (!abs_table && (d & 3) == 0) {  // 16-byte copies of the embedding row
    const float4* e4 = reinterpret_cast<const float4*>(e);
    float4* h4 = reinterpret_cast<float4*>(h + i * d);
#pragma unroll 4
    for (int j = threadIdx.x; j < (d >> 2); j += blockDim.x) h4[j] = e4[j];
  } else {
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
      float v = e[j];
      if (abs_table) v = __fadd_rn(v, abs_table[static_cast<int64_t>(pos[i]) * d + j]);
      h[i * d + j] = v;
    }
  }
  if (rope_tab) {
    const int64_t p = static_cast<int64_t>(pos[i]) * half;
    for (int j = threadIdx.x; j < half; j += blockDim.x) rope_tab[j * rope_ld + i] = make_float2(cos32[p + j], sin32[p + j]);
  }
}
void embed(const int32_t* tok, const int32_t* pos, int64_t n, const float* table, const float* abs_table, int d,
           float* h, cudaStream_t s, const float* cos32, const float* sin32, int half, float2* rope_tab,
           int64_t rope_ld) {
  if (n <= 0) return;
  PdlClass pc(PDL_EMBED);
  launch_k(k_embed, dim3(static_cast<unsigned>(n)), dim3(256), 0, s, 1, tok, pos, table, abs_table, d, h, cos32, sin32,
           half, rope_tab, rope_ld);
  PCB_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// LayerNorm (model.cpp:156-174): fp64 mean / variance, eps 1e-5, gamma 1, beta 0.
// ---------------------------------------------------------------------------
// One CTA per row; the row is read once into registers (up to 8 float4 per thread,
// d <= 8192 at 256 threads), with two block reductions (sum, centred sum of squares).
constexpr int kLnThreads = 256, kLnVec = 8;

__device__ __forceinline__ double ln_block_sum(double v, double* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0;
#pragma unroll
  for (int w = 0; w < kLnThreads / 32; ++w) t += red[w];
  __syncthreads();
  return t;
}

template <typename T>
__global__ void __launch_bounds__(kLnThreads) k_layernorm(const float* h, int d, T* out) {
  pdl_trigger();
  pdl_wait();
  __shared__ double red[kLnThreads / 32];
  const float* row = h + static_cast<int64_t>(blockIdx.x) * d;
  T* orow = out + static_cast<int64_t>(blockIdx.x) * d;
  const int nv = d >> 2;  // float4s in the row (d % 4 == 0 on this path)
  float4 x[kLnVec];
  double s = 0;
#pragma unroll
  for (int u = 0; u < kLnVec; ++u) {
    const int i = threadIdx.x + u * kLnThreads;
    x[u] = i < nv ? reinterpret_cast<const float4*>(row)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    s += (double)x[u].x + (double)x[u].y + (double)x[u].z + (double)x[u].w;
  }
  const double mean = ln_block_sum(s, red) / d;
  double v = 0;
#pragma unroll
  for (int u = 0; u < kLnVec; ++u)
    if (threadIdx.x + u * kLnThreads < nv) {
      const double a = x[u].x - mean, b = x[u].y - mean, c = x[u].z - mean, e = x[u].w - mean;
      v += a * a + b * b + c * c + e * e;
    }
  const double inv = 1.0 / sqrt(ln_block_sum(v, red) / d + 1e-5);
#pragma unroll
  for (int u = 0; u < kLnVec; ++u) {
    const int i = threadIdx.x + u * kLnThreads;
    if (i < nv) {
      const float a = static_cast<float>((x[u].x - mean) * inv), b = static_cast<float>((x[u].y - mean) * inv);
      const float c = static_cast<float>((x[u].z - mean) * inv), e = static_cast<float>((x[u].w - mean) * inv);
      if constexpr (std::is_same_v<T, float>) {  // one 16-byte store per 4 elements
        reinterpret_cast<float4*>(orow)[i] = make_float4(a, b, c, e);
      } else {  // bf16: one 8-byte store (2-byte stores left the kernel at ~2.2 TB/s)
        __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, e);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&lo);
        pk.y = *reinterpret_cast<uint32_t*>(&hi);
        reinterpret_cast<uint2*>(orow)[i] = pk;
      }
    }
  }
}

// gathered rows: out row i = LN(h row rows[i]) (rows null: the single row row_last)
template <typename T>
__global__ void __launch_bounds__(kLnThreads) k_layernorm_rows(const float* h, const int32_t* rows, int64_t row_last,
                                                                 int d, T* out) {
  pdl_trigger();
  pdl_wait();
  __shared__ double red[kLnThreads / 32];
  const int64_t r = rows ? rows[blockIdx.x] : row_last;
  const float* row = h + r * d;
  double s = 0;
  for (int j = threadIdx.x; j < d; j += kLnThreads) s += row[j];
  const double mean = ln_block_sum(s, red) / d;
  double v = 0;
  for (int j = threadIdx.x; j < d; j += kLnThreads) {
    const double c = row[j] - mean;
    v += c * c;
  }
  const double inv = 1.0 / sqrt(ln_block_sum(v, red) / d + 1e-5);
  for (int j = threadIdx.x; j < d; j += kLnThreads)
    st_f(out, static_cast<int64_t>(blockIdx.x) * d + j, static_cast<float>((row[j] - mean) * inv));
}

// general-d fallback (d % 4 != 0 or d > 8192): three strided passes
template <typename T>
__global__ void __launch_bounds__(kLnThreads) k_layernorm_any(const float* h, int d, T* out) {
  pdl_trigger();
  pdl_wait();
  __shared__ double red[kLnThreads / 32];
  const float* row = h + static_cast<int64_t>(blockIdx.x) * d;
  double s = 0;
  for (int j = threadIdx.x; j < d; j += kLnThreads) s += row[j];
  const double mean = ln_block_sum(s, red) / d;
  double v = 0;
  for (int j = threadIdx.x; j < d; j += kLnThreads) {
    const double c = row[j] - mean;
    v += c * c;
  }
  const double inv = 1.0 / sqrt(ln_block_sum(v, red) / d + 1e-5);
  for (int j = threadIdx.x; j < d; j += kLnThreads)
    st_f(out, static_cast<int64_t>(blockIdx.x) * d + j, static_cast<float>((row[j] - mean) * inv));
}
void layernorm(int dtype, const float* h, int64_t n, int d, void* out, cudaStream_t s) {
  if (n <= 0) return;
  PdlClass pc(PDL_LN);
  const bool fast = d % 4 == 0 && d <= 4 * kLnVec * kLnThreads;
  const dim3 g(static_cast<unsigned>(n)), b(kLnThreads);
  if (dtype == F32)
    launch_k(fast ? k_layernorm<float> : k_layernorm_any<float>, g, b, 0, s, 1, h, d, static_cast<float*>(out));
  else
    launch_k(fast ? k_layernorm<__nv_bfloat16> : k_layernorm_any<__nv_bfloat16>, g, b, 0, s, 1, h, d,
             static_cast<__nv_bfloat16*>(out));
  PCB_CUDA(cudaGetLastError());
}

void layernorm_rows(int dtype, const float* h, const int32_t* rows, int64_t n, int d, void* out, cudaStream_t s,
                    int64_t row_last) {
  if (n <= 0) return;
  PdlClass pc(PDL_LN);
  const dim3 g(static_cast<unsigned>(n)), b(kLnThreads);
  if (dtype == F32)
    launch_k(k_layernorm_rows<float>, g, b, 0, s, 1, h, rows, row_last, d, static_cast<float*>(out));
  else
    launch_k(k_layernorm_rows<__nv_bfloat16>, g, b, 0, s, 1, h, rows, row_last, d, static_cast<__nv_bfloat16*>(out));
  PCB_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// argmax_lowest (model.cpp:457-462): ties break to the lowest index.
// ---------------------------------------------------------------------------
__global__ void k_argmax(const float* logits, int V, int32_t* out) {
  pdl_trigger();
  pdl_wait();
  const float* row = logits + static_cast<int64_t>(blockIdx.x) * V;
  float best = -INFINITY;
  int bi = 0x7fffffff;
  auto take = [&](float v, int i) {
    if (v > best || (v == best && i < bi)) {
      best = v;
      bi = i;
    }
  };
  if ((V & 3) == 0 && (reinterpret_cast<uintptr_t>(row) & 15) == 0) {
    // 16-byte loads, all of a thread's loads in flight before the compares
    const float4* r4 = reinterpret_cast<const float4*>(row);
    const int n4 = V >> 2;
#pragma unroll 8
    for (int i = threadIdx.x; i < n4; i += blockDim.x) {
      const float4 v = r4[i];
      take(v.x, 4 * i);
      take(v.y, 4 * i + 1);
      take(v.z, 4 * i + 2);
      take(v.w, 4 * i + 3);
    }
  } else {
    for (int i = threadIdx.x; i < V; i += blockDim.x) take(row[i], i);
  }
  for (int o = 16; o; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) {
      best = ov;
      bi = oi;
    }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (sv[w] > best || (sv[w] == best && si[w] < bi)) {
        best = sv[w];
        bi = si[w];
      }
    out[blockIdx.x] = bi == 0x7fffffff ? 0 : bi;
  }
}
void argmax_rows(const float* logits, int64_t rows, int V, int32_t* out, cudaStream_t s) {
  if (rows <= 0) return;
  PdlClass pc(PDL_ARGMAX);
  launch_k(k_argmax, dim3(static_cast<unsigned>(rows)), dim3(1024), 0, s, 1, logits, V, out);
  PCB_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// GEMM epilogue on an adjacent column pair (n, n+1), n even.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void epi_pair(const Epilogue& e, int64_t m, int n, int N, float v0, float v1) {
  switch (e.kind) {
    case EPI_QKV: {
      const int seg = n / e.d, c = n - seg * e.d;
      if (seg < 2 && e.rope) {
        const int half = e.head_dim / 2;
        const int i = (c % e.head_dim) >> 1;
        const int64_t p = e.pos[m];
        if (e.rope_cos64) {
          double cs = e.rope_cos64[p * half + i], sn = e.rope_sin64[p * half + i];
          double a = v0, b = v1;
          v0 = static_cast<float>(__dsub_rn(__dmul_rn(a, cs), __dmul_rn(b, sn)));
          v1 = static_cast<float>(__dadd_rn(__dmul_rn(a, sn), __dmul_rn(b, cs)));
        } else {
          float cs = e.rope_cos32[p * half + i], sn = e.rope_sin32[p * half + i];
          float a = v0, b = v1;
          v0 = a * cs - b * sn;
          v1 = a * sn + b * cs;
        }
      }
      T* dst = seg == 0 ? static_cast<T*>(e.q_out) + m * e.d
                        : static_cast<T*>(seg == 1 ? e.k_out : e.v_out) + (e.kv_off ? e.kv_off[m] : (e.kv_row0 + m) * e.d);
      st_f(dst, c, v0);
      st_f(dst, c + 1, v1);
      return;
    }
    case EPI_RESID: {
      float* r = e.resid + m * N + n;
      r[0] = __fadd_rn(r[0], v0);
      r[1] = __fadd_rn(r[1], v1);
      return;
    }
    case EPI_GELU: {
      T* o = static_cast<T*>(e.out) + m * N + n;
      if constexpr (sizeof(T) == 4) {
        st_f(o, 0, gelu_ref(v0));
        st_f(o, 1, gelu_ref(v1));
      } else {
        st_f(o, 0, gelu_fast(v0));
        st_f(o, 1, gelu_fast(v1));
      }
      return;
    }
    default:
      e.outf[m * e.ldo + n] = v0;
      e.outf[m * e.ldo + n + 1] = v1;
  }
}

// ---------------------------------------------------------------------------
// SIMT GEMM.  Block = 16x16 threads; each thread owns one row and a column
// pair.  F32: four fp64 lane accumulators per output over k = 4j+lane, combined
// ((s0+s1)+(s2+s3)) — the reference dotf (model.cpp:136-147) bit for bit.
// ---------------------------------------------------------------------------
constexpr int TM = 16, TN = 32, TK = 32;

template <typename T, bool EXACT>
__global__ void k_gemm_simt(const T* __restrict__ A, const T* __restrict__ W, int64_t M, int N, int K, Epilogue e,
                            bool w_packed) {
  pdl_trigger();
  pdl_wait();
  auto widx = [&](int64_t n, int64_t k) -> int64_t {
    return w_packed ? static_cast<int64_t>(packed_index(static_cast<int>(n), static_cast<int>(k), K)) : n * K + k;
  };
  __shared__ float sA[TM][TK + 1];
  __shared__ float sW[TN][TK + 1];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t m = blockIdx.y * (int64_t)TM + ty;
  const int n0 = blockIdx.x * TN + 2 * tx;
  using Acc = typename std::conditional<EXACT, double, float>::type;
  Acc a0[4] = {0, 0, 0, 0}, a1[4] = {0, 0, 0, 0};
  const int K4 = K - (K & 3);
  for (int k0 = 0; k0 < K4; k0 += TK) {
    const int tid = ty * 16 + tx;
    for (int idx = tid; idx < TM * TK; idx += 256) {
      int r = idx / TK, c = idx % TK;
      int64_t gm = blockIdx.y * (int64_t)TM + r;
      sA[r][c] = (gm < M && k0 + c < K4) ? ld_f(A, gm * K + k0 + c) : 0.f;
    }
    for (int idx = tid; idx < TN * TK; idx += 256) {
      int r = idx / TK, c = idx % TK;
      int gn = blockIdx.x * TN + r;
      sW[r][c] = (gn < N && k0 + c < K4) ? ld_f(W, widx(gn, k0 + c)) : 0.f;
    }
    __syncthreads();
    const int kmax = min(TK, K4 - k0);
#pragma unroll 4
    for (int kk = 0; kk < kmax; kk += 4) {
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        Acc x = sA[ty][kk + l];
        a0[l] += x * (Acc)sW[2 * tx][kk + l];
        a1[l] += x * (Acc)sW[2 * tx + 1][kk + l];
      }
    }
    __syncthreads();
  }
  if (m >= M || n0 >= N) return;
  for (int k = K4; k < K; ++k) {  // reference tail goes to lane 0
    Acc x = ld_f(A, m * K + k);
    a0[0] += x * (Acc)ld_f(W, widx(n0, k));
    a1[0] += x * (Acc)ld_f(W, widx(n0 + 1, k));
  }
  float v0 = static_cast<float>((a0[0] + a0[1]) + (a0[2] + a0[3]));
  float v1 = static_cast<float>((a1[0] + a1[1]) + (a1[2] + a1[3]));
  epi_pair<T>(e, m, n0, N, v0, v1);
}

void gemm_simt(int dtype, const void* A, const void* W, int64_t M, int N, int K, const Epilogue& e,
               cudaStream_t s, bool w_packed) {
  if (M <= 0) return;
  dim3 grid((N + TN - 1) / TN, static_cast<unsigned>((M + TM - 1) / TM));
  dim3 block(16, 16);
  if (dtype == F32)
    launch_k(k_gemm_simt<float, true>, grid, block, 0, s, 1, static_cast<const float*>(A), static_cast<const float*>(W),
             M, N, K, e, false);
  else
    launch_k(k_gemm_simt<__nv_bfloat16, false>, grid, block, 0, s, 1, static_cast<const __nv_bfloat16*>(A),
             static_cast<const __nv_bfloat16*>(W), M, N, K, e, w_packed);
  PCB_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// SIMT attention (model.cpp:401-427).  One block per (head, query).  Scores are
// dotf(q, k_j) in fp32 storage (F32: fp64 4-lane dot), scaled by 1/sqrt(hd) in
// fp32; softmax weights in fp64 (F32) / fp32 (BF16); each output lane then
// accumulates w_j * v_j[x] and the denominator over j in sequence order.
// ---------------------------------------------------------------------------
template <typename T, bool EXACT>
__global__ void k_attn_simt(AttnArgs a, float inv_sqrt, float* scratch_f) {
  pdl_trigger();
  pdl_wait();
  using Acc = typename std::conditional<EXACT, double, float>::type;
  const int h = blockIdx.x;
  const int64_t i = a.i0 + blockIdx.y;
  const int64_t total = a.P + a.n;
  const T* q = static_cast<const T*>(a.q) + i * a.d + h * a.hd;
  const T* K = static_cast<const T*>(a.k);
  const T* V = static_cast<const T*>(a.v);
  Acc* w = reinterpret_cast<Acc*>(scratch_f) + (static_cast<int64_t>(blockIdx.y) * a.H + h) * total;
  const int64_t qrow = a.P + i;
  const int64_t limit = a.mask ? a.n - 1 : qrow;
  auto allowed = [&](int64_t j) -> bool {
    if (a.mask) return a.mask[i * a.n + j] != 0;
    if (a.block_id) {
      int bi = a.block_id[qrow], bj = a.block_id[j];
      return bi < 0 || bi == bj;
    }
    return true;
  };
  __shared__ Acc red[32];
  Acc mx = -1e30;
  for (int64_t j = threadIdx.x; j <= limit; j += blockDim.x) {
    if (!allowed(j)) continue;
    const T* kr = K + j * a.d + h * a.hd;
    Acc l[4] = {0, 0, 0, 0};
    int x = 0;
    for (; x + 4 <= a.hd; x += 4)
#pragma unroll
      for (int u = 0; u < 4; ++u) l[u] += (Acc)ld_f(q, x + u) * (Acc)ld_f(kr, x + u);
    for (; x < a.hd; ++x) l[0] += (Acc)ld_f(q, x) * (Acc)ld_f(kr, x);
    float sc = __fmul_rn(static_cast<float>((l[0] + l[1]) + (l[2] + l[3])), inv_sqrt);
    if (a.alibi) sc = __fadd_rn(sc, __fmul_rn(a.alibi[h], static_cast<float>(a.kv_pos[j] - a.kv_pos[qrow])));
    w[j] = sc;
    mx = sc > mx ? (Acc)sc : mx;
  }
  for (int o = 16; o; o >>= 1) {
    Acc t = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = t > mx ? t : mx;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = red[0];
  for (int t = 1; t < (int)(blockDim.x >> 5); ++t) mx = red[t] > mx ? red[t] : mx;
  for (int64_t j = threadIdx.x; j <= limit; j += blockDim.x) {
    if (!allowed(j)) continue;
    if constexpr (EXACT)
      w[j] = exp(w[j] - mx);
    else
      w[j] = __expf(w[j] - mx);
  }
  __syncthreads();
  for (int x = threadIdx.x; x < a.hd; x += blockDim.x) {
    Acc acc = 0, den = 0;
    const T* vc = V + h * a.hd + x;
    for (int64_t j = 0; j <= limit; ++j) {
      if (!allowed(j)) continue;
      Acc wj = w[j];
      den += wj;
      acc += wj * (Acc)ld_f(vc, j * a.d);
    }
    st_f(static_cast<T*>(a.out), i * a.d + h * a.hd + x, static_cast<float>(acc / den));
  }
}

size_t attention_simt_scratch(const AttnArgs& a) {
  return static_cast<size_t>(a.nq < 0 ? a.n : a.nq) * a.H * (a.P + a.n) * sizeof(double);
}

void attention_simt(int dtype, const AttnArgs& a, float* scratch, cudaStream_t s) {
  const int64_t nq = a.nq < 0 ? a.n : a.nq;
  if (nq <= 0) return;
  dim3 grid(a.H, static_cast<unsigned>(nq));
  float inv_sqrt = 1.0f / sqrtf(static_cast<float>(a.hd));
  if (dtype == F32)
    launch_k(k_attn_simt<float, true>, grid, dim3(128), 0, s, 1, a, inv_sqrt, scratch);
  else
    launch_k(k_attn_simt<__nv_bfloat16, false>, grid, dim3(128), 0, s, 1, a, inv_sqrt, scratch);
  PCB_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// KV assembly (reference concat_kv, engine.cpp:174-185, + KVState::append).
// Persistent grid of 148*k CTAs walks 32 KiB chunks of the concatenated segment
// list; each thread streams 16-byte vectors with 8 loads in flight, L1 bypassed.
// Bound: HBM (read + write every byte once).
// ---------------------------------------------------------------------------
constexpr uint64_t kChunk = 32768;

__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(int4* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

__global__ void __launch_bounds__(256) k_assemble(const CopySeg* __restrict__ segs, const uint64_t* __restrict__ first_chunk,
                                                  int n_segs, uint64_t n_chunks) {
  pdl_trigger();
  pdl_wait();
  for (uint64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    int lo = 0, hi = n_segs - 1;  // last segment with first_chunk <= c
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (first_chunk[mid] <= c) lo = mid;
      else hi = mid - 1;
    }
    const CopySeg sg = segs[lo];
    const uint64_t off = (c - first_chunk[lo]) * kChunk;
    const uint64_t len = min(kChunk, sg.bytes - off);
    const int4* src = reinterpret_cast<const int4*>(static_cast<const char*>(sg.src) + off);
    int4* dst = reinterpret_cast<int4*>(static_cast<char*>(sg.dst) + off);
    const uint64_t nv = len / 16;
    if (nv == kChunk / 16) {
      int4 r[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) r[u] = ld_stream(src + threadIdx.x + u * 256);
#pragma unroll
      for (int u = 0; u < 8; ++u) st_stream(dst + threadIdx.x + u * 256, r[u]);
    } else {
      for (uint64_t v = threadIdx.x; v < nv; v += 256) st_stream(dst + v, ld_stream(src + v));
    }
  }
}

uint64_t assemble_plan(const CopySeg* segs, int n_segs, uint64_t* first_chunk) {
  uint64_t c = 0;
  for (int i = 0; i < n_segs; ++i) {
    first_chunk[i] = c;
    c += (segs[i].bytes + kChunk - 1) / kChunk;
  }
  return c;
}

void assemble(const CopySeg* d_segs, const uint64_t* d_first_chunk, int n_segs, uint64_t n_chunks, cudaStream_t s) {
  if (n_chunks == 0) return;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t grid = std::min<uint64_t>(n_chunks, static_cast<uint64_t>(sms) * 8);
  PdlClass pc(PDL_ASM);
  launch_k(k_assemble, dim3(static_cast<unsigned>(grid)), dim3(256), 0, s, 1, d_segs, d_first_chunk, n_segs, n_chunks);
  PCB_CUDA(cudaGetLastError());
}

// Row gather for the decode working cache (reference assemble_working,
// engine.cpp:65-97): for every plane p (layer x K/V), dst[p][r] = src[p][map[r]].
__global__ void k_gather_map(const char* src, int64_t src_cap, char* dst, int64_t dst_cap, const int32_t* map,
                             int64_t row_bytes) {
  const int64_t r = blockIdx.x, p = blockIdx.y;
  const int4* s4 = reinterpret_cast<const int4*>(src + (p * src_cap + map[r]) * row_bytes);
  int4* d4 = reinterpret_cast<int4*>(dst + (p * dst_cap + r) * row_bytes);
  for (int64_t v = threadIdx.x; v < row_bytes / 16; v += blockDim.x) d4[v] = s4[v];
}
void gather_map(const void* src, int64_t src_cap, void* dst, int64_t dst_cap, const int32_t* d_map, int64_t rows,
                int64_t row_bytes, int planes, cudaStream_t s) {
  if (rows <= 0) return;
  dim3 grid(static_cast<unsigned>(rows), planes);
  k_gather_map<<<grid, 128, 0, s>>>(static_cast<const char*>(src), src_cap, static_cast<char*>(dst), dst_cap, d_map,
                                    row_bytes);
  PCB_CUDA(cudaGetLastError());
}

template <typename S, typename D>
__global__ void k_convert(const S* src, D* dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    st_f(dst, static_cast<int64_t>(i), ld_f(src, static_cast<int64_t>(i)));
}
void convert(int sd, const void* src, int dd, void* dst, uint64_t n, cudaStream_t s) {
  if (!n) return;
  if (sd == dd) {
    PCB_CUDA(cudaMemcpyAsync(dst, src, n * dtype_size(sd), cudaMemcpyDeviceToDevice, s));
    return;
  }
  if (sd == F32)
    k_convert<<<592, 256, 0, s>>>(static_cast<const float*>(src), static_cast<__nv_bfloat16*>(dst), n);
  else
    k_convert<<<592, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(src), static_cast<float*>(dst), n);
  PCB_CUDA(cudaGetLastError());
}

}  // namespace pcb::kern

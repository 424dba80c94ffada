// Device kernel entry points of the Prompt Cache hot path (sm_100a).
//
// Data layout in HBM:
//   weights   W[out][in] row-major (K-major for the tensor cores), bf16 or fp32;
//             per layer Wqkv fused [3d][d] (q rows, k rows, v rows), Wo [d][d],
//             W1 [4d][d], W2 [d][4d]; embed fp32 [V][d]; unembed [V][d].
//   KV block  [L][2][cap][d] (layer, K/V, row, head-interleaved hidden) — the
//             same layout for store entries and a request's assembled cache, so
//             KV assembly is one contiguous copy per (module, layer, K/V).
//   residual  fp32 [n][d]; activations in the model dtype.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace pcb::kern {

enum DType : int { F32 = 0, BF16 = 1 };

inline size_t dtype_size(int dt) { return dt == F32 ? 4 : 2; }

enum EpiKind : int {
  EPI_QKV = 0,     // N = 3d: q -> q_out[m][n]; k,v -> cache rows kv_row0+m; RoPE on q,k
  EPI_RESID = 1,   // resid[m][n] += acc
  EPI_GELU = 2,    // out[m][n] = gelu(acc)   (model dtype)
  EPI_F32 = 3,     // outf[m*ldo + n] = acc   (fp32 logits)
  EPI_NONE = 4,    // discard (timing probes only)
};

struct Epilogue {
  int kind = EPI_F32;
  int d = 0;  // hidden (EPI_QKV)
  void* q_out = nullptr;
  void* k_out = nullptr;  // layer K base of the cache, row stride d
  void* v_out = nullptr;
  int64_t kv_row0 = 0;
  const int64_t* kv_off = nullptr;  // batched: per token K/V element offset from k_out/v_out (row-major d)
  const int32_t* pos = nullptr;  // per token (EPI_QKV rope)
  int rope = 0;                  // apply RoPE
  int head_dim = 0;
  const double* rope_cos64 = nullptr;  // [max_pos][hd/2] (F32 path)
  const double* rope_sin64 = nullptr;
  const float* rope_cos32 = nullptr;   // (BF16 path)
  const float* rope_sin32 = nullptr;
  // per-request rows of the two tables: rope_tab[pair][m] = {cos, sin} of token m's position
  // (written by embed; contiguous in m, so a 16-token chunk is 8 vector loads, no pos lookup)
  const float2* rope_tab = nullptr;
  int64_t rope_ld = 0;  // multiple of 16
  float* resid = nullptr;
  void* out = nullptr;
  float* outf = nullptr;
  int64_t ldo = 0;
  // LayerNorm folded into the neighbouring GEMMs (chain kernel, bf16):
  //   EPI_RESID with x_out: also x_out[m][n] = bf16(new residual) (the next GEMM's raw input)
  //   ln_wsum (consumer):   acc -> rstd[m] * (acc - mean[m] * ln_wsum[n]),  ln_wsum[n] = sum_k W[n][k]
  //                         = LN(h) . W^T  (gamma 1, beta 0), row statistics passed per chunk
  void* x_out = nullptr;
  const float* ln_wsum = nullptr;
};

// ---- weights (PCG32 jump-ahead; bit-identical to the reference's fill_uniform) ----
void init_uniform(int dtype, void* dst, uint64_t count, uint64_t stream_seed, float scale, cudaStream_t s);
void fill_const(float* dst, uint64_t count, float v, cudaStream_t s);
void init_uniform_block(int dtype, void* dst, int64_t rows, int64_t cols, uint64_t seed, float scale, int64_t row0,
                        int64_t col0, int64_t full_cols, cudaStream_t s);
// tensor parallel helpers
void add_inplace(float* h, const float* part, int64_t n, cudaStream_t s);
void interleave_shards(const float* in, int T, int64_t rows, int64_t Vl, float* out, cudaStream_t s);

// ---- small ops ----
// rope_tab (optional): also rope_tab[j * rope_ld + i] = {cos32, sin32}[pos[i] * half + j], j < half
void embed(const int32_t* tok, const int32_t* pos, int64_t n, const float* table, const float* abs_table,
           int d, float* h, cudaStream_t s, const float* cos32 = nullptr, const float* sin32 = nullptr, int half = 0,
           float2* rope_tab = nullptr, int64_t rope_ld = 0);
// out = LN(h) (gamma=1, beta=0, eps 1e-5), rows [row0, row0+n)
void layernorm(int dtype, const float* h, int64_t n, int d, void* out, cudaStream_t s);
// out[n] = sum_k W[n][k] of a row-major bf16 [N][K] matrix (fp32, LN-fold weight sums)
void row_sums_bf16(const void* W, int N, int K, float* out, cudaStream_t s);
// out[i] = LN(h[rows[i]]) for i < n (rows null: h row row_last for the single row)
void layernorm_rows(int dtype, const float* h, const int32_t* rows, int64_t n, int d, void* out, cudaStream_t s,
                    int64_t row_last);
void argmax_rows(const float* logits, int64_t rows, int V, int32_t* out, cudaStream_t s);

// ---- packed bf16 weights (the tcgen05 GEMM's HBM layout) ----
// W[n][k] lives in 128x64 tiles [N/128][K/64], 16 KB each, each tile the SW128
// K-major shared-memory image: row r at r*128 B, 16-byte chunk c at (c ^ (r & 7)).
__host__ __device__ inline uint64_t packed_index(int n, int k, int K) {
  const int tn = n >> 7, r = n & 127, tk = k >> 6, kk = k & 63;
  const int c = kk >> 3, e = kk & 7;
  return ((static_cast<uint64_t>(tn) * (K >> 6) + tk) * 16384ull + r * 128 + ((c ^ (r & 7)) << 4)) / 2 + e;
}
bool weight_packable(int N, int K);
void pack_weight_bf16(const void* src_rowmajor, void* dst_packed, int N, int K, cudaStream_t s);

// ---- GEMM: C[m][n] = sum_k A[m][k] * W[n][k] with a fused epilogue ----
// SIMT: F32 = fp64 accumulation in the reference's 4-lane order (bit-exact
// dot products); BF16 = fp32 accumulation (bring-up / odd shapes), W packed or not.
void gemm_simt(int dtype, const void* A, const void* W, int64_t M, int N, int K, const Epilogue& e,
               cudaStream_t s, bool w_packed = false);
// tcgen05 persistent stream-K GEMM (bf16 in, fp32 accumulate) over PACKED weights.
// Requires K%64==0, N%128==0.  workspace >= 148*128*256*4 bytes; flags >= #SMs ints (zeroed once).
bool gemm_tc_supported(int64_t M, int N, int K);
// CTA-pair (cta_group::2) 256x256-tile GEMM for M >= 256 over the same packed weights
// (gemm_2sm.cu); gemm_tc dispatches to it.
bool gemm_2sm_supported(int64_t M, int N, int K);
void gemm_2sm(const void* A, const void* W_packed, int64_t M, int N, int K, const Epilogue& e, cudaStream_t s);
// debug: GEMM timeline probe (PCB_GEMM_PROBE=1); shapes [n][4] = {M,N,K,ctas}, times [n][160][4]
int gemm_probe_dump(int64_t* shapes, unsigned long long* times, int max_launches);
void gemm_tc(const void* A, const void* W_packed, int64_t M, int N, int K, const Epilogue& e, float* workspace,
             size_t workspace_bytes, int* flags, cudaStream_t s);

// ---- persistent GEMM / LayerNorm chain (few-token regime, M <= 128) ----
// One launch runs the phases in order with a grid barrier between them; the packed
// weights of later phases stream in while earlier phases finish (chain_tc.cu).
enum ChainKind : int { CHAIN_GEMM = 0, CHAIN_LN = 1, CHAIN_ATTN = 2 };
constexpr int kChainMaxPhases = 48;  // phases per chain launch
struct ChainStep {
  int kind = CHAIN_GEMM;
  int64_t M = 0;             // rows (tokens)
  const void* x = nullptr;   // GEMM: activations [M][K] bf16
  const void* w = nullptr;   // GEMM: packed weights [N][K]
  int N = 0, K = 0;
  Epilogue e;                // GEMM epilogue
  const float* ln_src = nullptr;  // LN: fp32 rows [M][ln_d]
  void* ln_dst = nullptr;         // LN: bf16 rows [M][ln_d]
  int ln_d = 0;
  // folded LayerNorm (GEMM steps): a residual step (e.x_out set) writes {sum h, sum h^2} per
  // (128-column tile, token) to stats_out [tiles][stats_ld][2]; a consumer step (e.ln_wsum
  // set) reads stats_in rows [stats_row0, stats_row0 + M) of stats_tiles tiles, ln_dim wide
  float* stats_out = nullptr;
  const float* stats_in = nullptr;
  int stats_tiles = 0, stats_ld = 0, stats_row0 = 0, ln_dim = 0;
  // attention phase (CHAIN_ATTN; one request per launch, any position): M = n <= 128 new rows
  // of one request, causal against P cached rows; q / out [n][a_d], k / v the layer's cache
  // planes [P + n][a_d]; a_H heads of 128; a_scratch holds the split partials
  const void* aq = nullptr;
  const void* ak = nullptr;
  const void* av = nullptr;
  void* aout = nullptr;
  int64_t aP = 0;
  int aH = 0, a_d = 0;
  float* a_scratch = nullptr;
  size_t a_scratch_bytes = 0;
  // zero-copy prefix (a_nseg > 0): the keys are a_seg[0].rows, a_seg[1].rows, ... in order,
  // each read in place from a KV block ([layer][K|V][cap][d] planes) -- the cached modules
  // straight from the store -- and the last segment is the request cache's own rows, of
  // which the first a_tail_vis are visible to every query and the rest causally (ak / av
  // unused).  Replaces the KV assembly copy for a single request.
  struct KVSeg {
    const void* base = nullptr;
    int64_t cap = 0;
    size_t plane_bytes = 0;
    int64_t row0 = 0, rows = 0;
  };
  static constexpr int kMaxSeg = 8;
  // ALiBi (a_alibi = slopes [a_H]): a_kpos holds the keys' positions in key-block order (each
  // segment padded to whole 64-key blocks; readable through the last block), a_qpos the n
  // queries' positions
  const float* a_alibi = nullptr;
  const int32_t* a_kpos = nullptr;
  const int32_t* a_qpos = nullptr;
  int a_nseg = 0;
  int a_layer = 0, a_planes = 0;
  KVSeg a_seg[kMaxSeg];
  int64_t a_tail_vis = 0;
};
// can a chain run this request's attention as its first phase (#SMs >= heads, hd 128)?
bool chain_attn_supported(int64_t n, int64_t P, int H, int hd);
bool chain_tc_supported(int64_t M, int N, int K);
bool chain_ln_supported(int d);
// debug: chain timeline probe (PCB_CHAIN_PROBE=1): times [n][8 phases][160 CTAs][4]
int chain_probe_dump(unsigned long long* times, int max_launches, int* phases);
// flags: >= #SMs ints (zeroed once, private to the chain); gbar: one zeroed u64 whose
// arrival count the caller tracks in gbar_count (advanced by this call).
// a stream that launched chains is going away: drop it from the cross-stream chain ordering
void chain_forget_stream(cudaStream_t s);
void chain_tc(const ChainStep* steps, int n_steps, float* ws, size_t ws_bytes, int* flags,
              unsigned long long* gbar, unsigned long long& gbar_count, cudaStream_t s);

// ---- attention over a KV cache ----
// q [n][d]; K/V layer bases [rows][d]; query i (sequence index P+i) attends keys
// j <= P+i (sequence-order causality) or, with mask [n][n] (P must be 0), the
// allowed set.  ALiBi uses per-row positions.
struct AttnArgs {
  const void* q = nullptr;
  const void* k = nullptr;
  const void* v = nullptr;
  void* out = nullptr;
  int64_t n = 0, P = 0;
  int H = 0, hd = 0, d = 0;
  const uint8_t* mask = nullptr;
  const int32_t* block_id = nullptr;   // block-causal (oracle) variant: [P+n]
  const float* alibi = nullptr;        // [H] or null
  const int32_t* kv_pos = nullptr;     // [P+n] positions (alibi)
  int64_t i0 = 0, nq = -1;             // query sub-range [i0, i0+nq) (nq < 0: all n)
  int* counters = nullptr;             // tc split-KV: [H] zeroed arrival counters
  // batched (tc only): n_req requests in one launch; req[r] = {first q row, n, P, 0} on the
  // device; k/v = request 0's layer planes, request r's at + r * req_stride bytes (caches
  // of one capacity kv_cap); q/out hold all requests' rows; n = total q rows
  const int4* req = nullptr;
  int n_req = 0;
  int64_t req_stride = 0, kv_cap = 0, max_P = 0, max_n = 0;
  // batched zero-copy (k/v unused): per request <= 16 segments {map, row0, rows, zbase}
  // (segs [n_req][16] int4, segn [n_req] {count, tail visible rows}) over the global
  // CUtensorMap array maps; layer selects plane zbase + 2 layer (+1 for V)
  const int4* segs = nullptr;
  const int2* segn = nullptr;
  const void* maps = nullptr;
  int layer = 0;
  int64_t max_blocks = 0;  // longest request's key blocks (with per-segment padding)
  int pair = 1;  // paired-tile prefill kernel: 0 off, 1 when pairs x heads fill the SMs, 2 whenever it applies
};
constexpr int kAttnMaxSeg = 16;
// 3-D bf16 TMA map {cols, rows, planes} (plane stride in bytes), box {64, box_rows, 1}, SW128
CUtensorMap tmap_bf16_3d(const void* ptr, uint64_t cols, uint64_t rows, uint64_t planes, uint64_t plane_stride,
                         uint32_t box_rows);
void attention_simt(int dtype, const AttnArgs& a, float* scratch, cudaStream_t s);
size_t attention_simt_scratch(const AttnArgs& a);
bool attention_tc_supported(const AttnArgs& a);
void attention_tc(const AttnArgs& a, float* scratch, size_t scratch_bytes, cudaStream_t s);
// causal prefill over long query ranges (hd 128): two 128-query tiles per CTA (attn_prefill.cu)
bool attention_prefill_supported(const AttnArgs& a, int sms);
// micro-batched suffix attention (<= 64 rows per request, hd 128): persistent over (request, head)
bool attention_batch_supported(const AttnArgs& a);
void attention_batch(const AttnArgs& a, cudaStream_t s);
void attention_prefill(const AttnArgs& a, cudaStream_t s);
int attn_tl_dump(unsigned long long* out, int max_ctas);  // debug: last launch's per-CTA phases (PCB_ATTN_TL)

// ---- KV assembly: batched contiguous copies (one descriptor per segment) ----
struct CopySeg {
  const void* src;
  void* dst;
  uint64_t bytes;  // multiple of 16
};
// Host planning: fills first_chunk[i] (chunk index where segment i starts) and
// returns the total chunk count.  Segment bytes must be multiples of 16.
uint64_t assemble_plan(const CopySeg* segs, int n_segs, uint64_t* first_chunk);
void assemble(const CopySeg* d_segs, const uint64_t* d_first_chunk, int n_segs, uint64_t n_chunks, cudaStream_t s);
// Row gather across all 2L planes of a KV block: dst[p][r] = src[p][map[r]],
// used for the decode working cache (reference assemble_working, engine.cpp:65-97).
void gather_map(const void* src, int64_t src_cap, void* dst, int64_t dst_cap, const int32_t* d_map, int64_t rows,
                int64_t row_bytes, int planes, cudaStream_t s);

// Convert between storage types (fp32 <-> bf16) for host interchange.
void convert(int src_dtype, const void* src, int dst_dtype, void* dst, uint64_t count, cudaStream_t s);

}  // namespace pcb::kern

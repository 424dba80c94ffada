// tcgen05 flash attention for the bf16 hot path: a 128-query tile of one head
// against a range of key rows of the assembled cache (reference model.cpp:401-427:
// causal by sequence order, query i sees keys j <= P + i).
//
//   warp 0     TMA: Q tile once, then K/V blocks of 64 keys (ring as deep as smem allows)
//   warp 1     TMEM alloc + MMA issue: S_j = Q K_j^T (M=128, N=64, K=hd) into one of
//              three TMEM score buffers, O += P_j V_j (M=128, N=hd, K=64; P is the A
//              operand straight from TMEM, V an MN-major smem operand) accumulated in TMEM
//   warps 2-5  softmax: one thread per query row (TMEM lane); online max/sum in
//              fp32, P_j (bf16) written back over the first 32 columns of S_j
// Pipelining: S(j+2) is issued right after PV(j), so the scores of block j+1 are ready
// when the softmax of block j ends.  The running max is rescaled lazily: O (in TMEM) is
// corrected only when a row's max grows by more than 2^8, so the common step never touches O.
// Suffix prefill (few queries, long cache) splits the key range across the CTAs of a
// cluster and merges the (O, m, l) partials through DSMEM in split order (deterministic).
// Prefill (P = 0) tiles queries and skips blocks above the diagonal; long prefills use the
// paired-tile kernel (attn_prefill.cu).
#include <cuda.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace pcb::kern {

using namespace tc;
CUtensorMap tmap_bf16_2d(const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows);

namespace {

constexpr int BQ = 128, BKV = 64, kAttnThreads = 192;
constexpr int kSmemMax = 232448;  // 227 KB opt-in dynamic shared memory per CTA
#ifndef PCB_ATTN_STAGES
#define PCB_ATTN_STAGES 6
#endif
constexpr float kRescaleThreshold = 8.0f;  // log2 domain: stale max tolerated up to 2^8
constexpr int kSeg = 16;                    // K/V segments per request (zero-copy batched mode)

template <int HD, bool AL>
struct AttnSmem {
  static constexpr int kAtoms = HD / 64;
  static constexpr int kQ = BQ * HD * 2;
  static constexpr int kKV = BKV * HD * 2;
  static constexpr int kStage = 2 * kKV;  // K + V
  static constexpr int kPos = AL ? BKV * 4 : 0;  // ALiBi: the stage's key positions (int32)
  // as many K/V stages as fit next to Q (a stage is held from its TMA load through the PV
  // MMA, so depth is what keeps HBM busy on long caches); P lives in TMEM
  static constexpr int kStagesFit = (kSmemMax - kQ - 2048) / (kStage + kPos);
  static constexpr int kStages = kStagesFit > PCB_ATTN_STAGES ? PCB_ATTN_STAGES : kStagesFit;
  static constexpr int kBytes = kQ + kStages * (kStage + kPos) + 1024 + 1024;
  // three 64-column score buffers (P written back over the first 32 columns of its buffer)
  // and O: 3 BKV + HD columns
  static constexpr uint32_t kTmemCols = 3 * BKV + HD <= 256 ? 256 : 512;
};

struct AttnParams {
  int64_t n, P, total;
  int H, d;
  int splits;
  float scale_log2;  // log2(e) / sqrt(hd)
  __nv_bfloat16* out;
  float* part_o;   // [H][splits][BQ][HD]
  float* part_ml;  // [H][splits][BQ][2]
  int* counters;    // [H] split arrival counters (zero between launches)
  // batched requests (one launch for a micro-batch): blockIdx.x = request, per request
  // {first q row, n, P}; K/V come from a 3-D tensor map {d, rows, request}
  const int4* req = nullptr;
  // batched zero-copy: request r's keys are segments segs[r][0 .. segn[r].x) = {map, row0,
  // rows, zbase} read in place through maps[map] (3-D {d, cap, planes}, plane zbase + 2 layer
  // + K/V); the last segment is the request's own rows, the first segn[r].y of them visible
  // to every query, the rest causal
  const int4* segs = nullptr;
  const int2* segn = nullptr;
  const CUtensorMap* maps = nullptr;
  int layer = 0;
  // ALiBi (reference model.cpp:231-235, 410-411): score += slope_h (pos_key - pos_query);
  // kv_pos[P + n] holds every key's position in key order (the queries are keys P..P+n-1),
  // readable up to the last 64-key block (the producer copies whole blocks)
  const float* alibi = nullptr;
  const int32_t* kv_pos = nullptr;
  // duplicated queries (batched requests of <= 64 rows, one split): the Q tile holds the
  // request's rows twice; TMEM lanes [0, 64) take keys [0, 32) of every 64-key block and
  // lanes [64, 128) keys [32, 64), and the two halves of a query merge at the end -- all
  // four softmax warps work, each on half a block (with one copy, half the lanes idled)
  int dup = 0;
  unsigned long long* dbg = nullptr;  // timeline probe (CTA 0): [event][iteration] globaltimer ns
  unsigned long long* tl = nullptr;   // per-CTA phase timeline [cta][8] (PCB_ATTN_TL)
};

__device__ __forceinline__ void tlm(const AttnParams& p, int ev) {
  if (p.tl) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const int cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    p.tl[cta * 8 + ev] = t;
  }
}
__device__ __forceinline__ void probe(const AttnParams& p, int ev, int it) {
  if (p.dbg && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && it < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.dbg[ev * 64 + it] = t;
  }
}

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

template <int HD, bool AL>
__global__ void __launch_bounds__(kAttnThreads, 1)
    k_attn_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
              const __grid_constant__ CUtensorMap tmV, AttnParams p) {
  using S = AttnSmem<HD, AL>;
  constexpr int KV_STAGES = S::kStages;
  constexpr int kRedRow = HD + 4;  // padded fp32 row of a parked partial O
  static_assert(BQ * (kRedRow + 2) * 4 <= KV_STAGES * S::kStage, "split merge buffer must fit the K/V stages");
  extern __shared__ uint8_t smem_raw[];
  // pointer arithmetic on the __shared__ symbol (not an integer round trip) keeps the
  // shared address space visible to the compiler: LDS/STS instead of generic LD/ST
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + S::kQ;
  int32_t* sPos = reinterpret_cast<int32_t*>(sKV + KV_STAGES * S::kStage);  // [KV_STAGES][BKV] (ALiBi)
  uint64_t* bar = reinterpret_cast<uint64_t*>(sKV + KV_STAGES * S::kStage + KV_STAGES * S::kPos);
  uint64_t* q_full = bar;
  uint64_t* kv_full = bar + 1;                // [KV_STAGES]
  uint64_t* kv_empty = kv_full + KV_STAGES;   // [KV_STAGES]
  // Score buffer b (of 3) holds blocks it with it % 3 == b; P(it) is written back over the first
  // 32 columns of S(it) and read from TMEM by the PV MMA.  S(it + 2) is issued right after
  // PV(it), so S(it + 1) is ready when the softmax of block it ends.  One p_full per buffer:
  // with a single barrier the softmax could complete block it+1's phase before the MMA thread
  // observed block it's, and two completions restore the parity it waits on (a hang seen in
  // the chain version).
  uint64_t* s_full = kv_empty + KV_STAGES;  // [3] S(it) in TMEM, phase (it / 3) & 1
  uint64_t* p_full = s_full + 3;            // [3] P(it) in TMEM (128 arrivals)
  uint64_t* pv_done = p_full + 3;           // [3] PV(it) completed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 3);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) tlm(p, 0);  // entry
  const int h = blockIdx.y, split = blockIdx.z;
  int64_t n_ = p.n, P_ = p.P, qrow0 = 0;
  int breq = 0, q_tile = gridDim.x - 1 - blockIdx.x;  // heaviest tiles first
  if (p.req) {
    breq = blockIdx.x;
    const int4 rq = p.req[breq];
    qrow0 = rq.x;
    n_ = rq.y;
    P_ = rq.z;
    q_tile = 0;
  }
  const int64_t total_ = P_ + n_;
  const int64_t q0 = static_cast<int64_t>(q_tile) * BQ;
  const int64_t key_end = min(total_, P_ + q0 + BQ);  // causal key range of this tile
  // zero-copy segment table of this request (read by every role; small, from L2)
  int* seg_first = reinterpret_cast<int*>(tmem_slot + 16);  // [kSeg + 1] first key block per segment
  int nseg = 0, tail_vis = 0;
  if (p.segs) {
    const int2 sn = p.segn[breq];
    nseg = sn.x;
    tail_vis = sn.y;
    if (threadIdx.x == 0) {
      int f = 0;
      for (int g = 0; g < nseg; ++g) {
        seg_first[g] = f;
        f += (p.segs[breq * kSeg + g].z + BKV - 1) / BKV;
      }
      seg_first[nseg] = f;
    }
    __syncthreads();
  }
  const int64_t nblk = p.segs ? seg_first[nseg] : (key_end + BKV - 1) / BKV;
  const int64_t b0 = nblk * split / p.splits, b1 = nblk * (split + 1) / p.splits;
  const int nb = static_cast<int>(b1 - b0);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < KV_STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int b = 0; b < 3; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 128);
      mbar_init(&pv_done[b], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, S::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem + 3 * BKV;  // S buffers at columns [0, 64), [64, 128), [128, 192)
  // No early trigger: a GEMM / chain launched programmatically after this kernel was
  // seen to deadlock with it (the dependent's CTAs resident and waiting in
  // griddepcontrol.wait while the attention grid never completed -- tools/pdl_bisect2.sh,
  // test_cached_serve_equals_oracle_7b_shape), so dependents start at completion.
  pdl_wait();  // Q/K/V come from the QKV GEMM (and the assembly) just before
  if (threadIdx.x == 0) tlm(p, 1);  // prologue done

  if (warp == 0) {
    if (elect_one() && nb > 0) {
      // maps written by the host between launches: acquire them for the async proxy
      for (int g = 0; g < nseg; ++g)
        asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(p.maps + p.segs[breq * kSeg + g].x)
                     : "memory");
      mbar_expect_tx(q_full, S::kQ);
      for (int a = 0; a < S::kAtoms; ++a)  // 64-row boxes: rows [q0, q0 + 128), or [q0, q0 + 64) twice (dup)
        for (int hh = 0; hh < 2; ++hh)
          tma_load_2d(sQ + a * (BQ * 128) + hh * (64 * 128), &tmQ, q_full, h * HD + a * 64,
                      static_cast<int>(qrow0 + q0 + (p.dup ? 0 : 64 * hh)));
      for (int it = 0, sg = 0; it < nb; ++it) {
        const int s = it % KV_STAGES;
        mbar_wait(&kv_empty[s], ((it / KV_STAGES) & 1) ^ 1);
        probe(p, 4, it);
        uint8_t* st = sKV + s * S::kStage;
        const int j0 = static_cast<int>((b0 + it) * BKV);
        mbar_expect_tx(&kv_full[s], S::kStage + S::kPos);
        if constexpr (AL)  // the block's 64 key positions ride on the same barrier
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(sPos + s * BKV)),
              "l"(p.kv_pos + j0), "r"(S::kPos), "r"(smem_u32(&kv_full[s]))
              : "memory");
        // head-interleaved cache [rows][H*hd]: x = h*hd + a*64, y = key row;
        // head-major cache [H][rows][hd]:     x = a*64,        y = h*rows + key row
        const int kx = h * HD, ky = j0;
        if (p.segs) {
          const int b = static_cast<int>(b0) + it;
          while (b >= seg_first[sg + 1]) ++sg;
          const int4 g = p.segs[breq * kSeg + sg];  // {map, row0, rows, zbase}
          const CUtensorMap* mp = p.maps + g.x;
          const int row = g.y + (b - seg_first[sg]) * BKV, z = g.w + 2 * p.layer;
          for (int a = 0; a < S::kAtoms; ++a) {
            tma_load_3d(st + a * (BKV * 128), mp, &kv_full[s], kx + a * 64, row, z);
            tma_load_3d(st + S::kKV + a * (BKV * 128), mp, &kv_full[s], kx + a * 64, row, z + 1);
          }
          continue;
        }
        for (int a = 0; a < S::kAtoms; ++a) {
          if (p.req) {
            tma_load_3d(st + a * (BKV * 128), &tmK, &kv_full[s], kx + a * 64, ky, breq);
            tma_load_3d(st + S::kKV + a * (BKV * 128), &tmV, &kv_full[s], kx + a * 64, ky, breq);
          } else {
            tma_load_2d(st + a * (BKV * 128), &tmK, &kv_full[s], kx + a * 64, ky);
            tma_load_2d(st + S::kKV + a * (BKV * 128), &tmV, &kv_full[s], kx + a * 64, ky);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one() && nb > 0) {
      constexpr uint32_t idS = idesc_bf16(BQ, BKV);
      constexpr uint32_t idO = idesc_bf16(BQ, HD, false, true);  // V is MN-major
      const uint32_t q_addr = smem_u32(sQ);
      mbar_wait(q_full, 0);
      auto issue_qk = [&](int it) {
        const int s = it % KV_STAGES;
        mbar_wait(&kv_full[s], (it / KV_STAGES) & 1);
        if (it == 0) tlm(p, 2);  // first K/V block landed
        probe(p, 5, it);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sKV + s * S::kStage);
        const uint32_t tS = tmem + (it % 3) * BKV;
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const int a = k >> 2, kk = k & 3;
          umma_bf16(tS, sw128_kmajor_desc(q_addr + a * (BQ * 128) + kk * 32),
                    sw128_kmajor_desc(k_addr + a * (BKV * 128) + kk * 32), idS, k > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[it % 3]);
      };
      issue_qk(0);
      if (nb > 1) issue_qk(1);
      for (int it = 0; it < nb; ++it) {
        mbar_wait(&p_full[it % 3], (it / 3) & 1);  // P(it) in TMEM (and any O correction done)
        probe(p, 2, it);
        tc_fence_after();
        const uint32_t v_addr = smem_u32(sKV + (it % KV_STAGES) * S::kStage + S::kKV);
        const uint32_t pt = tmem + (it % 3) * BKV;  // P(it): A operand from TMEM
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k)
          umma_bf16_ts(tO, pt + k * 8, sw128_mnmajor_desc(v_addr + k * 2048, BKV * 128, 1024), idO,
                       (it > 0 || k > 0) ? 1u : 0u);
        umma_commit(&pv_done[it % 3]);
        umma_commit(&kv_empty[it % KV_STAGES]);
        probe(p, 3, it);
        // S(it + 2) into the buffer of P(it - 1), whose PV was issued an iteration ago
        if (it + 2 < nb) issue_qk(it + 2);
      }
      tlm(p, 3);  // last PV issued
    }
  } else {
    // ---- softmax warps: query row = TMEM lane ----
    const int qd = warp & 3;
    const int r = qd * 32 + lane;
    const bool dup = p.dup != 0;
    const int64_t qi = dup ? (r & 63) : q0 + r;  // query index within the n new rows
    const int64_t limit = P_ + qi;              // last visible key (sequence order)
    const int c0 = dup ? (r >> 6) * 32 : 0;     // dup: this lane's half of every key block
    const uint32_t lane_off = static_cast<uint32_t>(qd * 32) << 16;
    float m = -INFINITY, l = 0.f;
    // a warp whose 32 query rows are all past n (the suffix fills half a 128-row tile)
    // only keeps the barrier protocol: its P rows feed O rows nobody reads
    const bool live = (dup ? (qd & 1) * 32 : q0 + qd * 32) < n_;
    // ALiBi in raw score units: (s + slope sqrt(hd) (pk - pq)) * log2(e)/sqrt(hd)
    //   = (s / sqrt(hd) + slope (pk - pq)) log2(e)
    int32_t qpos = 0;
    float slope_raw = 0.f;
    if constexpr (AL) {
      qpos = qi < n_ ? p.kv_pos[P_ + qi] : 0;
      slope_raw = p.alibi[h] * sqrtf(static_cast<float>(HD));
    }
    // one key block: NC score columns of this lane ([c0, c0 + NC) of the block; NC = 32 in dup mode)
    auto blocks = [&](auto ncols) {
      constexpr int NC = decltype(ncols)::value;
      for (int it = 0, sg = 0; it < nb; ++it) {
        int64_t j0 = (b0 + it) * BKV, lim_seg = 0;
        if (p.segs) {  // zero-copy: mask per segment (module padding rows; causal tail)
          const int b = static_cast<int>(b0) + it;
          while (b >= seg_first[sg + 1]) ++sg;
          const int64_t local = static_cast<int64_t>(b - seg_first[sg]) * BKV;
          lim_seg = sg == nseg - 1 ? tail_vis + qi - local : p.segs[breq * kSeg + sg].z - 1 - local;
          j0 = limit - lim_seg;  // so that key c is masked iff c > lim_seg, as below
        }
        j0 += c0;  // first key of this lane's columns
        if (!live) {
          // S(it) was issued after p_full(it - 2) completed: arriving after it keeps this warp
          // out of block it - 3's phase of the same barrier
          mbar_wait(&s_full[it % 3], (it / 3) & 1);
          mbar_arrive(&p_full[it % 3]);
          continue;
        }
        mbar_wait(&s_full[it % 3], (it / 3) & 1);
        if (threadIdx.x == 128) probe(p, 0, it);
        tc_fence_after();
        float sv[NC];
        {
          uint32_t raw[NC];
#pragma unroll
          for (int c = 0; c < NC; c += 16) tmem_ld16_nowait(tmem + (it % 3) * BKV + lane_off + c0 + c, raw + c);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < NC; ++c) sv[c] = __uint_as_float(raw[c]);
        }
        if (threadIdx.x == 128) probe(p, 6, it);
        if constexpr (AL) {
          const int s = it % KV_STAGES;
          mbar_wait(&kv_full[s], (it / KV_STAGES) & 1);  // the positions' bulk copy (already complete)
          const int4* kp = reinterpret_cast<const int4*>(sPos + s * BKV + c0);
#pragma unroll
          for (int c = 0; c < NC; c += 4) {
            const int4 k4 = kp[c >> 2];
            sv[c] = fmaf(slope_raw, static_cast<float>(k4.x - qpos), sv[c]);
            sv[c + 1] = fmaf(slope_raw, static_cast<float>(k4.y - qpos), sv[c + 1]);
            sv[c + 2] = fmaf(slope_raw, static_cast<float>(k4.z - qpos), sv[c + 2]);
            sv[c + 3] = fmaf(slope_raw, static_cast<float>(k4.w - qpos), sv[c + 3]);
          }
        }
        // scores stay raw (unscaled); the 1/sqrt(hd) * log2(e) factor is folded into
        // one FFMA per element in front of ex2.approx
        if (j0 + NC - 1 > limit) {  // diagonal block (or a segment's padding) only
#pragma unroll
          for (int c = 0; c < NC; ++c)
            if (j0 + c > limit) sv[c] = -INFINITY;
        }
        // 8 independent max chains + a 3-level tree (a single chain is 63 dependent FMNMX)
        float mx[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) mx[c] = sv[c];
#pragma unroll
        for (int c = 8; c < NC; ++c) mx[c & 7] = fmaxf(mx[c & 7], sv[c]);
#pragma unroll
        for (int w = 4; w; w >>= 1)
#pragma unroll
          for (int c = 0; c < w; ++c) mx[c] = fmaxf(mx[c], mx[c + w]);
        const float bm = mx[0];
        // lazy max update: move the reference max only when it grows by > 2^8
        const bool grow = bm > m + kRescaleThreshold / p.scale_log2 || (m == -INFINITY && bm > -INFINITY);
        if (__any_sync(0xffffffffu, grow) && it > 0) {
          // O holds blocks < it: wait for PV(it-1), then scale the rows that grow
          mbar_wait(&pv_done[(it - 1) % 3], ((it - 1) / 3) & 1);
          tc_fence_after();
          const float f = grow ? fast_exp2((m - bm) * p.scale_log2) : 1.f;  // m = -inf -> 0
#pragma unroll 1
          for (int c = 0; c < HD; c += 16) {
            float ov[16];
            tmem_ld16(tO + lane_off + c, ov);
#pragma unroll
            for (int x = 0; x < 16; ++x) ov[x] *= f;
            tmem_st16(tO + lane_off + c, ov);
          }
          tmem_st_wait();
        }
        if (grow) {
          l *= fast_exp2((m - bm) * p.scale_log2);
          m = bm;
        }
        const float mb = (m == -INFINITY) ? 0.f : m * p.scale_log2;  // all scores -inf when m is
        float bs[4] = {0.f, 0.f, 0.f, 0.f};  // independent partial sums
        uint32_t packed[NC / 2];
#pragma unroll
        for (int c = 0; c < NC; c += 2) {
          const float p0 = fast_exp2(fmaf(sv[c], p.scale_log2, -mb));
          const float p1 = fast_exp2(fmaf(sv[c + 1], p.scale_log2, -mb));
          bs[(c >> 1) & 3] += p0 + p1;
          __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
          packed[c >> 1] = *reinterpret_cast<uint32_t*>(&b2);
        }
        l += (bs[0] + bs[1]) + (bs[2] + bs[3]);
        if (threadIdx.x == 128) probe(p, 7, it);
        // P row (64 keys) into TMEM over the first 32 columns of its score buffer; dup: this
        // lane's half of the keys, zeros in the other half
        {
          const uint32_t pa = tmem + (it % 3) * BKV + lane_off;
          if constexpr (NC == 64) {
            tmem_st16u(pa, packed);
            tmem_st16u(pa + 16, packed + 16);
          } else {
            const uint32_t z[16] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
            tmem_st16u(pa + 16 * (r >> 6), packed);
            tmem_st16u(pa + 16 * (1 - (r >> 6)), z);
          }
          tmem_st_wait();
        }
        if (threadIdx.x == 128) probe(p, 8, it);
        tc_fence_before();
        mbar_arrive(&p_full[it % 3]);  // after block it-3's phase: S(it) needed p_full(it-2)
        if (threadIdx.x == 128) probe(p, 1, it);
      }
    };
    if (dup) blocks(std::integral_constant<int, 32>{});
    else blocks(std::integral_constant<int, BKV>{});
    if (nb > 0) {
      mbar_wait(&pv_done[(nb - 1) % 3], ((nb - 1) / 3) & 1);
      tc_fence_after();
      if (p.splits == 1) {
        // dup: lane r + 64 holds query r's other half-keys partial; it parks (O, m, l) in the
        // idle K/V stages and lane r merges (tcgen05.ld is warp-collective: lane conditions
        // guard only the memory operations)
        float w0 = 1.f, w1 = 0.f;
        float* xo = reinterpret_cast<float*>(sKV);
        float2* xml = reinterpret_cast<float2*>(sKV + 64 * (HD + 4) * 4);
        if (dup) {
          if (r >= 64) {
#pragma unroll 1
            for (int c = 0; c < HD; c += 16) {
              float ov[16];
              tmem_ld16(tO + lane_off + c, ov);
#pragma unroll
              for (int x = 0; x < 16; x += 4)
                *reinterpret_cast<float4*>(xo + qi * (HD + 4) + c + x) = make_float4(ov[x], ov[x + 1], ov[x + 2], ov[x + 3]);
            }
            xml[qi] = make_float2(m, l);
          }
          named_bar(1, 128);
          if (r < 64) {
            const float2 o = xml[qi];
            const float M = l > 0.f && o.y > 0.f ? fmaxf(m, o.x) : (l > 0.f ? m : o.x);
            w0 = l > 0.f ? fast_exp2((m - M) * p.scale_log2) : 0.f;
            w1 = o.y > 0.f ? fast_exp2((o.x - M) * p.scale_log2) : 0.f;
            l = w0 * l + w1 * o.y;
          }
        }
        const float inv = 1.f / l;
        __nv_bfloat16* dst = p.out + (qrow0 + qi) * p.d + h * HD;
        if (!dup || r < 64) {
#pragma unroll 1
          for (int c = 0; c < HD; c += 16) {
            float ov[16];
            tmem_ld16(tO + lane_off + c, ov);
            if (qi < n_) {
              if (dup) {
#pragma unroll
                for (int y = 0; y < 16; ++y) ov[y] = w0 * ov[y] + w1 * xo[qi * (HD + 4) + c + y];
              }
              uint4 w[2];
              __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(w);
#pragma unroll
              for (int y = 0; y < 8; ++y) b[y] = __floats2bfloat162_rn(ov[2 * y] * inv, ov[2 * y + 1] * inv);
              *reinterpret_cast<uint4*>(dst + c) = w[0];
              *reinterpret_cast<uint4*>(dst + c + 8) = w[1];
            }
          }
        }
      } else {
        // park the unnormalised O row and (m, l) in this CTA's idle K/V stage smem
        // for the cluster-wide merge below
        float* red = reinterpret_cast<float*>(sKV);
#pragma unroll 1
        for (int c = 0; c < HD; c += 16) {
          float ov[16];
          tmem_ld16(tO + lane_off + c, ov);
#pragma unroll
          for (int x = 0; x < 16; x += 4)
            *reinterpret_cast<float4*>(red + r * kRedRow + c + x) = make_float4(ov[x], ov[x + 1], ov[x + 2], ov[x + 3]);
        }
        red[BQ * kRedRow + 2 * r] = nb > 0 ? m : -INFINITY;
        red[BQ * kRedRow + 2 * r + 1] = nb > 0 ? l : 0.f;
      }
    }
  }
  if (threadIdx.x == 64) tlm(p, 4);  // softmax / output done
  if (p.splits > 1) {
    // The split CTAs of one head form a thread-block cluster.  After every partial
    // is parked, CTA rank s merges query rows {s, s+S, s+2S, ...} of all S partials
    // through DSMEM in rank order (deterministic):
    //   O = sum_s w_s O_s / sum_s w_s l_s,  w_s = 2^((m_s - M) * scale),  M = max_s m_s
    cluster_sync_all();
    if (warp >= 2) {
      const int t = threadIdx.x - 64;             // 0..127
      constexpr int kTpr = 8;                     // threads per row
      constexpr int kXs = HD / kTpr;              // hd values per thread
      const uint32_t red0 = smem_u32(sKV);
      for (int64_t row = split + static_cast<int64_t>(t / kTpr) * p.splits; row < n_;
           row += static_cast<int64_t>(128 / kTpr) * p.splits) {
        // every DSMEM load of a phase is issued before any is consumed (the merge was a
        // chain of ~10 dependent cluster round trips: 6.7 us of a 26 us launch)
        float ms[8], ls[8];
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2) {
          ms[s2] = -INFINITY;
          ls[s2] = 0.f;
          if (s2 < p.splits) {
            const uint32_t ml = mapa_shared(red0 + (BQ * kRedRow + 2 * static_cast<uint32_t>(row)) * 4, s2);
            ms[s2] = ld_dsmem_f32(ml);
            ls[s2] = ld_dsmem_f32(ml + 4);
          }
        }
        float M = -INFINITY;
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2)
          if (s2 < p.splits && ls[s2] > 0.f) M = fmaxf(M, ms[s2]);
        float den = 0.f, acc[kXs];
#pragma unroll
        for (int x = 0; x < kXs; ++x) acc[x] = 0.f;
        const int x0 = (t % kTpr) * kXs;
#pragma unroll
        for (int g = 0; g < 8; g += 4) {  // splits in groups of 4: 16 outstanding 16-byte loads
          if (g >= p.splits) break;
          float f[4][kXs];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (g + u < p.splits) {
              const uint32_t src = mapa_shared(red0 + (static_cast<uint32_t>(row) * kRedRow + x0) * 4, g + u);
#pragma unroll
              for (int x = 0; x < kXs; x += 4) ld_dsmem_v4(src + x * 4, f[u] + x);
            }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int s2 = g + u;
            if (s2 >= p.splits || !(ls[s2] > 0.f)) continue;
            const float w = fast_exp2((ms[s2] - M) * p.scale_log2);
            den += w * ls[s2];
#pragma unroll
            for (int x = 0; x < kXs; ++x) acc[x] += w * f[u][x];
          }
        }
        const float inv = 1.f / den;
        __nv_bfloat16* dst = p.out + (qrow0 + row) * p.d + h * HD + x0;
#pragma unroll
        for (int x = 0; x < kXs; x += 8) {
          uint4 v;
          __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
          for (int y = 0; y < 4; ++y) b[y] = __floats2bfloat162_rn(acc[x + 2 * y] * inv, acc[x + 2 * y + 1] * inv);
          *reinterpret_cast<uint4*>(dst + x) = v;
        }
      }
    }
    cluster_sync_all();  // peers are done reading this CTA's smem
  }
  if (threadIdx.x == 0) tlm(p, 5);  // merge done
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, S::kTmemCols);
}

}  // namespace

// 3-D bf16 map {cols, rows, planes} (plane stride in bytes), box {64, box_rows, 1}, SW128
// (also the chain attention phase's in-place KV sources)
CUtensorMap tmap_bf16_3d(const void* ptr, uint64_t cols, uint64_t rows, uint64_t planes, uint64_t plane_stride,
                         uint32_t box_rows) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn fn = [] {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult qr;
    PCB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &qr));
    return reinterpret_cast<EncodeFn>(q);
  }();
  CUtensorMap m;
  cuuint64_t dims[3] = {cols, rows, planes};
  cuuint64_t strides[2] = {cols * 2, plane_stride};
  cuuint32_t box[3] = {64, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (3-D) failed: " + std::to_string((int)r));
  return m;
}

namespace {

unsigned long long* g_tlbuf = nullptr;
int g_tl_ctas = 0;

template <int HD, bool AL>
void launch_attn(const AttnArgs& a, float* scratch, size_t scratch_bytes, cudaStream_t s) {
  using Sm = AttnSmem<HD, AL>;
  static bool attr = [] {
    PCB_CUDA(cudaFuncSetAttribute(k_attn_tc<HD, AL>, cudaFuncAttributeMaxDynamicSharedMemorySize, Sm::kBytes));
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
  p.alibi = a.alibi;
  p.kv_pos = a.kv_pos;
  const bool batched = a.n_req > 0;  // one launch over the requests of a micro-batch
  const int q_tiles = batched ? a.n_req : static_cast<int>((a.n + BQ - 1) / BQ);
  const int64_t nblk0 = a.segs ? a.max_blocks
                      : batched ? (a.max_P + a.max_n + BKV - 1) / BKV
                                : (std::min<int64_t>(p.total, a.P + BQ) + BKV - 1) / BKV;  // tile 0 key blocks
  // one CTA per SM; for single-tile (suffix) launches pick the split count that
  // minimises waves x blocks per CTA (+ a per-split fixed cost)
  const int base = q_tiles * a.H;
  int splits = 1;
  if ((q_tiles == 1 || batched) && base < 2 * sms) {
    int64_t best = -1;
    for (int s2 = 1; s2 <= std::max<int64_t>(1, std::min<int64_t>(nblk0 / 2, 8)); ++s2) {  // cluster <= 8
      const size_t need = static_cast<size_t>(a.H) * s2 * BQ * (HD + 2) * sizeof(float);
      if (s2 > 1 && need > scratch_bytes) break;
      const int64_t waves = (static_cast<int64_t>(base) * s2 + sms - 1) / sms;
      const int64_t cost = waves * ((nblk0 + s2 - 1) / s2 + 6) * 16 + s2;
      if (best < 0 || cost < best) {
        best = cost;
        splits = s2;
      }
    }
  }
  static const int splits_env = [] {  // tuning override (environment read once)
    const char* v = std::getenv("PCB_ATTN_SPLITS");
    return v ? std::max(1, std::atoi(v)) : 0;
  }();
  if (splits_env) splits = splits_env;
  p.splits = splits;
  p.part_o = scratch;
  p.part_ml = scratch + static_cast<size_t>(a.H) * splits * BQ * HD;
  p.counters = a.counters;
  if (splits > 8) splits = 8;
  p.splits = splits;
  CUtensorMap tq = tmap_bf16_2d(a.q, static_cast<uint64_t>(a.n), static_cast<uint64_t>(a.d), 64);  // 64-row boxes
  static const bool nodup = std::getenv("PCB_ATTN_NODUP") != nullptr;  // A/B switch
  p.dup = batched && a.max_n <= 64 && splits == 1 && !nodup ? 1 : 0;
  static const bool tl_on = std::getenv("PCB_ATTN_TL") != nullptr;
  if (tl_on) {  // per-CTA phase timeline of the LAST launch (attn_tl_dump)
    if (!g_tlbuf) PCB_CUDA(cudaMalloc(&g_tlbuf, 8192 * 8 * sizeof(unsigned long long)));
    p.tl = g_tlbuf;
    g_tl_ctas = q_tiles * a.H * std::min(splits, 8);
  }
  static unsigned long long* dbg = nullptr;
  static const bool probe_on = std::getenv("PCB_ATTN_DBG") != nullptr;  // timeline probe of CTA 0 (debug)
  if (probe_on) {
    if (!dbg) PCB_CUDA(cudaMallocManaged(&dbg, 12 * 64 * sizeof(unsigned long long)));
    std::memset(dbg, 0, 12 * 64 * sizeof(unsigned long long));
    p.dbg = dbg;
  }
  CUtensorMap tk, tv;
  if (a.segs) {  // K/V through the per-segment maps in global memory
    p.req = a.req;
    p.segs = a.segs;
    p.segn = a.segn;
    p.maps = static_cast<const CUtensorMap*>(a.maps);
    p.layer = a.layer;
    tk = tq;
    tv = tq;
  } else if (batched) {
    // request r's cache rows: {d, rows, request} with the request stride between planes
    p.req = a.req;
    tk = tmap_bf16_3d(a.k, a.d, a.kv_cap, a.n_req, a.req_stride, BKV);
    tv = tmap_bf16_3d(a.v, a.d, a.kv_cap, a.n_req, a.req_stride, BKV);
  } else {
    tk = tmap_bf16_2d(a.k, static_cast<uint64_t>(p.total), static_cast<uint64_t>(a.d), BKV);
    tv = tmap_bf16_2d(a.v, static_cast<uint64_t>(p.total), static_cast<uint64_t>(a.d), BKV);
  }
  dim3 grid(q_tiles, a.H, splits);
  PdlClass pc(PDL_ATTN);
  launch_k(k_attn_tc<HD, AL>, grid, dim3(kAttnThreads), Sm::kBytes, s, splits, tq, tk, tv, p);  // cluster = splits
  if (probe_on) {
    PCB_CUDA(cudaDeviceSynchronize());
    const unsigned long long t0 = dbg[4 * 64];
    std::fprintf(stderr, "attn probe (ns from first load): it | kv_empty->load  kv_full(MMA)  s_full(softmax)  p_arrive  p_full(MMA)  pv_issued\n");
    for (int it = 0; it < 16; ++it)
      std::fprintf(stderr, "%2d | %8lld %8lld %8lld %8lld %8lld %8lld\n", it, (long long)(dbg[4 * 64 + it] - t0),
                   (long long)(dbg[5 * 64 + it] - t0), (long long)(dbg[0 * 64 + it] - t0),
                   (long long)(dbg[1 * 64 + it] - t0), (long long)(dbg[2 * 64 + it] - t0),
                   (long long)(dbg[3 * 64 + it] - t0));
    std::fprintf(stderr, "softmax detail: it | s_full  ld_done  exp_done  pvdone_wait  arrive\n");
    for (int it = 0; it < 16; ++it)
      std::fprintf(stderr, "%2d | %8lld %8lld %8lld %8lld %8lld\n", it, (long long)(dbg[0 * 64 + it] - t0),
                   (long long)(dbg[6 * 64 + it] - t0), (long long)(dbg[7 * 64 + it] - t0),
                   (long long)(dbg[8 * 64 + it] - t0), (long long)(dbg[1 * 64 + it] - t0));
  }
}

}  // namespace

int attn_tl_dump(unsigned long long* out, int max_ctas) {
  if (!g_tlbuf) return 0;
  PCB_CUDA(cudaDeviceSynchronize());
  const int n = std::min(g_tl_ctas, max_ctas);
  PCB_CUDA(cudaMemcpy(out, g_tlbuf, static_cast<size_t>(n) * 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  return n;
}

bool attention_tc_supported(const AttnArgs& a) {
  // ALiBi: single request, contiguous key positions (kv_pos padded to whole 64-key blocks)
  const bool alibi_ok = !a.alibi || (a.kv_pos && !a.segs && !a.req && a.n_req == 0);
  return (a.hd == 128 || a.hd == 64) && !a.mask && !a.block_id && alibi_ok && a.n >= 1 && a.d % 64 == 0 &&
         (a.P + a.n) < (1LL << 31);
}

void attention_tc(const AttnArgs& a, float* scratch, size_t scratch_bytes, cudaStream_t s) {
  static const int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  static const bool pair_off = [] {  // A/B switch: the single-tile kernel for long prefills too
    const char* v = std::getenv("PCB_ATTN_PAIR");
    return v && v[0] == '0';
  }();
  if (!pair_off && attention_prefill_supported(a, sms)) {
    attention_prefill(a, s);
    return;
  }
  static const bool batch_off = [] {  // A/B switch: PCB_ATTN_BATCH=0 keeps one CTA per (request, head)
    const char* v = std::getenv("PCB_ATTN_BATCH");
    return v && v[0] == '0';
  }();
  if (!batch_off && attention_batch_supported(a)) {
    attention_batch(a, s);
    return;
  }
  if (a.alibi) {
    if (a.hd == 128) launch_attn<128, true>(a, scratch, scratch_bytes, s);
    else launch_attn<64, true>(a, scratch, scratch_bytes, s);
  } else {
    if (a.hd == 128) launch_attn<128, false>(a, scratch, scratch_bytes, s);
    else launch_attn<64, false>(a, scratch, scratch_bytes, s);
  }
}

}  // namespace pcb::kern

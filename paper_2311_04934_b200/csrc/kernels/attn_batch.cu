// Persistent suffix attention for a micro-batch of requests (configs[3]: serve_batch): every
// request's <= 64 new rows against its own keys -- the cached modules read in place through
// per-request segment tables (zero-copy), or its assembled cache through a 3-D map over the
// request caches -- causal in sequence order (reference model.cpp:401-427).
//
// One CTA per SM walks the (request, head) items, head-major (all requests of head h before
// head h + 1: modules shared by several requests of the micro-batch are read while their
// head-h K/V is in L2); per item the pipeline is the attn_tc.cu one
// in its duplicated-query form (the Q tile holds the request's rows twice, TMEM lanes [0, 64)
// take keys [0, 32) of every 64-key block and lanes [64, 128) keys [32, 64); three score
// buffers with P written back to TMEM for a TS-form PV).  What the persistent form removes
// (tools/attn_phases_c4.py on the one-CTA-per-item kernel: 2.0 us of prologue and 1.8 us of
// first-K/V latency per 22 us item, 21 % of the SM-time idle between CTAs): the K/V ring and
// every barrier sequence run on across items, TMEM is allocated once, and the next item's Q
// and first K/V blocks load while the current item's softmax tail and output run.  The two
// query halves combine through a 4 KB chunk buffer, so the K/V stages are never scratch.
//
//   warp 0     TMA: per item Q (q_empty -> q_full), then K/V blocks through a 5-stage ring
//   warp 1     TMEM (512 columns) + MMA: S = Q K^T into score buffer g % 3, PV from TMEM
//   warps 2-5  softmax (one thread per TMEM lane), then the item's output
#include <cuda.h>

#include "common.cuh"
#include "tc_common.cuh"

namespace pcb::kern {

using namespace tc;
CUtensorMap tmap_bf16_2d(const void* ptr, uint64_t rows, uint64_t cols, uint32_t box_rows);
CUtensorMap tmap_bf16_3d(const void* ptr, uint64_t cols, uint64_t rows, uint64_t planes, uint64_t plane_stride,
                         uint32_t box_rows);

namespace {

constexpr int HD = 128, BKV = 64, kThreads = 192, kSeg = 16;
constexpr int kQ = 128 * HD * 2;       // Q tile (rows twice), two 64-column atoms
constexpr int kKV = BKV * HD * 2;      // K or V block
constexpr int kStage = 2 * kKV;        // K + V
constexpr int kStages = 5;
constexpr int kChunk = 64 * 17 * 4;    // merge chunk: [64 rows][16 floats + pad]
constexpr int kSmem = kQ + kStages * kStage + kChunk + 64 * 8 + 1024 + 1024;
static_assert(kSmem <= 232448, "batched attention shared memory");
constexpr float kThr = 8.0f;  // log2 domain: stale running max tolerated up to 2^8

struct BatchParams {
  int n_items, n_req, H, d, layer;
  float scale_log2;
  __nv_bfloat16* out;
  const int4* req;   // [n_req] {first q row, n, P, 0}
  const int4* segs;  // zero-copy: [n_req][16] {map, row0, rows, zbase}
  const int2* segn;  // [n_req] {segments, tail visible rows}
  const CUtensorMap* maps;
};

__device__ __forceinline__ void tmem_st16u(uint32_t addr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st16f(uint32_t addr, const float* v) {
  uint32_t u[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) u[i] = __float_as_uint(v[i]);
  tmem_st16u(addr, u);
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float ex2(float x) {  // MUFU.EX2; ex2(-inf) = +0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// key blocks of request b: per segment ceil(rows / 64) (zero-copy), else ceil((P + n) / 64)
struct Keys {
  int nseg, tail_vis, nb;
  int first[kSeg + 1];
};
__device__ __forceinline__ void keys_of(const BatchParams& p, int b, int4 rq, Keys& k) {
  if (p.segs) {
    const int2 sn = p.segn[b];
    k.nseg = sn.x;
    k.tail_vis = sn.y;
    int f = 0;
    for (int g = 0; g < k.nseg; ++g) {
      k.first[g] = f;
      f += (p.segs[b * kSeg + g].z + BKV - 1) / BKV;
    }
    k.first[k.nseg] = f;
    k.nb = f;
  } else {
    k.nseg = 0;
    k.tail_vis = 0;
    k.nb = (rq.z + rq.y + BKV - 1) / BKV;
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    k_attn_batch(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmV, BatchParams p) {
  extern __shared__ uint8_t smem_raw[];
  // pointer arithmetic on the __shared__ symbol (not an integer round trip) keeps the
  // shared address space visible to the compiler: LDS/STS instead of generic LD/ST
  uint8_t* smem = smem_raw + ((1024u - (static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw)) & 1023u)) & 1023u);
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + kQ;
  float* sX = reinterpret_cast<float*>(sKV + kStages * kStage);  // merge chunk [64][17]
  float2* sML = reinterpret_cast<float2*>(sX + 64 * 17);           // [64] partner (m, l)
  uint64_t* q_full = reinterpret_cast<uint64_t*>(sML + 64);
  uint64_t* q_empty = q_full + 1;
  uint64_t* kv_full = q_empty + 1;        // [kStages]
  uint64_t* kv_empty = kv_full + kStages;  // [kStages]
  uint64_t* s_full = kv_empty + kStages;  // [3] block g -> buffer g % 3, phase (g / 3) & 1
  uint64_t* p_full = s_full + 3;          // [3] (128 arrivals; one per buffer, see attn_tc.cu)
  uint64_t* pv_done = p_full + 3;         // [3]
  uint64_t* o_full = pv_done + 3;         // last PV of an item complete
  uint64_t* o_empty = o_full + 1;         // O read out by the softmax warps (128 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int C = gridDim.x;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    if (!p.segs) {
      tma_prefetch(&tmK);
      tma_prefetch(&tmV);
    }
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int b = 0; b < 3; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 128);
      mbar_init(&pv_done[b], 1);
    }
    mbar_init(o_full, 1);
    mbar_init(o_empty, 128);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tO = tmem + 3 * BKV;  // score buffers at [0, 192)
  pdl_wait();

  if (warp == 0) {
    if (elect_one()) {
      int g = 0, k = 0;
      Keys K;
      for (int it = blockIdx.x; it < p.n_items; it += C, ++k) {
        const int h = it / p.n_req, b = it - h * p.n_req;
        const int4 rq = p.req[b];
        keys_of(p, b, rq, K);
        if (p.segs)  // maps written by the host between launches: acquire them for the async proxy
          for (int s = 0; s < K.nseg; ++s)
            asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(p.maps + p.segs[b * kSeg + s].x)
                         : "memory");
        mbar_wait(q_empty, (k & 1) ^ 1);  // every S MMA of the previous item is done with Q
        mbar_expect_tx(q_full, kQ);
        for (int a = 0; a < 2; ++a)
          for (int hh = 0; hh < 2; ++hh)  // the request's rows twice (64-row boxes)
            tma_load_2d(sQ + a * (128 * 128) + hh * (64 * 128), &tmQ, q_full, h * HD + a * 64, rq.x);
        for (int j = 0, sg = 0; j < K.nb; ++j, ++g) {
          const int s = g % kStages;
          mbar_wait(&kv_empty[s], ((g / kStages) & 1) ^ 1);
          uint8_t* st = sKV + s * kStage;
          mbar_expect_tx(&kv_full[s], kStage);
          if (p.segs) {
            while (j >= K.first[sg + 1]) ++sg;
            const int4 gs = p.segs[b * kSeg + sg];  // {map, row0, rows, zbase}
            const CUtensorMap* mp = p.maps + gs.x;
            const int row = gs.y + (j - K.first[sg]) * BKV, z = gs.w + 2 * p.layer;
            for (int a = 0; a < 2; ++a) {
              tma_load_3d(st + a * (BKV * 128), mp, &kv_full[s], h * HD + a * 64, row, z);
              tma_load_3d(st + kKV + a * (BKV * 128), mp, &kv_full[s], h * HD + a * 64, row, z + 1);
            }
          } else {
            for (int a = 0; a < 2; ++a) {
              tma_load_3d(st + a * (BKV * 128), &tmK, &kv_full[s], h * HD + a * 64, j * BKV, b);
              tma_load_3d(st + kKV + a * (BKV * 128), &tmV, &kv_full[s], h * HD + a * 64, j * BKV, b);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idS = idesc_bf16(128, BKV);
      constexpr uint32_t idO = idesc_bf16(128, HD, false, true);  // V: MN-major
      const uint32_t q_addr = smem_u32(sQ);
      int g0 = 0, k = 0;
      Keys K;
      for (int it = blockIdx.x; it < p.n_items; it += C, ++k) {
        const int b = it % p.n_req;
        keys_of(p, b, p.req[b], K);
        const int nb = K.nb;
        mbar_wait(q_full, k & 1);
        auto issue_qk = [&](int j) {
          const int g = g0 + j, s = g % kStages;
          mbar_wait(&kv_full[s], (g / kStages) & 1);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(sKV + s * kStage);
#pragma unroll
          for (int x = 0; x < HD / 16; ++x)
            umma_bf16(tmem + (g % 3) * BKV, sw128_kmajor_desc(q_addr + (x >> 2) * (128 * 128) + (x & 3) * 32),
                      sw128_kmajor_desc(k_addr + (x >> 2) * (BKV * 128) + (x & 3) * 32), idS, x > 0 ? 1u : 0u);
          umma_commit(&s_full[g % 3]);
        };
        issue_qk(0);
        if (nb > 1) issue_qk(1);
        for (int j = 0; j < nb; ++j) {
          const int g = g0 + j;
          if (j == 0) mbar_wait(o_empty, (k & 1) ^ 1);  // the previous item's O is read out
          mbar_wait(&p_full[g % 3], (g / 3) & 1);
          tc_fence_after();
          const uint32_t v_addr = smem_u32(sKV + (g % kStages) * kStage + kKV);
#pragma unroll
          for (int x = 0; x < BKV / 16; ++x)
            umma_bf16_ts(tO, tmem + (g % 3) * BKV + x * 8, sw128_mnmajor_desc(v_addr + x * 2048, BKV * 128, 1024), idO,
                         (j > 0 || x > 0) ? 1u : 0u);
          umma_commit(&pv_done[g % 3]);
          umma_commit(&kv_empty[g % kStages]);
          if (j + 2 < nb) issue_qk(j + 2);
          if (j + 1 == nb) umma_commit(q_empty);  // after the item's last S (issued before)
        }
        if (nb == 0) umma_commit(q_empty);
        umma_commit(o_full);
        g0 += nb;
      }
    }
  } else {
    // ---- softmax: TMEM lane r = query r & 63 (dup), half r >> 6 of every key block ----
    const int qd = warp & 3;
    const int r = qd * 32 + lane;
    const int qi = r & 63, hi = r >> 6, c0 = hi * 32;
    const int et = threadIdx.x - 64;
    const uint32_t lane_off = static_cast<uint32_t>(qd * 32) << 16;
    const float sc = p.scale_log2, thr = kThr / sc;
    int g0 = 0, k = 0;
    Keys K;
    for (int it = blockIdx.x; it < p.n_items; it += C, ++k) {
      const int h = it / p.n_req, b = it - h * p.n_req;
      const int4 rq = p.req[b];
      keys_of(p, b, rq, K);
      const int n_ = rq.y, P_ = rq.z, nb = K.nb;
      const bool live = (qd & 1) * 32 < n_;  // else this warp keeps the barrier protocol only
      float m = -INFINITY, l = 0.f;
      for (int j = 0, sg = 0; j < nb; ++j) {
        const int g = g0 + j;
        // key c of this lane's 32 columns visible iff c <= lim
        int lim;
        if (K.nseg) {
          while (j >= K.first[sg + 1]) ++sg;
          const int local = (j - K.first[sg]) * BKV;
          lim = (sg == K.nseg - 1 ? K.tail_vis + qi : p.segs[b * kSeg + sg].z - 1) - local - c0;
        } else {
          lim = P_ + qi - j * BKV - c0;
        }
        mbar_wait(&s_full[g % 3], (g / 3) & 1);
        if (!live) {  // S(g) was issued after p_full(g - 2): the arrival stays out of block g - 3's phase
          mbar_arrive(&p_full[g % 3]);
          continue;
        }
        tc_fence_after();
        float sv[32];
        {
          uint32_t raw[32];
          tmem_ld16_nowait(tmem + (g % 3) * BKV + lane_off + c0, raw);
          tmem_ld16_nowait(tmem + (g % 3) * BKV + lane_off + c0 + 16, raw + 16);
          tmem_wait_ld();
#pragma unroll
          for (int x = 0; x < 32; ++x) sv[x] = __uint_as_float(raw[x]);
        }
        if (lim < 31) {
#pragma unroll
          for (int x = 0; x < 32; ++x)
            if (x > lim) sv[x] = -INFINITY;
        }
        float mx[8];
#pragma unroll
        for (int x = 0; x < 8; ++x) mx[x] = sv[x];
#pragma unroll
        for (int x = 8; x < 32; ++x) mx[x & 7] = fmaxf(mx[x & 7], sv[x]);
#pragma unroll
        for (int w = 4; w; w >>= 1)
#pragma unroll
          for (int x = 0; x < w; ++x) mx[x] = fmaxf(mx[x], mx[x + w]);
        const float bm = mx[0];
        const bool grow = bm > m + thr || (m == -INFINITY && bm > -INFINITY);
        if (__any_sync(0xffffffffu, grow) && j > 0) {
          mbar_wait(&pv_done[(g - 1) % 3], ((g - 1) / 3) & 1);  // O holds blocks < j
          tc_fence_after();
          const float f = grow ? ex2((m - bm) * sc) : 1.f;
#pragma unroll 1
          for (int c = 0; c < HD; c += 16) {
            float ov[16];
            tmem_ld16(tO + lane_off + c, ov);
#pragma unroll
            for (int y = 0; y < 16; ++y) ov[y] *= f;
            tmem_st16f(tO + lane_off + c, ov);
          }
          tmem_st_wait();
        }
        if (grow) {
          l *= ex2((m - bm) * sc);
          m = bm;
        }
        const float mb = m == -INFINITY ? 0.f : m * sc;
        float bs[4] = {0.f, 0.f, 0.f, 0.f};
        uint32_t packed[16];
#pragma unroll
        for (int x = 0; x < 32; x += 2) {
          const float p0 = ex2(fmaf(sv[x], sc, -mb)), p1 = ex2(fmaf(sv[x + 1], sc, -mb));
          bs[(x >> 1) & 3] += p0 + p1;
          __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
          packed[x >> 1] = *reinterpret_cast<uint32_t*>(&b2);
        }
        l += (bs[0] + bs[1]) + (bs[2] + bs[3]);
        {  // P row: this lane's half of the 64 keys, zeros in the other half
          const uint32_t pa = tmem + (g % 3) * BKV + lane_off;
          const uint32_t z[16] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
          tmem_st16u(pa + 16 * hi, packed);
          tmem_st16u(pa + 16 * (1 - hi), z);
          tmem_st_wait();
        }
        tc_fence_before();
        mbar_arrive(&p_full[g % 3]);
      }
      g0 += nb;
      // ---- output: the two halves of a query combine through a 4 KB chunk buffer ----
      mbar_wait(o_full, k & 1);
      tc_fence_after();
      if (hi && qi < n_) sML[qi] = make_float2(m, l);
      named_bar(1, 128);
      float w0 = 1.f, w1 = 0.f, inv = 0.f;
      if (!hi && qi < n_) {
        const float2 o = sML[qi];
        const float M = l > 0.f && o.y > 0.f ? fmaxf(m, o.x) : (l > 0.f ? m : o.x);
        w0 = l > 0.f ? ex2((m - M) * sc) : 0.f;
        w1 = o.y > 0.f ? ex2((o.x - M) * sc) : 0.f;
        const float lt = w0 * l + w1 * o.y;
        inv = lt > 0.f ? 1.f / lt : 0.f;
      }
      __nv_bfloat16* dst = p.out + static_cast<int64_t>(rq.x + qi) * p.d + h * HD;
#pragma unroll 1
      for (int c = 0; c < HD; c += 16) {
        float ov[16];
        tmem_ld16(tO + lane_off + c, ov);  // warp-collective: every lane loads its row
        if (hi && qi < n_)
#pragma unroll
          for (int y = 0; y < 16; ++y) sX[qi * 17 + y] = ov[y];
        named_bar(1, 128);
        if (!hi && qi < n_) {
          uint4 w[2];
          __nv_bfloat162* bb = reinterpret_cast<__nv_bfloat162*>(w);
#pragma unroll
          for (int y = 0; y < 8; ++y) {
            const float a = (w0 * ov[2 * y] + w1 * sX[qi * 17 + 2 * y]) * inv;
            const float e = (w0 * ov[2 * y + 1] + w1 * sX[qi * 17 + 2 * y + 1]) * inv;
            bb[y] = __floats2bfloat162_rn(a, e);
          }
          *reinterpret_cast<uint4*>(dst + c) = w[0];
          *reinterpret_cast<uint4*>(dst + c + 8) = w[1];
        }
        named_bar(1, 128);
      }
      (void)et;
      tc_fence_before();
      mbar_arrive(o_empty);  // the next item's first PV may overwrite O
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

}  // namespace

bool attention_batch_supported(const AttnArgs& a) {
  return a.hd == HD && a.n_req > 0 && a.max_n <= 64 && !a.alibi && !a.mask && !a.block_id && a.d % 64 == 0;
}

void attention_batch(const AttnArgs& a, cudaStream_t s) {
  static bool attr = [] {
    PCB_CUDA(cudaFuncSetAttribute(k_attn_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    return true;
  }();
  (void)attr;
  static const int sms = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  BatchParams p;
  p.n_items = a.n_req * a.H;
  p.n_req = a.n_req;
  p.H = a.H;
  p.d = a.d;
  p.layer = a.layer;
  p.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(HD));
  p.out = static_cast<__nv_bfloat16*>(a.out);
  p.req = a.req;
  p.segs = a.segs;
  p.segn = a.segn;
  p.maps = static_cast<const CUtensorMap*>(a.maps);
  CUtensorMap tq = tmap_bf16_2d(a.q, static_cast<uint64_t>(a.n), static_cast<uint64_t>(a.d), 64);
  CUtensorMap tk = tq, tv = tq;
  if (!a.segs) {
    tk = tmap_bf16_3d(a.k, a.d, a.kv_cap, a.n_req, a.req_stride, BKV);
    tv = tmap_bf16_3d(a.v, a.d, a.kv_cap, a.n_req, a.req_stride, BKV);
  }
  PdlClass pc(PDL_ATTN);
  launch_k(k_attn_batch, dim3(static_cast<unsigned>(std::min(p.n_items, sms))), dim3(kThreads), kSmem, s, 1, tq, tk,
           tv, p);
}

}  // namespace pcb::kern

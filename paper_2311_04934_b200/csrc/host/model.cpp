// Device model: weights generated in HBM by the PCG jump-ahead kernel, and the
// per-layer launch sequence of the reference forward (model.cpp:304-443):
//   embed -> [LN1 -> QKV GEMM (+RoPE at schema positions, K/V written straight
//   into the request cache) -> attention -> O GEMM (+residual) -> LN2 -> W1 GEMM
//   (+GELU) -> W2 GEMM (+residual)] x L -> final LN -> unembed (last rows only).
#include "model.hpp"
#include "collective.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "../kernels/kernels.cuh"
#include "cuda_check.hpp"
#include "json.hpp"


namespace pcb::model {

uint64_t fnv1a64(const void* data, size_t len) {
  const auto* p = static_cast<const unsigned char*>(data);
  uint64_t h = 14695981039346656037ULL;
  for (size_t i = 0; i < len; ++i) {
    h ^= p[i];
    h *= 1099511628211ULL;
  }
  return h;
}

uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

// ---------------------------------------------------------------------------
// Config (reference model.cpp:59-96): same JSON keys, defaults and canonical
// serialization, so config hashes (and PCST files) interoperate.
// ---------------------------------------------------------------------------
static const char* pos_name(PosEncoding p) {
  return p == PosEncoding::Rope ? "rope" : p == PosEncoding::Alibi ? "alibi" : "abs_table";
}

ModelConfig ModelConfig::from_json(const std::string& text) {
  nlohmann::json j;
  try {
    j = nlohmann::json::parse(text);
  } catch (const std::exception& e) {
    throw Error(ErrorCode::InvalidConfig, std::string("bad config JSON: ") + e.what());
  }
  ModelConfig c;
  try {
    c.n_layers = j.value("n_layers", c.n_layers);
    c.n_heads = j.value("n_heads", c.n_heads);
    c.head_dim = j.value("head_dim", c.head_dim);
    c.hidden = j.value("hidden", c.n_heads * c.head_dim);
    c.vocab_size = j.value("vocab_size", c.vocab_size);
    std::string pe = j.value("pos_encoding", std::string("rope"));
    if (pe == "rope") c.pos_encoding = PosEncoding::Rope;
    else if (pe == "alibi") c.pos_encoding = PosEncoding::Alibi;
    else if (pe == "abs_table") c.pos_encoding = PosEncoding::AbsTable;
    else throw Error(ErrorCode::InvalidConfig, "unknown pos_encoding \"" + pe + "\"");
    c.max_position = j.value("max_position", c.max_position);
    c.bytes_per_element = j.value("bytes_per_element", c.bytes_per_element);
    c.seed = j.value("seed", c.seed);
  } catch (const nlohmann::json::exception& e) {
    throw Error(ErrorCode::InvalidConfig, std::string("bad config field: ") + e.what());
  }
  if (c.n_layers < 1 || c.n_heads < 1 || c.head_dim < 1 || c.hidden < 1 || c.vocab_size < 1 || c.max_position < 1 ||
      c.bytes_per_element < 1)
    throw Error(ErrorCode::InvalidConfig, "config fields must be positive");
  return c;
}

std::string ModelConfig::to_json() const {
  nlohmann::json j;
  j["n_layers"] = n_layers;
  j["n_heads"] = n_heads;
  j["head_dim"] = head_dim;
  j["hidden"] = hidden;
  j["vocab_size"] = vocab_size;
  j["pos_encoding"] = pos_name(pos_encoding);
  j["max_position"] = max_position;
  j["bytes_per_element"] = bytes_per_element;
  j["seed"] = seed;
  return j.dump();
}

uint64_t ModelConfig::hash() const {
  std::string s = to_json();
  return fnv1a64(s.data(), s.size());
}

// ---------------------------------------------------------------------------
KVBlock::~KVBlock() {
  if (data && !view) {
    if (host) cudaFreeHost(data);
    else cudaFree(data);
  }
}

struct Weights {
  float* embed = nullptr;
  void* unembed = nullptr;
  std::vector<void*> wqkv, wo, w1, w2;
  double *cos64 = nullptr, *sin64 = nullptr;
  float *cos32 = nullptr, *sin32 = nullptr;
  float* alibi = nullptr;
  float* abs_table = nullptr;
  bool packed = false;  // every bf16 GEMM weight in the tcgen05 tile layout
  bool pk_qkv = false, pk_o = false, pk_1 = false, pk_2 = false, pk_un = false;  // per weight kind
  // LN fold (bf16 chain): sum_k W[n][k] of the GEMMs that consume a LayerNorm output
  std::vector<float*> wsum_qkv, wsum_1;
  float* wsum_un = nullptr;
  std::vector<void*> owned;
  ~Weights() {
    for (void* p : owned) cudaFree(p);
  }
  void* alloc(size_t bytes) {
    void* p = nullptr;
    CK(cudaMalloc(&p, bytes));
    owned.push_back(p);
    return p;
  }
};

struct Workspace {
  int64_t cap_n = 0, cap_rows = 0, cap_logit = 0, cap_mask = 0;
  int d = 0, V = 0, dt = BF16;
  int32_t *tok = nullptr, *pos = nullptr, *kvpos = nullptr, *block = nullptr, *argmax = nullptr, *lrows = nullptr;
  int64_t* kvoff = nullptr;
  int4* req = nullptr;  // batched attention: {first q row, n, P, 0} per request
  uint8_t* mask = nullptr;
  float* h = nullptr;
  void *x = nullptr, *q = nullptr, *attn = nullptr, *mid = nullptr;
  float* logits = nullptr;
  float *part = nullptr, *logits_loc = nullptr, *logits_gath = nullptr;  // tensor parallel
  float* lnstats = nullptr;  // LN fold: [hidden/128 tiles][cap_n][2]
  float2* rope_tab = nullptr;  // [rope_half + 1][rope_ld] {cos, sin} per (pair, token), few-token forwards
  // batched zero-copy attention tables: one device blob [maps (128 B each)][segs int4 [B][16]][segn int2 [B]]
  char* segblob = nullptr;
  size_t segblob_cap = 0;
  char* seg_host = nullptr;  // pinned staging of the blob
  cudaEvent_t seg_ev = nullptr;  // the staging's last H2D ran
  int rope_half = 0;
  int64_t rope_ld = 0;
  int tp = 1, Vl = 0;
  float* gemm_ws = nullptr;
  size_t gemm_ws_bytes = 0;
  int* counters = nullptr;
  float* attn_scratch = nullptr;
  size_t attn_scratch_bytes = 0;
  int32_t* host_ints = nullptr;  // pinned staging
  int64_t host_ints_cap = 0;
  unsigned long long chain_bar = 0;  // arrivals issued so far on the chain's grid-barrier counter
  // counters layout (ints): [0, 8192) GEMM stream-K flags, [8192, 16384) attention split
  // counters, [16384, 32768) chain stream-K flags, [32768, 32770) chain grid barrier (u64)
  int* chain_flags() const { return counters + 16384; }
  unsigned long long* chain_gbar() const { return reinterpret_cast<unsigned long long*>(counters + 32768); }

  ~Workspace() {
    for (void* p : {(void*)tok, (void*)pos, (void*)kvpos, (void*)block, (void*)argmax, (void*)lrows, (void*)kvoff,
                    (void*)req,
                    (void*)mask, (void*)h, x, q,
                    attn, mid, (void*)logits, (void*)part, (void*)logits_loc, (void*)logits_gath, (void*)lnstats,
                    (void*)rope_tab, (void*)segblob, (void*)gemm_ws,
                    (void*)counters, (void*)attn_scratch})
      if (p) cudaFree(p);
    for (auto& e : staged)
      if (e) {
        cudaEventSynchronize(e);
        cudaEventDestroy(e);
      }
    if (host_ints) cudaFreeHost(host_ints);
    if (seg_host) cudaFreeHost(seg_host);
    if (seg_ev) cudaEventDestroy(seg_ev);
  }
  template <typename T>
  static void regrow(T*& p, size_t bytes) {
    if (p) cudaFree(p);
    p = nullptr;
    CK(cudaMalloc(reinterpret_cast<void**>(&p), bytes));
  }
  void ensure(int64_t n, int64_t rows, int64_t logit_rows, bool want_mask) {
    const size_t es = dt == F32 ? 4 : 2;
    if (n > cap_n) {
      int64_t c = std::max<int64_t>(n, 64);
      regrow(tok, c * 4);
      regrow(pos, c * 4);
      regrow(block, c * 4);
      regrow(kvoff, c * 8);
      regrow(lrows, c * 4);
      regrow(req, c * 16);
      regrow(h, c * d * 4);
      regrow(x, c * d * es);
      regrow(q, c * d * es);
      regrow(attn, c * d * es);
      regrow(mid, c * 4 * d * es);
      if (tp > 1) regrow(part, c * d * 4);
      regrow(lnstats, ((d + 127) / 128) * c * 8);
      if (rope_half > 0) {
        rope_ld = (c + 15) / 16 * 16 + 16;  // slack: split slices may read a chunk past n
        regrow(rope_tab, (rope_half + 1) * rope_ld * sizeof(float2));
      }
      cap_n = c;
    }
    if (rows > cap_rows) {
      int64_t c = std::max<int64_t>(rows, 256);
      // ALiBi key positions: per-segment padding to 64-key blocks + one block of slack
      regrow(kvpos, (c + 64 * (kern::ChainStep::kMaxSeg + 2)) * 4);
      cap_rows = c;
    }
    if (logit_rows > cap_logit) {
      int64_t c = std::max<int64_t>(logit_rows, 1);
      regrow(logits, c * V * 4);
      if (tp > 1) {
        regrow(logits_loc, c * Vl * 4);
        regrow(logits_gath, c * V * 4);
      }
      cap_logit = c;
    }
    if (want_mask && n * n > cap_mask) {
      regrow(mask, n * n);
      cap_mask = n * n;
    }
    if (!argmax) regrow(argmax, 1024 * 4);
    if (!gemm_ws) {
      gemm_ws_bytes = 64ull << 20;
      regrow(gemm_ws, gemm_ws_bytes);
      regrow(counters, 65536 * 4);
      CK(cudaMemset(counters, 0, 65536 * 4));
    }
    int64_t need_ints = 10 * n + rows + 64 * (kern::ChainStep::kMaxSeg + 2) + 32;
    if (need_ints > host_ints_cap) {
      for (int sl = 0; sl < 2; ++sl)
        if (staged[sl]) CK(cudaEventSynchronize(staged[sl]));
      if (host_ints) cudaFreeHost(host_ints);
      CK(cudaMallocHost(reinterpret_cast<void**>(&host_ints), 2 * need_ints * 4));
      host_ints_cap = need_ints;
    }
  }
  // Pinned staging for the per-call token / position uploads: two slots, each
  // reused only after the async H2D copies that read it have executed (the host
  // can run far ahead of the stream, e.g. back-to-back module precomputes).
  cudaEvent_t staged[2] = {nullptr, nullptr};
  int slot = 0;
  int32_t* acquire_staging() {
    slot ^= 1;
    if (!staged[slot]) CK(cudaEventCreateWithFlags(&staged[slot], cudaEventDisableTiming));
    else CK(cudaEventSynchronize(staged[slot]));
    return host_ints + slot * host_ints_cap;
  }
  void release_staging(cudaStream_t s) { CK(cudaEventRecord(staged[slot], s)); }
  void ensure_attn_scratch(size_t bytes) {
    if (bytes > attn_scratch_bytes) {
      regrow(attn_scratch, bytes);
      attn_scratch_bytes = bytes;
    }
  }
};

static std::string tname(int l, const char* t) { return "layer" + std::to_string(l) + "." + t; }

static uint64_t stream_seed(const std::string& name, uint64_t seed) {
  return splitmix64(fnv1a64(name.data(), name.size()) ^ splitmix64(seed));
}

Model::Model(const ModelConfig& c, int dtype, int device, int tp_rank, int tp_size,
             std::shared_ptr<coll::Collective> comm)
    : cfg_(c), dtype_(dtype), device_(device), tp_rank_(tp_rank), tp_size_(tp_size), comm_(std::move(comm)) {
  if (tp_size < 1 || tp_rank < 0 || tp_rank >= tp_size) throw Error(ErrorCode::InvalidConfig, "bad tensor-parallel rank");
  if (tp_size > 1 && (!comm_ || comm_->size != tp_size || comm_->rank != tp_rank))
    throw Error(ErrorCode::InvalidConfig, "tensor parallel needs a collective of the same size and rank");
  if (c.n_heads % tp_size || c.vocab_size % tp_size)
    throw Error(ErrorCode::InvalidConfig, "n_heads and vocab_size must divide by the tensor-parallel size");
  if (tp_size > 1 && c.pos_encoding == PosEncoding::Alibi)
    throw Error(ErrorCode::InvalidConfig, "tensor parallel: ALiBi is not sharded");
  dl_ = c.hidden / tp_size;
  fl_ = 4 * c.hidden / tp_size;
  vl_ = c.vocab_size / tp_size;
  if (const char* v = std::getenv("PCB_CHAIN")) use_chain = v[0] != '0';
  if (const char* v = std::getenv("PCB_LN_FOLD")) ln_fold = v[0] != '0';
  if (const char* v = std::getenv("PCB_CHAIN_ATTN")) chain_attn = v[0] != '0';
  if (const char* v = std::getenv("PCB_ZERO_COPY")) zero_copy = v[0] != '0';
  if (c.hidden != c.n_heads * c.head_dim) throw Error(ErrorCode::InvalidConfig, "hidden must equal n_heads * head_dim");
  if (c.n_layers < 1 || c.n_heads < 1 || c.head_dim < 2 || c.head_dim % 2 != 0)
    throw Error(ErrorCode::InvalidConfig, "bad layer/head geometry");
  if (c.vocab_size < 259)
    throw Error(ErrorCode::InvalidConfig, "vocab_size must be at least 259 to cover bytes plus specials");
  if (c.max_position < 1) throw Error(ErrorCode::InvalidConfig, "max_position must be positive");
  if (c.max_position > (1LL << 31) - 1) throw Error(ErrorCode::InvalidConfig, "max_position exceeds int32 device range");
  if (dtype != F32 && dtype != BF16) throw Error(ErrorCode::InvalidConfig, "dtype must be f32 or bf16");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Error(ErrorCode::CudaError, "no CUDA device: the Prompt Cache engine has no CPU fallback");
  CK(cudaSetDevice(device));
  CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  w_ = std::make_unique<Weights>();
  ws_ = std::make_unique<Workspace>();
  ws_->d = c.hidden;
  ws_->V = c.vocab_size;
  ws_->Vl = vl_;
  ws_->tp = tp_size;
  ws_->dt = dtype;
  if (c.pos_encoding == PosEncoding::Rope && dtype == BF16) ws_->rope_half = c.head_dim / 2;

  const int d = c.hidden;
  const size_t es = dtype == F32 ? 4 : 2;
  const float ws = 1.0f / std::sqrt(static_cast<float>(d));
  const float ws2 = 1.0f / std::sqrt(static_cast<float>(4 * d));
  const size_t Vd = static_cast<size_t>(c.vocab_size) * d;
  // weight init (reference model.cpp:191-218): same tensor names, scales, streams
  w_->embed = static_cast<float*>(w_->alloc(Vd * 4));
  kern::init_uniform(F32, w_->embed, Vd, stream_seed("embed", c.seed), 0.1f, stream_);
  // bf16 GEMM weights are stored pre-packed for the tcgen05 kernel (kernels.cuh
  // packed_index); fp32 weights stay row-major for the exact SIMT path.
  w_->pk_qkv = dtype == BF16 && kern::weight_packable(3 * dl_, d);
  w_->pk_o = dtype == BF16 && kern::weight_packable(d, dl_);
  w_->pk_1 = dtype == BF16 && kern::weight_packable(fl_, d);
  w_->pk_2 = dtype == BF16 && kern::weight_packable(d, fl_);
  w_->pk_un = dtype == BF16 && kern::weight_packable(vl_, d);
  w_->packed = w_->pk_qkv && w_->pk_o && w_->pk_1 && w_->pk_2 && w_->pk_un;
  void* staging = nullptr;
  if (dtype == BF16) CK(cudaMalloc(&staging, std::max<size_t>(4 * static_cast<size_t>(d) * d, Vd) * es));
  // One [N][K] weight from named stream blocks: each part is rows [row0, row0+rows) x
  // columns [col0, col0+K) of a full [*][full_cols] reference tensor (tensor-parallel
  // shards are row ranges of column-parallel and column ranges of row-parallel weights).
  struct Part {
    std::string name;
    float scale;
    int64_t rows, row0, col0, full_cols;
  };
  auto make = [&](int N, int K, std::vector<Part> parts, bool pack, float** row_sums = nullptr) {
    void* dst = w_->alloc(static_cast<size_t>(N) * K * es);
    char* gen = static_cast<char*>(pack ? staging : dst);
    size_t off = 0;
    for (auto& p : parts) {
      if (p.row0 == 0 && p.col0 == 0 && p.full_cols == K)
        kern::init_uniform(dtype, gen + off * es, static_cast<size_t>(p.rows) * K, stream_seed(p.name, c.seed), p.scale,
                           stream_);
      else
        kern::init_uniform_block(dtype, gen + off * es, p.rows, K, stream_seed(p.name, c.seed), p.scale, p.row0, p.col0,
                                 p.full_cols, stream_);
      off += static_cast<size_t>(p.rows) * K;
    }
    if (row_sums && dtype == BF16) {
      *row_sums = static_cast<float*>(w_->alloc(static_cast<size_t>(N) * 4));
      kern::row_sums_bf16(gen, N, K, *row_sums, stream_);
    }
    if (pack) kern::pack_weight_bf16(staging, dst, N, K, stream_);
    return dst;
  };
  const int r = tp_rank_;
  w_->unembed = make(vl_, d, {{"unembed", ws, vl_, static_cast<int64_t>(r) * vl_, 0, d}}, w_->pk_un, &w_->wsum_un);
  for (int l = 0; l < c.n_layers; ++l) {
    const int64_t h0 = static_cast<int64_t>(r) * dl_;
    float *sq = nullptr, *s1 = nullptr;
    w_->wqkv.push_back(make(3 * dl_, d,
                            {{tname(l, "wq"), ws, dl_, h0, 0, d}, {tname(l, "wk"), ws, dl_, h0, 0, d},
                             {tname(l, "wv"), ws, dl_, h0, 0, d}},
                            w_->pk_qkv, &sq));
    w_->wsum_qkv.push_back(sq);
    w_->wo.push_back(make(d, dl_, {{tname(l, "wo"), ws, d, 0, h0, d}}, w_->pk_o));
    w_->w1.push_back(make(fl_, d, {{tname(l, "w1"), ws, fl_, static_cast<int64_t>(r) * fl_, 0, d}}, w_->pk_1, &s1));
    w_->wsum_1.push_back(s1);
    w_->w2.push_back(make(d, fl_, {{tname(l, "w2"), ws2, d, 0, static_cast<int64_t>(r) * fl_, 4 * d}}, w_->pk_2));
  }
  if (staging) {
    CK(cudaStreamSynchronize(stream_));
    cudaFree(staging);
  }
  if (c.pos_encoding == PosEncoding::Rope) {  // model.cpp:220-230, glibc fp64 table
    const int half = c.head_dim / 2;
    const size_t cnt = static_cast<size_t>(c.max_position) * half;
    std::vector<double> cs(cnt), sn(cnt);
    for (int64_t p = 0; p < c.max_position; ++p)
      for (int i = 0; i < half; ++i) {
        double theta = std::pow(10000.0, -2.0 * i / c.head_dim);
        cs[p * half + i] = std::cos(static_cast<double>(p) * theta);
        sn[p * half + i] = std::sin(static_cast<double>(p) * theta);
      }
    if (dtype == F32) {
      w_->cos64 = static_cast<double*>(w_->alloc(cnt * 8));
      w_->sin64 = static_cast<double*>(w_->alloc(cnt * 8));
      CK(cudaMemcpy(w_->cos64, cs.data(), cnt * 8, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(w_->sin64, sn.data(), cnt * 8, cudaMemcpyHostToDevice));
    } else {
      std::vector<float> c32(cnt), s32(cnt);
      for (size_t i = 0; i < cnt; ++i) {
        c32[i] = static_cast<float>(cs[i]);
        s32[i] = static_cast<float>(sn[i]);
      }
      w_->cos32 = static_cast<float*>(w_->alloc(cnt * 4));
      w_->sin32 = static_cast<float*>(w_->alloc(cnt * 4));
      CK(cudaMemcpy(w_->cos32, c32.data(), cnt * 4, cudaMemcpyHostToDevice));
      CK(cudaMemcpy(w_->sin32, s32.data(), cnt * 4, cudaMemcpyHostToDevice));
    }
  }
  if (c.pos_encoding == PosEncoding::Alibi) {  // model.cpp:231-236
    std::vector<float> sl(c.n_heads);
    for (int h = 0; h < c.n_heads; ++h) sl[h] = static_cast<float>(std::pow(2.0, -8.0 * (h + 1) / c.n_heads));
    w_->alibi = static_cast<float*>(w_->alloc(c.n_heads * 4));
    CK(cudaMemcpy(w_->alibi, sl.data(), c.n_heads * 4, cudaMemcpyHostToDevice));
  }
  if (c.pos_encoding == PosEncoding::AbsTable) {  // model.cpp:237-245
    const size_t cnt = static_cast<size_t>(c.max_position) * d;
    std::vector<float> t(cnt);
    for (int64_t p = 0; p < c.max_position; ++p)
      for (int i = 0; i < d / 2; ++i) {
        double theta = static_cast<double>(p) / std::pow(10000.0, 2.0 * i / d);
        t[p * d + 2 * i] = static_cast<float>(std::sin(theta));
        t[p * d + 2 * i + 1] = static_cast<float>(std::cos(theta));
      }
    w_->abs_table = static_cast<float*>(w_->alloc(cnt * 4));
    CK(cudaMemcpy(w_->abs_table, t.data(), cnt * 4, cudaMemcpyHostToDevice));
  }
  CK(cudaStreamSynchronize(stream_));
}

struct Model::Prof {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  struct Rec {
    int cat;
    cudaEvent_t a, b;
    double bytes, flops;
  };
  std::vector<Rec> recs;
  cudaEvent_t pending = nullptr;
  double ms[PROF_N] = {}, bytes[PROF_N] = {}, flops[PROF_N] = {};
  int64_t count[PROF_N] = {};
  cudaEvent_t get() {
    if (pool.empty()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  ~Prof() {
    for (auto e : pool) cudaEventDestroy(e);
    for (auto& r : recs) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
  }
};

void Model::set_profiling(bool on) {
  if (!prof_) prof_ = std::make_unique<Prof>();
  prof_->on = on;
}
void Model::prof_begin() {
  if (!prof_ || !prof_->on) return;
  prof_->pending = prof_->get();
  CK(cudaEventRecord(prof_->pending, stream_));
}
void Model::prof_end(int cat, double alg_bytes, double alg_flops) {
  ++launches;
  static const bool sync_debug = std::getenv("PCB_SYNC_DEBUG") != nullptr;  // hang bisection aid
  if (sync_debug) {
    static const char* names[PROF_N] = {"gemm", "attention", "assembly", "other"};
    std::fprintf(stderr, "[pcb] launch %lld (%s, %.0f bytes) ...", static_cast<long long>(launches), names[cat], alg_bytes);
    CK(cudaStreamSynchronize(stream_));
    std::fprintf(stderr, " done\n");
  }
  if (!prof_ || !prof_->on || !prof_->pending) return;
  cudaEvent_t b = prof_->get();
  CK(cudaEventRecord(b, stream_));
  prof_->recs.push_back({cat, prof_->pending, b, alg_bytes, alg_flops});
  prof_->pending = nullptr;
}
std::string Model::profile_json() {
  nlohmann::json j = nlohmann::json::object();
  if (!prof_) return j.dump();
  CK(cudaStreamSynchronize(stream_));
  for (auto& r : prof_->recs) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, r.a, r.b));
    prof_->ms[r.cat] += ms;
    prof_->bytes[r.cat] += r.bytes;
    prof_->flops[r.cat] += r.flops;
    prof_->count[r.cat] += 1;
    prof_->pool.push_back(r.a);
    prof_->pool.push_back(r.b);
  }
  prof_->recs.clear();
  const char* names[PROF_N] = {"gemm", "attention", "assembly", "other"};
  for (int c = 0; c < PROF_N; ++c) {
    j[names[c]] = {{"ms", prof_->ms[c]}, {"launches", prof_->count[c]}, {"bytes", prof_->bytes[c]},
                   {"flops", prof_->flops[c]}};
    prof_->ms[c] = prof_->bytes[c] = prof_->flops[c] = 0;
    prof_->count[c] = 0;
  }
  return j.dump();
}

Model::~Model() {
  if (stream_) {
    cudaStreamSynchronize(stream_);
    kern::chain_forget_stream(stream_);
    cudaStreamDestroy(stream_);
  }
}

KVPtr Model::alloc_kv(int64_t cap, bool host) const {
  auto kv = std::make_shared<KVBlock>();
  kv->dtype = dtype_;
  kv->n_layers = cfg_.n_layers;
  kv->hidden = dl_;
  kv->cap = cap;
  kv->host = host;
  if (cap > 0) {
    if (host) CK(cudaMallocHost(&kv->data, kv->bytes()));
    else CK(cudaMalloc(&kv->data, kv->bytes()));
  }
  return kv;
}

void Model::copy_rows(const KVBlock& src, KVBlock& dst, int64_t dst_row) const {
  if (src.rows == 0) return;
  if (dst_row + src.rows > dst.cap) throw Error(ErrorCode::Internal, "copy_rows: destination too small");
  const cudaMemcpyKind kind = src.host ? (dst.host ? cudaMemcpyHostToHost : cudaMemcpyHostToDevice)
                                       : (dst.host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
  const size_t rb = src.row_bytes();
  // every plane is one strided 2-D copy: L*2 rows of src.rows*rb bytes
  CK(cudaMemcpy2DAsync(dst.data == nullptr ? nullptr : dst.plane(0, 0) + dst_row * rb, dst.plane_bytes(),
                       src.plane(0, 0), src.plane_bytes(), src.rows * rb, 2 * src.n_layers, kind, stream_));
}

KVPtr Model::to_host(const KVBlock& src) const {
  KVPtr h = alloc_kv(src.rows, true);
  copy_rows(src, *h, 0);
  h->rows = src.rows;
  h->positions = src.positions;
  CK(cudaStreamSynchronize(stream_));
  return h;
}

void Model::validate(const int32_t* tokens, const int64_t* positions, int64_t n, const KVBlock& kv) const {
  for (int64_t i = 0; i < n; ++i) {
    if (positions[i] < 0 || positions[i] >= cfg_.max_position)
      throw Error(ErrorCode::PositionOutOfRange, "position " + std::to_string(positions[i]) + " outside [0, " +
                                                     std::to_string(cfg_.max_position) + ")");
    if (tokens[i] < 0 || tokens[i] >= cfg_.vocab_size)
      throw Error(ErrorCode::ShapeMismatch, "token id out of vocab range");
  }
  if (kv.n_layers != cfg_.n_layers || kv.hidden != dl_ || kv.dtype != dtype_)
    throw Error(ErrorCode::ShapeMismatch, "past KV shape mismatch");
  if (kv.host) throw Error(ErrorCode::ShapeMismatch, "forward needs a device-resident KV block");
  if (kv.rows + n > kv.cap) throw Error(ErrorCode::ShapeMismatch, "KV block capacity exceeded");
}

static double gemm_alg_bytes(int dtype, int64_t M, int N, int K, int epi_kind) {
  const double es = dtype == F32 ? 4.0 : 2.0;
  const double out_b = epi_kind == kern::EPI_RESID ? 8.0 : (epi_kind == kern::EPI_F32 ? 4.0 : es);
  return (double)N * K * es + (double)M * K * es + (double)M * N * out_b;
}

void Model::chain(const void* steps_v, int n_steps) {
  const auto* steps = static_cast<const kern::ChainStep*>(steps_v);
  double bytes = 0, flops = 0;
  for (int i = 0; i < n_steps; ++i) {
    const auto& st = steps[i];
    if (st.kind == kern::CHAIN_GEMM) {
      bytes += gemm_alg_bytes(dtype_, st.M, st.N, st.K, st.e.kind);
      flops += 2.0 * st.M * st.N * st.K;
    } else if (st.kind == kern::CHAIN_ATTN) {
      bytes += 2.0 * (st.aP + st.M) * st.a_d * 2 + 2.0 * st.M * st.a_d * 2;
      flops += 4.0 * st.M * st.a_d * (st.aP + (st.M + 1) / 2.0);
    } else {
      bytes += 6.0 * st.M * st.ln_d;
    }
  }
  prof_begin();
  kern::chain_tc(steps, n_steps, ws_->gemm_ws, ws_->gemm_ws_bytes, ws_->chain_flags(), ws_->chain_gbar(),
                 ws_->chain_bar, stream_);
  prof_end(PROF_GEMM, bytes, flops);
}

void Model::gemm(const void* A, const void* W, int64_t M, int N, int K, const void* epi, bool packed) {
  const auto& e = *static_cast<const kern::Epilogue*>(epi);
  prof_begin();
  if (packed && !force_simt && !force_simt_gemm && kern::gemm_tc_supported(M, N, K))
    kern::gemm_tc(A, W, M, N, K, e, ws_->gemm_ws, ws_->gemm_ws_bytes, ws_->counters, stream_);
  else
    kern::gemm_simt(dtype_, A, W, M, N, K, e, stream_, packed);
  // algorithmic bytes: weights + activations in + outputs (residual: read + write fp32)
  prof_end(PROF_GEMM, gemm_alg_bytes(dtype_, M, N, K, e.kind), 2.0 * M * N * K);
}

void Model::set_kv_prefix(const std::vector<const KVBlock*>& blocks) {
  if (static_cast<int>(blocks.size()) + 1 > kern::ChainStep::kMaxSeg)
    throw Error(ErrorCode::ShapeMismatch, "zero-copy prefix: too many blocks");
  kv_prefix_.clear();
  kv_prefix_rows_ = 0;
  for (const KVBlock* b : blocks) {
    if (b->host || b->dtype != dtype_ || b->hidden != cfg_.hidden || b->n_layers != cfg_.n_layers)
      throw Error(ErrorCode::ShapeMismatch, "zero-copy prefix: block must be a device block of this model");
    if (b->rows == 0) continue;
    kv_prefix_.push_back(b);
    kv_prefix_rows_ += b->rows;
  }
}

void Model::set_kv_prefix_batch(const std::vector<std::vector<const KVBlock*>>& per_request) {
  kv_prefix_batch_.clear();
  for (const auto& blocks : per_request) {
    if (static_cast<int>(blocks.size()) + 1 > kern::kAttnMaxSeg)
      throw Error(ErrorCode::ShapeMismatch, "zero-copy prefix: too many blocks");
    std::vector<const KVBlock*> keep;
    for (const KVBlock* b : blocks) {
      if (b->host || b->dtype != dtype_ || b->hidden != cfg_.hidden || b->n_layers != cfg_.n_layers)
        throw Error(ErrorCode::ShapeMismatch, "zero-copy prefix: block must be a device block of this model");
      if (b->rows) keep.push_back(b);
    }
    kv_prefix_batch_.push_back(std::move(keep));
  }
}

bool Model::batched_zero_copy_ok() const {
  const auto& c = cfg_;
  kern::AttnArgs a;
  a.hd = c.head_dim;
  a.d = c.hidden;
  a.n = 1;
  return zero_copy && tp_size_ == 1 && dtype_ == BF16 && !force_simt && !force_simt_attn &&
         c.pos_encoding != PosEncoding::Alibi && kern::attention_tc_supported(a);
}

bool Model::fused_attention_ok(int64_t n) const {
  const auto& c = cfg_;
  const int d = c.hidden;
  return use_chain && chain_attn && tp_size_ == 1 && dtype_ == BF16 && w_->packed && !force_simt && !force_simt_gemm &&
         !force_simt_attn && c.head_dim == 128 && kern::chain_ln_supported(d) &&
         kern::chain_tc_supported(n, 3 * d, d) && kern::chain_tc_supported(n, 4 * d, d) &&
         kern::chain_tc_supported(n, d, 4 * d) && kern::chain_tc_supported(1, c.vocab_size, d) &&
         kern::chain_attn_supported(n, 0, c.n_heads, c.head_dim);
}

void Model::run(const int32_t* tokens, const int64_t* positions, int64_t n, KVBlock& kv, const uint8_t* mask,
                const int32_t* block_ids, int64_t logit_rows) {
  BatchItem it{tokens, positions, n, &kv};
  run_impl(&it, 1, mask, block_ids, logit_rows, false);
}

void Model::run_batch(const std::vector<BatchItem>& items, bool last_row_logits) {
  if (items.empty()) return;
  for (size_t i = 1; i < items.size(); ++i)
    if (items[i].kv->cap != items[0].kv->cap)
      throw Error(ErrorCode::ShapeMismatch, "run_batch: every request cache must have the same capacity");
  run_impl(items.data(), static_cast<int>(items.size()), nullptr, nullptr, last_row_logits ? 1 : 0, true);
}

// One forward over B token segments (requests) concatenated along the token axis:
// GEMMs, LayerNorm and the fused epilogues see all M = sum(n_i) rows at once (one
// weight stream for the micro-batch); attention runs per segment over that
// segment's own cache; QKV writes each token's K/V row into its own request cache.
// Logits: the last `logit_rows` rows (B == 1), or the last row of every segment
// (gathered, per_segment_logits).
void Model::run_impl(const BatchItem* items, int B, const uint8_t* mask, const int32_t* block_ids,
                     int64_t logit_rows, bool per_segment_logits) {
  CK(cudaSetDevice(device_));
  int64_t n = 0, max_total = 0;
  for (int b = 0; b < B; ++b) {
    validate(items[b].tokens, items[b].positions, items[b].n, *items[b].kv);
    n += items[b].n;
    max_total = std::max(max_total, items[b].kv->rows + items[b].n);
  }
  KVBlock& kv = *items[0].kv;
  if (B > 1 && (mask || block_ids || cfg_.pos_encoding == PosEncoding::Alibi))
    throw Error(ErrorCode::ShapeMismatch, "batched forward: masks, block ids and ALiBi take one request");
  if (mask && kv.rows) throw Error(ErrorCode::ShapeMismatch, "masked forward takes no past KV");
  if (mask)
    for (int64_t i = 0; i < n; ++i)
      if (!mask[i * n + i]) throw Error(ErrorCode::ShapeMismatch, "mask diagonal must be true");
  if (n <= 0) return;
  for (int b = 0; b < B; ++b)
    if (items[b].n <= 0) throw Error(ErrorCode::ShapeMismatch, "batched forward: empty request");
  if (!kv_prefix_.empty() && (B != 1 || mask || block_ids || !fused_attention_ok(n)))
    throw Error(ErrorCode::ShapeMismatch, "zero-copy prefix set for a forward that cannot read it in place");
  if (!kv_prefix_batch_.empty() && (static_cast<int>(kv_prefix_batch_.size()) != B || B < 2 || !batched_zero_copy_ok()))
    throw Error(ErrorCode::ShapeMismatch, "zero-copy batch prefixes do not match this forward");
  logit_rows = per_segment_logits ? (logit_rows > 0 ? B : 0) : std::min(logit_rows, n);
  forward_tokens.fetch_add(n, std::memory_order_relaxed);
  const auto& c = cfg_;
  const int d = c.hidden, H = c.n_heads, hd = c.head_dim;
  const int64_t P = kv.rows, total = P + n;
  const double es = dtype_ == F32 ? 4.0 : 2.0;
  Workspace& W = *ws_;
  W.ensure(n, std::max(total, max_total), logit_rows, mask != nullptr);
  cudaStream_t s = stream_;
  const int32_t* tokens = items[0].tokens;
  const int64_t* positions = items[0].positions;
  std::vector<int32_t> cat_tok;
  std::vector<int64_t> cat_pos;
  if (B > 1) {
    cat_tok.reserve(n);
    cat_pos.reserve(n);
    for (int b = 0; b < B; ++b) {
      cat_tok.insert(cat_tok.end(), items[b].tokens, items[b].tokens + items[b].n);
      cat_pos.insert(cat_pos.end(), items[b].positions, items[b].positions + items[b].n);
    }
    tokens = cat_tok.data();
    positions = cat_pos.data();
  }

  // stage token ids / int32 positions (positions < max_position < 2^31, checked)
  int32_t* hi = W.acquire_staging();
  for (int64_t i = 0; i < n; ++i) {
    hi[i] = tokens[i];
    hi[n + i] = static_cast<int32_t>(positions[i]);
  }
  CK(cudaMemcpyAsync(W.tok, hi, n * 4, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(W.pos, hi + n, n * 4, cudaMemcpyHostToDevice, s));
  if (device_token_ && B == 1 && n == 1)  // decode: the previous step's argmax, no host round trip
    CK(cudaMemcpyAsync(W.tok, device_token_, 4, cudaMemcpyDeviceToDevice, s));
  const bool alibi = c.pos_encoding == PosEncoding::Alibi;
  int64_t kp_len = 0;
  if (alibi) {
    // every key's position in key order; with a zero-copy prefix in key-BLOCK order (each
    // segment -- a store block read in place, then the request's own rows -- padded to whole
    // 64-key blocks, as the chain's attention phase walks them).  Zero slack after the last
    // block: the attention kernels copy whole blocks of positions.
    int32_t* kp = hi + 2 * n;
    auto pad = [&]() {
      while (kp_len % 64) kp[kp_len++] = 0;
    };
    if (!kv_prefix_.empty()) {
      for (const KVBlock* b : kv_prefix_) {
        for (int64_t p : b->positions) kp[kp_len++] = static_cast<int32_t>(p);
        pad();
      }
      for (int64_t j = kv_prefix_rows_; j < P; ++j) kp[kp_len++] = static_cast<int32_t>(kv.positions[j]);
    } else {
      for (int64_t j = 0; j < P; ++j) kp[kp_len++] = static_cast<int32_t>(kv.positions[j]);
    }
    for (int64_t i = 0; i < n; ++i) kp[kp_len++] = static_cast<int32_t>(positions[i]);
    pad();
    for (int i = 0; i < 64; ++i) kp[kp_len++] = 0;
    CK(cudaMemcpyAsync(W.kvpos, kp, kp_len * 4, cudaMemcpyHostToDevice, s));
  }
  if (mask) CK(cudaMemcpyAsync(W.mask, mask, n * n, cudaMemcpyHostToDevice, s));
  if (block_ids) {
    int32_t* bp = hi + 2 * n + kp_len;
    std::memcpy(bp, block_ids, n * 4);
    CK(cudaMemcpyAsync(W.block, bp, n * 4, cudaMemcpyHostToDevice, s));
  }
  std::vector<int64_t> seg_start(B);
  if (B > 1) {
    // per token: K/V element offset of its cache row relative to request 0's layer planes
    // (equal capacities make the offset layer-independent); gathered logit rows
    int64_t* ko = reinterpret_cast<int64_t*>((reinterpret_cast<uintptr_t>(hi + 2 * n) + 7) & ~uintptr_t(7));
    int32_t* lr = reinterpret_cast<int32_t*>(ko + n);
    int64_t m = 0;
    for (int b = 0; b < B; ++b) {
      seg_start[b] = m;
      const int64_t base = (static_cast<char*>(items[b].kv->data) - static_cast<char*>(kv.data)) /
                           static_cast<int64_t>(items[b].kv->elem());
      for (int64_t j = 0; j < items[b].n; ++j, ++m) ko[m] = base + (items[b].kv->rows + j) * dl_;
      lr[b] = static_cast<int32_t>(m - 1);
    }
    int4* rq = reinterpret_cast<int4*>((reinterpret_cast<uintptr_t>(lr + B) + 15) & ~uintptr_t(15));
    for (int b = 0; b < B; ++b)
      rq[b] = make_int4(static_cast<int>(seg_start[b]), static_cast<int>(items[b].n),
                        static_cast<int>(items[b].kv->rows), 0);
    CK(cudaMemcpyAsync(W.kvoff, ko, n * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(W.lrows, lr, B * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(W.req, rq, B * 16, cudaMemcpyHostToDevice, s));
  }
  W.release_staging(s);

  prof_begin();
  // few-token forwards: the QKV epilogue reads this request's RoPE rows from a compact table
  const bool rope_tab = W.rope_half > 0 && n <= 128;
  if (rope_tab)
    kern::embed(W.tok, W.pos, n, w_->embed, w_->abs_table, d, W.h, s, w_->cos32, w_->sin32, W.rope_half, W.rope_tab,
                W.rope_ld);
  else
    kern::embed(W.tok, W.pos, n, w_->embed, w_->abs_table, d, W.h, s);
  prof_end(PROF_OTHER, 8.0 * n * d, 0);

  kern::AttnArgs aa;
  aa.n = n;
  aa.P = P;
  aa.H = H / tp_size_;
  aa.hd = hd;
  aa.d = dl_;
  aa.q = W.q;
  aa.out = W.attn;
  aa.mask = mask ? W.mask : nullptr;
  aa.block_id = block_ids ? W.block : nullptr;
  aa.alibi = alibi ? w_->alibi : nullptr;
  aa.kv_pos = alibi ? W.kvpos : nullptr;
  aa.counters = W.counters + 8192;  // [0, #SMs) are the GEMM's stream-K flags
  aa.pair = attn_pair;
  const bool tc_attn = dtype_ == BF16 && !force_simt && !force_simt_attn && kern::attention_tc_supported(aa);
  int64_t nq = n;
  if (!tc_attn) {
    const size_t per_q = static_cast<size_t>(H) * total * sizeof(double);
    const size_t budget = 512ull << 20;
    nq = std::max<int64_t>(1, std::min<int64_t>(n, static_cast<int64_t>(budget / per_q)));
    W.ensure_attn_scratch(per_q * nq);
  } else {
    W.ensure_attn_scratch(64ull << 20);
  }

  auto qkv_epi = [&](int l) {
    kern::Epilogue e;
    e.kind = kern::EPI_QKV;
    e.d = dl_;
    e.q_out = W.q;
    e.k_out = kv.k(l);
    e.v_out = kv.v(l);
    e.kv_row0 = P;
    e.kv_off = B > 1 ? W.kvoff : nullptr;
    e.pos = W.pos;
    e.rope = c.pos_encoding == PosEncoding::Rope;
    e.head_dim = hd;
    e.rope_cos64 = w_->cos64;
    e.rope_sin64 = w_->sin64;
    e.rope_cos32 = w_->cos32;
    e.rope_sin32 = w_->sin32;
    if (rope_tab) {
      e.rope_tab = W.rope_tab;
      e.rope_ld = W.rope_ld;
    }
    return e;
  };
  kern::Epilogue eo;
  eo.kind = kern::EPI_RESID;
  eo.resid = W.h;
  kern::Epilogue eg;
  eg.kind = kern::EPI_GELU;
  eg.out = W.mid;
  kern::Epilogue ef;
  ef.kind = kern::EPI_F32;
  ef.outf = tp_size_ > 1 ? W.logits_loc : W.logits;
  ef.ldo = vl_;
  // tensor parallel: row-parallel GEMM partials -> all-reduce -> residual add
  kern::Epilogue epart;
  epart.kind = kern::EPI_F32;
  epart.outf = W.part;
  epart.ldo = d;
  auto tp_reduce_into_h = [&]() {
    comm_->all_reduce_sum(W.part, static_cast<size_t>(n) * d, s);
    prof_begin();
    kern::add_inplace(W.h, W.part, n * d, s);
    prof_end(PROF_OTHER, 12.0 * n * d, 0);
  };
  // logits of `rows` LN'd rows in W.x: this rank's vocab rows, gathered over ranks
  auto unembed = [&](int64_t rows) {
    gemm(W.x, w_->unembed, rows, vl_, d, &ef, w_->pk_un);
    if (tp_size_ > 1) {
      comm_->all_gather(W.logits_loc, W.logits_gath, static_cast<size_t>(rows) * vl_, s);
      kern::interleave_shards(W.logits_gath, tp_size_, rows, vl_, W.logits, s);
    }
  };

  // batched attention in one launch when the request caches sit at a uniform stride
  int64_t req_stride = 0, max_P = 0, max_nb = 0;
  bool batched_attn = B > 1 && tc_attn;
  if (batched_attn) {
    req_stride = static_cast<char*>(items[1].kv->data) - static_cast<char*>(items[0].kv->data);
    for (int b = 0; b < B; ++b) {
      batched_attn = batched_attn && req_stride > 0 && items[b].n <= 128 &&
                     static_cast<char*>(items[b].kv->data) - static_cast<char*>(items[0].kv->data) == b * req_stride;
      max_P = std::max(max_P, items[b].kv->rows);
      max_nb = std::max(max_nb, items[b].n);
    }
  }
  // Batched attention reads every request's keys through per-request segment tables: the
  // request's own cache rows [0, P + n) (one 3-D map per request, rows ending at its last
  // valid row so the rest of a 64-row block is TMA zero fill -- a masked key has P = 0 but
  // 0 * NaN of stale memory in PV is NaN), preceded, on the zero-copy path, by its module
  // blocks read in place (plane = 2 layer + K/V).
  int64_t seg_max_blocks = 0;
  const int4* d_segs = nullptr;
  const int2* d_segn = nullptr;
  const void* d_maps = nullptr;
  if (!kv_prefix_batch_.empty() && !batched_attn)
    throw Error(ErrorCode::ShapeMismatch, "zero-copy batch needs the batched attention path");
  if (batched_attn) {
    const int L2 = 2 * c.n_layers;
    std::vector<CUtensorMap> maps;
    std::map<const void*, int> map_of;
    std::vector<int4> tab(static_cast<size_t>(B) * kern::kAttnMaxSeg, make_int4(0, 0, 0, 0));
    std::vector<int2> segn(B);
    for (int b = 0; b < B; ++b) {
      int g = 0;
      int64_t pre = 0, blocks = 0;
      if (!kv_prefix_batch_.empty())
        for (const KVBlock* blk : kv_prefix_batch_[b]) {
          auto it = map_of.find(blk->data);
          if (it == map_of.end()) {
            it = map_of.emplace(blk->data, static_cast<int>(maps.size())).first;
            maps.push_back(kern::tmap_bf16_3d(blk->data, d, blk->rows, L2, blk->plane_bytes(), 64));
          }
          tab[b * kern::kAttnMaxSeg + g++] = make_int4(it->second, 0, static_cast<int>(blk->rows), 0);
          pre += blk->rows;
          blocks += (blk->rows + 63) / 64;
        }
      const KVBlock& rk = *items[b].kv;
      const int64_t Pb = rk.rows, nb = items[b].n;
      if (pre > Pb) throw Error(ErrorCode::ShapeMismatch, "zero-copy batch: prefix longer than the cache");
      const int own = static_cast<int>(maps.size());
      maps.push_back(kern::tmap_bf16_3d(rk.data, d, Pb + nb, L2, rk.plane_bytes(), 64));
      tab[b * kern::kAttnMaxSeg + g++] = make_int4(own, static_cast<int>(pre), static_cast<int>(Pb + nb - pre), 0);
      blocks += (Pb + nb - pre + 63) / 64;
      segn[b] = make_int2(g, static_cast<int>(Pb - pre));
      seg_max_blocks = std::max(seg_max_blocks, blocks);
    }
    const size_t mb = maps.size() * sizeof(CUtensorMap), tb = tab.size() * sizeof(int4), nbb = segn.size() * sizeof(int2);
    const size_t need = mb + tb + nbb;
    if (W.seg_ev) CK(cudaEventSynchronize(W.seg_ev));  // the pinned staging's previous H2D ran
    else CK(cudaEventCreateWithFlags(&W.seg_ev, cudaEventDisableTiming));
    if (need > W.segblob_cap) {
      CK(cudaStreamSynchronize(s));
      if (W.segblob) cudaFree(W.segblob);
      if (W.seg_host) cudaFreeHost(W.seg_host);
      W.segblob_cap = std::max<size_t>(need * 2, 64 << 10);
      CK(cudaMalloc(reinterpret_cast<void**>(&W.segblob), W.segblob_cap));
      CK(cudaMallocHost(reinterpret_cast<void**>(&W.seg_host), W.segblob_cap));
    }
    std::memcpy(W.seg_host, maps.data(), mb);
    std::memcpy(W.seg_host + mb, tab.data(), tb);
    std::memcpy(W.seg_host + mb + tb, segn.data(), nbb);
    CK(cudaMemcpyAsync(W.segblob, W.seg_host, need, cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(W.seg_ev, s));
    d_maps = W.segblob;
    d_segs = reinterpret_cast<const int4*>(W.segblob + mb);
    d_segn = reinterpret_cast<const int2*>(W.segblob + mb + tb);
  }
  std::vector<cudaEvent_t> layer_ev;
  layer_ev.swap(layer_events_);  // consumed by this call
  auto attention = [&](int l) {
    if (l < static_cast<int>(layer_ev.size())) CK(cudaStreamWaitEvent(s, layer_ev[l], 0));
    if (batched_attn) {
      kern::AttnArgs ab = aa;
      ab.n = n;
      ab.P = 0;
      ab.k = kv.k(l);
      ab.v = kv.v(l);
      ab.req = W.req;
      ab.n_req = B;
      ab.req_stride = req_stride;
      ab.kv_cap = kv.cap;
      ab.max_P = max_P;
      ab.max_n = max_nb;
      if (d_segs) {
        ab.segs = d_segs;
        ab.segn = d_segn;
        ab.maps = d_maps;
        ab.layer = l;
        ab.max_blocks = seg_max_blocks;
      }
      double bytes = 0, flops = 0;
      for (int b = 0; b < B; ++b) {
        const int64_t nb = items[b].n, Pb = items[b].kv->rows;
        bytes += 2.0 * (Pb + nb) * dl_ * es + 2.0 * nb * dl_ * es;
        flops += 4.0 * (double)nb * dl_ * (Pb + (nb + 1) / 2.0);
      }
      prof_begin();
      kern::attention_tc(ab, W.attn_scratch, W.attn_scratch_bytes, s);
      prof_end(PROF_ATTN, bytes, flops);
      return;
    }
    if (B > 1) {
      double bytes = 0, flops = 0;
      prof_begin();
      for (int b = 0; b < B; ++b) {
        const KVBlock& kb = *items[b].kv;
        const int64_t nb = items[b].n, Pb = kb.rows;
        kern::AttnArgs ab = aa;
        ab.n = nb;
        ab.P = Pb;
        ab.q = static_cast<const char*>(aa.q) + seg_start[b] * dl_ * static_cast<int64_t>(es);
        ab.out = static_cast<char*>(aa.out) + seg_start[b] * dl_ * static_cast<int64_t>(es);
        ab.k = kb.k(l);
        ab.v = kb.v(l);
        if (tc_attn && kern::attention_tc_supported(ab)) {
          kern::attention_tc(ab, W.attn_scratch, W.attn_scratch_bytes, s);
        } else {
          const size_t per_q = static_cast<size_t>(H) * (Pb + nb) * sizeof(double);
          const int64_t nqb = std::max<int64_t>(1, std::min<int64_t>(nb, static_cast<int64_t>((512ull << 20) / per_q)));
          W.ensure_attn_scratch(per_q * nqb);
          for (int64_t i0 = 0; i0 < nb; i0 += nqb) {
            ab.i0 = i0;
            ab.nq = std::min(nqb, nb - i0);
            kern::attention_simt(dtype_, ab, W.attn_scratch, s);
          }
        }
        if (b) ++launches;
        bytes += 2.0 * (Pb + nb) * dl_ * es + 2.0 * nb * dl_ * es;
        flops += 4.0 * (double)nb * dl_ * (Pb + (nb + 1) / 2.0);
      }
      prof_end(PROF_ATTN, bytes, flops);
      return;
    }
    aa.k = kv.k(l);
    aa.v = kv.v(l);
    // algorithmic work: every visible key/value row read once, q in, out written
    const double attn_bytes = 2.0 * total * dl_ * es + 2.0 * n * dl_ * es;
    const double attn_flops = 4.0 * (double)n * dl_ * (mask || block_ids || P == 0 ? (total + 1) / 2.0 : (P + (n + 1) / 2.0));
    if (tc_attn) {
      prof_begin();
      kern::attention_tc(aa, W.attn_scratch, W.attn_scratch_bytes, s);
      prof_end(PROF_ATTN, attn_bytes, attn_flops);
    } else {
      prof_begin();
      for (int64_t i0 = 0; i0 < n; i0 += nq) {
        aa.i0 = i0;
        aa.nq = std::min(nq, n - i0);
        kern::attention_simt(dtype_, aa, W.attn_scratch, s);
        if (i0 + nq < n) ++launches;
      }
      prof_end(PROF_ATTN, attn_bytes, attn_flops);
      aa.i0 = 0;
      aa.nq = -1;
    }
  };

  // Few-token regime (suffix prefill, decode): the GEMM/LayerNorm segments between two
  // attention launches run as one persistent chain kernel each (chain_tc.cu), so the
  // weight stream does not stop at GEMM boundaries.
  const bool chain_now = use_chain && tp_size_ == 1 && dtype_ == BF16 && w_->packed && !force_simt && !force_simt_gemm &&
                         kern::chain_ln_supported(d) && kern::chain_tc_supported(n, 3 * d, d) &&
                         kern::chain_tc_supported(n, 4 * d, d) && kern::chain_tc_supported(n, d, 4 * d) &&
                         (logit_rows == 0 || kern::chain_tc_supported(logit_rows, c.vocab_size, d));
  if (chain_now) {
    auto ln = [&](const float* src, int64_t rows) {
      kern::ChainStep st;
      st.kind = kern::CHAIN_LN;
      st.M = rows;
      st.ln_src = src;
      st.ln_dst = W.x;
      st.ln_d = d;
      return st;
    };
    auto mm = [&](const void* x, const void* w, int64_t M, int N, int K, const kern::Epilogue& e) {
      kern::ChainStep st;
      st.kind = kern::CHAIN_GEMM;
      st.M = M;
      st.x = x;
      st.w = w;
      st.N = N;
      st.K = K;
      st.e = e;
      return st;
    };
    // one request's attention joins the chain as its first phase (no launch, no prologue,
    // the next weights stream in as soon as each CTA's softmax is done)
    const bool fuse_attn = chain_attn && B == 1 && tc_attn && hd == 128 && !mask && !block_ids &&
                           kern::chain_attn_supported(n, P, H, hd);
    if (!kv_prefix_.empty() && (!fuse_attn || P < kv_prefix_rows_))
      throw Error(ErrorCode::ShapeMismatch, "zero-copy prefix set for a forward that cannot read it in place");
    // Layers per launch: with the attention as a chain phase and no per-layer event gating it
    // (slow-tier uploads), one launch spans up to chain_group layers -- no launch gap, prologue
    // or cold attention start between them; otherwise one launch per layer.
    const int group = fuse_attn && layer_ev.empty() ? std::max(1, chain_group) : 1;
    kern::ChainStep steps[kern::kChainMaxPhases];
    int k = 0, in_launch = 0;
    auto flush = [&] {
      if (k) chain(steps, k);
      k = 0;
      in_launch = 0;
    };
    steps[k++] = ln(W.h, n);
    steps[k++] = mm(W.x, w_->wqkv[0], n, 3 * d, d, qkv_epi(0));
    if (group == 1) flush();
    for (int l = 0; l < c.n_layers; ++l) {
      if (in_launch == group || k + 8 > kern::kChainMaxPhases) flush();
      if (fuse_attn) {
        if (l < static_cast<int>(layer_ev.size())) CK(cudaStreamWaitEvent(s, layer_ev[l], 0));
        kern::ChainStep st;
        st.kind = kern::CHAIN_ATTN;
        st.M = n;
        st.aq = W.q;
        st.ak = kv.k(l);
        st.av = kv.v(l);
        st.aout = W.attn;
        st.aP = P;
        st.aH = H;
        st.a_d = d;
        st.a_scratch = W.attn_scratch;
        st.a_scratch_bytes = W.attn_scratch_bytes;
        if (alibi) {
          st.a_alibi = w_->alibi;
          st.a_kpos = W.kvpos;
          st.a_qpos = W.pos;
        }
        if (!kv_prefix_.empty()) {  // cached modules read in place, then this request's rows
          st.a_layer = l;
          st.a_planes = 2 * c.n_layers;
          for (const KVBlock* b : kv_prefix_)
            st.a_seg[st.a_nseg++] = {b->data, b->cap, b->plane_bytes(), 0, b->rows};
          st.a_seg[st.a_nseg++] = {kv.data, kv.cap, kv.plane_bytes(), kv_prefix_rows_, P + n - kv_prefix_rows_};
          st.a_tail_vis = P - kv_prefix_rows_;
        }
        steps[k++] = st;
      } else {
        flush();
        attention(l);
      }
      if (ln_fold && d % 128 == 0) {
        // LayerNorm folded into the GEMMs around it (no LN phases, two fewer grid
        // barriers per layer): the residual phases (Wo, W2) also write bf16(h) and
        // per-tile row sums; the next GEMM runs on bf16(h) and corrects its accumulator,
        // LN(h) W^T = rstd (h W^T - mean * sum_k W)
        auto res = [&](const void* x, const void* w, int K) {
          kern::Epilogue e = eo;
          e.x_out = W.x;
          kern::ChainStep st = mm(x, w, n, d, K, e);
          st.stats_out = W.lnstats;
          st.stats_ld = static_cast<int>(n);
          return st;
        };
        auto cons = [&](const void* w, int64_t rows, int N, kern::Epilogue e, const float* wsum, int64_t row0) {
          e.ln_wsum = wsum;
          kern::ChainStep st = mm(W.x, w, rows, N, d, e);
          st.x = static_cast<const char*>(W.x) + row0 * d * static_cast<int64_t>(es);
          st.stats_in = W.lnstats;
          st.stats_tiles = d / 128;
          st.stats_ld = static_cast<int>(n);
          st.stats_row0 = static_cast<int>(row0);
          st.ln_dim = d;
          return st;
        };
        steps[k++] = res(W.attn, w_->wo[l], d);
        steps[k++] = cons(w_->w1[l], n, 4 * d, eg, w_->wsum_1[l], 0);
        steps[k++] = res(W.mid, w_->w2[l], 4 * d);
        if (l + 1 < c.n_layers)
          steps[k++] = cons(w_->wqkv[l + 1], n, 3 * d, qkv_epi(l + 1), w_->wsum_qkv[l + 1], 0);
        else if (logit_rows > 0 && !per_segment_logits)
          steps[k++] = cons(w_->unembed, logit_rows, c.vocab_size, ef, w_->wsum_un, n - logit_rows);
      } else {
        steps[k++] = mm(W.attn, w_->wo[l], n, d, d, eo);
        steps[k++] = ln(W.h, n);
        steps[k++] = mm(W.x, w_->w1[l], n, 4 * d, d, eg);
        steps[k++] = mm(W.mid, w_->w2[l], n, d, 4 * d, eo);
        if (l + 1 < c.n_layers) {
          steps[k++] = ln(W.h, n);
          steps[k++] = mm(W.x, w_->wqkv[l + 1], n, 3 * d, d, qkv_epi(l + 1));
        } else if (logit_rows > 0 && !per_segment_logits) {
          steps[k++] = ln(W.h + (n - logit_rows) * d, logit_rows);
          steps[k++] = mm(W.x, w_->unembed, logit_rows, c.vocab_size, d, ef);
        }
      }
      ++in_launch;
      if (group == 1) flush();
    }
    flush();
  } else {
    for (int l = 0; l < c.n_layers; ++l) {
      prof_begin();
      kern::layernorm(dtype_, W.h, n, d, W.x, s);
      prof_end(PROF_OTHER, (4.0 + es) * n * d, 0);
      kern::Epilogue e = qkv_epi(l);
      gemm(W.x, w_->wqkv[l], n, 3 * dl_, d, &e, w_->pk_qkv);
      attention(l);
      if (tp_size_ > 1) {
        gemm(W.attn, w_->wo[l], n, d, dl_, &epart, w_->pk_o);  // partial over this rank's heads
        tp_reduce_into_h();
      } else {
        gemm(W.attn, w_->wo[l], n, d, d, &eo, w_->pk_o);
      }
      prof_begin();
      kern::layernorm(dtype_, W.h, n, d, W.x, s);
      prof_end(PROF_OTHER, (4.0 + es) * n * d, 0);
      gemm(W.x, w_->w1[l], n, fl_, d, &eg, w_->pk_1);
      if (tp_size_ > 1) {
        gemm(W.mid, w_->w2[l], n, d, fl_, &epart, w_->pk_2);
        tp_reduce_into_h();
      } else {
        gemm(W.mid, w_->w2[l], n, d, 4 * d, &eo, w_->pk_2);
      }
    }
    if (logit_rows > 0 && !per_segment_logits) {
      const int64_t r0 = n - logit_rows;
      prof_begin();
      kern::layernorm(dtype_, W.h + r0 * d, logit_rows, d, W.x, s);
      prof_end(PROF_OTHER, (4.0 + es) * logit_rows * d, 0);
      unembed(logit_rows);
    }
  }
  if (logit_rows > 0 && per_segment_logits) {
    // last row of every request: gathered LayerNorm, then one unembed GEMM of B rows
    prof_begin();
    kern::layernorm_rows(dtype_, W.h, B > 1 ? W.lrows : nullptr, logit_rows, d, W.x, s, n - 1);
    prof_end(PROF_OTHER, (4.0 + es) * logit_rows * d, 0);
    unembed(logit_rows);
  }
  for (int b = 0; b < B; ++b) {
    KVBlock& kb = *items[b].kv;
    kb.rows += items[b].n;
    kb.positions.insert(kb.positions.end(), items[b].positions, items[b].positions + items[b].n);
  }
}

const float* Model::device_logits() const { return ws_->logits; }
int32_t* Model::device_argmax() const { return ws_->argmax; }

void Model::argmax_last(int64_t logit_rows) {
  prof_begin();
  kern::argmax_rows(ws_->logits, logit_rows, cfg_.vocab_size, ws_->argmax, stream_);
  prof_end(PROF_OTHER, 4.0 * logit_rows * cfg_.vocab_size, 0);
}

// ---------------------------------------------------------------------------
// Reference-shaped API
// ---------------------------------------------------------------------------
ForwardOutput Model::forward(const std::vector<int>& tokens, const std::vector<int64_t>& positions,
                             const KVBlock* past) {
  if (tokens.size() != positions.size())
    throw Error(ErrorCode::ShapeMismatch, "tokens/position_ids length mismatch");
  if (past && (past->n_layers != cfg_.n_layers || past->hidden != dl_ || past->dtype != dtype_))
    throw Error(ErrorCode::ShapeMismatch, "past KV shape mismatch");
  if (past)
    for (int64_t p : past->positions)
      if (p < 0 || p >= cfg_.max_position) throw Error(ErrorCode::PositionOutOfRange, "past position out of range");
  const int64_t n = static_cast<int64_t>(tokens.size());
  const int64_t P = past ? past->rows : 0;
  KVPtr kv = alloc_kv(P + n);
  if (past) {
    copy_rows(*past, *kv, 0);
    kv->rows = P;
    kv->positions = past->positions;
  }
  std::vector<int32_t> t32(tokens.begin(), tokens.end());
  run(t32.data(), positions.data(), n, *kv, nullptr, nullptr, n);
  ForwardOutput out;
  out.seq = n;
  out.vocab = cfg_.vocab_size;
  out.logits.resize(static_cast<size_t>(n) * cfg_.vocab_size);
  if (n) CK(cudaMemcpyAsync(out.logits.data(), ws_->logits, out.logits.size() * 4, cudaMemcpyDeviceToHost, stream_));
  out.new_kv = alloc_kv(n);
  if (n) {
    const size_t rb = kv->row_bytes();
    CK(cudaMemcpy2DAsync(out.new_kv->plane(0, 0), out.new_kv->plane_bytes(), kv->plane(0, 0) + P * rb,
                         kv->plane_bytes(), n * rb, 2 * cfg_.n_layers, cudaMemcpyDeviceToDevice, stream_));
  }
  out.new_kv->rows = n;
  out.new_kv->positions = positions;
  CK(cudaStreamSynchronize(stream_));
  return out;
}

ForwardOutput Model::forward_masked(const std::vector<int>& tokens, const std::vector<int64_t>& positions,
                                    const std::vector<uint8_t>& mask) {
  const int64_t n = static_cast<int64_t>(tokens.size());
  if (positions.size() != tokens.size()) throw Error(ErrorCode::ShapeMismatch, "tokens/position_ids length mismatch");
  if (static_cast<int64_t>(mask.size()) != n * n) throw Error(ErrorCode::ShapeMismatch, "mask must be [seq, seq]");
  KVPtr kv = alloc_kv(n);
  std::vector<int32_t> t32(tokens.begin(), tokens.end());
  run(t32.data(), positions.data(), n, *kv, mask.data(), nullptr, n);
  ForwardOutput out;
  out.seq = n;
  out.vocab = cfg_.vocab_size;
  out.logits.resize(static_cast<size_t>(n) * cfg_.vocab_size);
  if (n) CK(cudaMemcpyAsync(out.logits.data(), ws_->logits, out.logits.size() * 4, cudaMemcpyDeviceToHost, stream_));
  out.new_kv = kv;
  CK(cudaStreamSynchronize(stream_));
  return out;
}

std::vector<int> Model::generate(KVBlock& kv, int last_token, int64_t last_position, int n_steps) {
  std::vector<int> out;
  int32_t cur = last_token;
  int64_t pos = last_position;
  // Every step's token stays on the device (argmax -> the next step's embedding input), so the
  // host queues all steps without waiting for any: one device->host copy of the tokens at the
  // end instead of a round trip per token (reference generate, model.cpp:464-477: fixed count)
  int32_t* host = nullptr;
  int32_t* dev = nullptr;
  CK(cudaMallocHost(reinterpret_cast<void**>(&host), std::max(1, n_steps) * 4));
  CK(cudaMalloc(reinterpret_cast<void**>(&dev), std::max(1, n_steps) * 4));
  struct Reset {
    Model* m;
    int32_t *h, *d;
    ~Reset() {
      m->device_token_ = nullptr;
      cudaFreeHost(h);
      cudaFree(d);
    }
  } reset{this, host, dev};
  for (int s = 0; s < n_steps; ++s) {
    if (kv.rows + 1 > kv.cap) {  // grow: reference KVState::append semantics
      KVPtr bigger = alloc_kv(std::max<int64_t>(kv.cap * 2, kv.rows + n_steps - s));
      copy_rows(kv, *bigger, 0);
      std::swap(kv.data, bigger->data);
      std::swap(kv.cap, bigger->cap);
    }
    device_token_ = s > 0 ? dev + (s - 1) : nullptr;
    run(&cur, &pos, 1, kv, nullptr, nullptr, 1);  // (cur: the host value only for step 0)
    argmax_last(1);
    CK(cudaMemcpyAsync(dev + s, ws_->argmax, 4, cudaMemcpyDeviceToDevice, stream_));
    ++pos;
  }
  device_token_ = nullptr;
  if (n_steps > 0) {
    CK(cudaMemcpyAsync(host, dev, n_steps * 4, cudaMemcpyDeviceToHost, stream_));
    CK(cudaStreamSynchronize(stream_));
    out.assign(host, host + n_steps);
  }
  return out;
}

uint64_t Model::weight_checksum(const std::string& name) const {
  // FNV-1a over the fp32 tensor as generated (reference model.cpp:248-267).  The
  // generator is re-run into a scratch buffer so the check is independent of the
  // storage dtype (the bf16 model stores RNE of exactly these values).
  const int d = cfg_.hidden;
  size_t count = 0;
  float scale = 1.0f / std::sqrt(static_cast<float>(d));
  if (name == "embed") {
    count = static_cast<size_t>(cfg_.vocab_size) * d;
    scale = 0.1f;
  } else if (name == "unembed") {
    count = static_cast<size_t>(cfg_.vocab_size) * d;
  } else {
    for (int l = 0; l < cfg_.n_layers && !count; ++l)
      for (const char* t : {"wq", "wk", "wv", "wo", "w1", "w2"})
        if (name == tname(l, t)) {
          count = static_cast<size_t>(d) * d * ((t[1] == '1' || t[1] == '2') ? 4 : 1);
          if (t[1] == '2') scale = 1.0f / std::sqrt(static_cast<float>(4 * d));
        }
  }
  if (!count) throw Error(ErrorCode::Internal, "unknown tensor \"" + name + "\"");
  float* tmp = nullptr;
  CK(cudaMalloc(&tmp, count * 4));
  kern::init_uniform(F32, tmp, count, stream_seed(name, cfg_.seed), scale, stream_);
  std::vector<float> h(count);
  CK(cudaMemcpyAsync(h.data(), tmp, count * 4, cudaMemcpyDeviceToHost, stream_));
  CK(cudaStreamSynchronize(stream_));
  cudaFree(tmp);
  return fnv1a64(h.data(), count * 4);
}

int argmax_lowest(const float* logits, int n) {
  int best = 0;
  for (int i = 1; i < n; ++i)
    if (logits[i] > logits[best]) best = i;
  return best;
}

}  // namespace pcb::model

// extern "C" boundary (include/promptcache_b200.h): no exception crosses it.
#include <cuda_runtime.h>

#include <cstdlib>
#include <functional>
#include <cstring>
#include <memory>
#include <string>

#include "../../include/promptcache_b200.h"
#include "host/cache.hpp"
#include "host/engine.hpp"
#include "host/collective.hpp"
#include "host/cuda_check.hpp"
#include "host/layout.hpp"
#include "host/model.hpp"
#include "host/pml.hpp"
#include "json.hpp"
#include "kernels/kernels.cuh"

using namespace pcb;

struct pcb_schema {
  engine::Schema s;
  bool planned = false;  // an unexpanded schema (chat tags kept) has no layout plan
  std::string plan_error;
  int plan_code = 0;
  const engine::Schema& P() const {
    if (!planned) throw pcb::Error(static_cast<pcb::ErrorCode>(plan_code), plan_error);
    return s;
  }
};
struct pcb_prompt {
  pml::PromptDoc p;
};
struct pcb_model {
  std::unique_ptr<model::Model> m;
};
struct pcb_kv {
  model::KVPtr kv;
};
struct pcb_store {
  std::unique_ptr<cache::ModuleStore> s;
};
struct pcb_peer {
  std::shared_ptr<coll::PeerRegion> r;
};
struct pcb_response {
  engine::ServeResponse r;
};

namespace {
thread_local std::string g_msg;
thread_local int g_code = 0;

template <typename F>
int guard(F&& f) {
  try {
    f();
    g_code = 0;
    return PCB_OK;
  } catch (const Error& e) {
    g_msg = e.what();
    g_code = static_cast<int>(e.code()) + 1;
  } catch (const std::exception& e) {
    g_msg = std::string("Internal: ") + e.what();
    g_code = PCB_ERR_INTERNAL;
  } catch (...) {
    g_msg = "Internal: unknown exception";
    g_code = PCB_ERR_INTERNAL;
  }
  return g_code;
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

template <typename F>
char* guard_str(F&& f) {
  char* out = nullptr;
  guard([&] { out = dup(f()); });
  return out;
}

pcb_schema* make_schema(pml::SchemaDoc doc) {
  auto* b = new pcb_schema;
  try {
    b->s.plan = layout::plan_layout(doc);
    b->planned = true;
  } catch (const Error& e) {
    b->plan_error = e.what();
    b->plan_code = static_cast<int>(e.code());
  }
  b->s.doc = std::move(doc);
  return b;
}
}  // namespace

extern "C" {

const char* pcb_last_error(void) { return g_msg.c_str(); }
int pcb_last_error_code(void) { return g_code; }
void pcb_free(void* p) { std::free(p); }
const char* pcb_version(void) { return "promptcache_b200 0.1 (sm_100a)"; }

// ---- PML / layout ----
int pcb_schema_parse(const char* pml_text, int expand, pcb_schema** out) {
  return guard([&] {
    pml::SchemaDoc d = pml::parse_schema(pml_text);
    if (expand) d = pml::expand_chat_tags(d, pml::ChatTemplate::llama2());
    *out = make_schema(std::move(d));
  });
}
int pcb_schema_from_ast(const char* ast, pcb_schema** out) {
  return guard([&] { *out = make_schema(pml::schema_from_ast_json(ast)); });
}
void pcb_schema_destroy(pcb_schema* s) { delete s; }
char* pcb_schema_to_ast(const pcb_schema* s) { return guard_str([&] { return pml::schema_to_ast_json(s->s.doc); }); }
char* pcb_schema_serialize(const pcb_schema* s) { return guard_str([&] { return pml::serialize(s->s.doc); }); }
char* pcb_schema_plan_json(const pcb_schema* s) { return guard_str([&] { return s->P().plan.to_json(); }); }
int pcb_prompt_parse(const char* text, pcb_prompt** out) {
  return guard([&] { *out = new pcb_prompt{pml::parse_prompt(text)}; });
}
int pcb_prompt_from_ast(const char* ast, pcb_prompt** out) {
  return guard([&] { *out = new pcb_prompt{pml::prompt_from_ast_json(ast)}; });
}
void pcb_prompt_destroy(pcb_prompt* p) { delete p; }
char* pcb_prompt_to_ast(const pcb_prompt* p) { return guard_str([&] { return pml::prompt_to_ast_json(p->p); }); }
char* pcb_prompt_serialize(const pcb_prompt* p) { return guard_str([&] { return pml::serialize(p->p); }); }
char* pcb_validate(const pcb_prompt* p, const pcb_schema* s) {
  return guard_str([&] { return pml::validate_prompt(p->p, s->s.doc).to_json(); });
}
char* pcb_resolve(const pcb_prompt* p, const pcb_schema* s) {
  return guard_str([&] { return layout::resolve_prompt(p->p, s->P().plan).to_json(); });
}

// ---- config ----
char* pcb_config_canonical(const char* j) { return guard_str([&] { return model::ModelConfig::from_json(j).to_json(); }); }
int pcb_config_hash(const char* j, uint64_t* out) {
  return guard([&] { *out = model::ModelConfig::from_json(j).hash(); });
}
int64_t pcb_per_token_bytes(const char* j) {
  int64_t r = -1;
  guard([&] { r = cache::per_token_bytes(model::ModelConfig::from_json(j)); });
  return r;
}

// ---- model ----
int pcb_model_create(const char* cfg, int dtype, int device, pcb_model** out) {
  return guard([&] {
    *out = new pcb_model{std::make_unique<model::Model>(model::ModelConfig::from_json(cfg), dtype, device)};
  });
}
struct pcb_group {
  std::shared_ptr<coll::LocalGroup> g;
};
int pcb_nccl_unique_id(uint8_t* out) {
  return guard([&] { coll::nccl_unique_id(out); });
}
int pcb_group_create(int size, pcb_group** out) {
  return guard([&] {
    if (size < 1) throw Error(ErrorCode::InvalidConfig, "group size must be positive");
    *out = new pcb_group{std::make_shared<coll::LocalGroup>(size)};
  });
}
void pcb_group_destroy(pcb_group* g) { delete g; }
int pcb_peer_create(int tp_rank, int tp_size, int device, int64_t cap_floats, uint8_t* handle_out, pcb_peer** out) {
  return guard([&] {
    auto r = std::make_shared<coll::PeerRegion>(tp_rank, tp_size, device, static_cast<size_t>(cap_floats));
    r->handle(handle_out);
    *out = new pcb_peer{r};
  });
}
int pcb_peer_open(pcb_peer* p, const uint8_t* handles) {
  return guard([&] { p->r->open(handles); });
}
void pcb_peer_destroy(pcb_peer* p) { delete p; }
int pcb_model_create_tp_peer(const char* cfg, int dtype, pcb_peer* peer, pcb_model** out) {
  return guard([&] {
    auto& r = *peer->r;
    *out = new pcb_model{std::make_unique<model::Model>(model::ModelConfig::from_json(cfg), dtype, r.device, r.rank,
                                                         r.size, coll::make_peer(peer->r))};
  });
}
int pcb_model_create_tp(const char* cfg, int dtype, int device, int tp_rank, int tp_size, const uint8_t* nccl_id,
                        pcb_group* group, pcb_model** out) {
  return guard([&] {
    std::shared_ptr<coll::Collective> comm;
    if (tp_size > 1) {
      if (group) comm = coll::make_local(group->g, tp_rank);
      else if (nccl_id) comm = coll::make_nccl(nccl_id, tp_rank, tp_size, device);
      else throw Error(ErrorCode::InvalidConfig, "tensor parallel needs an NCCL id or a local group");
    }
    *out = new pcb_model{
        std::make_unique<model::Model>(model::ModelConfig::from_json(cfg), dtype, device, tp_rank, tp_size, comm)};
  });
}
void pcb_model_destroy(pcb_model* m) { delete m; }
int pcb_model_set_option(pcb_model* m, const char* key, int64_t v) {
  return guard([&] {
    if (std::strcmp(key, "force_simt") == 0) m->m->force_simt = v != 0;
    else if (std::strcmp(key, "force_simt_gemm") == 0) m->m->force_simt_gemm = v != 0;
    else if (std::strcmp(key, "force_simt_attn") == 0) m->m->force_simt_attn = v != 0;
    else if (std::strcmp(key, "profile") == 0) m->m->set_profiling(v != 0);
    else if (std::strcmp(key, "chain") == 0) m->m->use_chain = v != 0;
    else if (std::strcmp(key, "ln_fold") == 0) m->m->ln_fold = v != 0;
    else if (std::strcmp(key, "chain_attn") == 0) m->m->chain_attn = v != 0;
    else if (std::strcmp(key, "zero_copy") == 0) m->m->zero_copy = v != 0;
    else if (std::strcmp(key, "attn_pair") == 0) m->m->attn_pair = v;
    else if (std::strcmp(key, "chain_group") == 0) m->m->chain_group = v;
    else throw Error(ErrorCode::InvalidConfig, std::string("unknown option ") + key);
  });
}
int pcb_model_weight_checksum(pcb_model* m, const char* t, uint64_t* out) {
  return guard([&] { *out = m->m->weight_checksum(t); });
}
int pcb_model_forward(pcb_model* m, const int32_t* tokens, const int64_t* positions, int64_t n, const pcb_kv* past,
                      const uint8_t* mask, float* logits_out, pcb_kv** new_kv) {
  return guard([&] {
    std::vector<int> t(tokens, tokens + n);
    std::vector<int64_t> p(positions, positions + n);
    model::ForwardOutput o;
    if (mask) {
      if (past && past->kv->rows) throw Error(ErrorCode::ShapeMismatch, "masked forward takes no past KV");
      o = m->m->forward_masked(t, p, std::vector<uint8_t>(mask, mask + n * n));
    } else {
      o = m->m->forward(t, p, past ? past->kv.get() : nullptr);
    }
    if (logits_out) std::memcpy(logits_out, o.logits.data(), o.logits.size() * sizeof(float));
    if (new_kv) *new_kv = new pcb_kv{o.new_kv};
  });
}
int pcb_model_generate(pcb_model* m, pcb_kv* kv, int32_t last_token, int64_t last_pos, int32_t n_steps, int32_t* out) {
  return guard([&] {
    if (kv->kv.use_count() > 1) {  // shared with a store entry: generate on a private copy
      model::KVPtr c = m->m->alloc_kv(kv->kv->rows + n_steps);
      m->m->copy_rows(*kv->kv, *c, 0);
      c->rows = kv->kv->rows;
      c->positions = kv->kv->positions;
      kv->kv = c;
    }
    auto r = m->m->generate(*kv->kv, last_token, last_pos, n_steps);
    for (size_t i = 0; i < r.size(); ++i) out[i] = r[i];
  });
}
int64_t pcb_model_forward_tokens(const pcb_model* m) { return m->m->forward_tokens.load(); }
int64_t pcb_model_launches(const pcb_model* m) { return m->m->launches; }
char* pcb_model_profile_json(pcb_model* m) { return guard_str([&] { return m->m->profile_json(); }); }
int pcb_model_timer(pcb_model* m, int stop, double* ms_out) {
  return guard([&] {
    static thread_local cudaEvent_t a = nullptr, b = nullptr;
    if (!a) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
    }
    if (!stop) {
      if (cudaEventRecord(a, m->m->stream()) != cudaSuccess) throw Error(ErrorCode::CudaError, "event record");
      return;
    }
    cudaEventRecord(b, m->m->stream());
    cudaEventSynchronize(b);
    float ms = 0;
    if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) throw Error(ErrorCode::CudaError, "event elapsed");
    if (ms_out) *ms_out = ms;
  });
}
int pcb_model_sync(pcb_model* m) {
  return guard([&] {
    cudaError_t e = cudaStreamSynchronize(m->m->stream());
    if (e != cudaSuccess) throw Error(ErrorCode::CudaError, cudaGetErrorString(e));
  });
}

// ---- kernel microbenchmarks (tuning aid; random bf16 operands on the device) ----
int pcb_debug_gemm_probe(int64_t* shapes, unsigned long long* times, int max_launches, int* n_out) {
  return guard([&] { *n_out = kern::gemm_probe_dump(shapes, times, max_launches); });
}

int pcb_debug_chain_probe(unsigned long long* times, int max_launches, int* n_out, int* phases_out) {
  return guard([&] { *n_out = kern::chain_probe_dump(times, max_launches, phases_out); });
}

int pcb_debug_attn_tl(unsigned long long* out, int max_ctas, int* n_out) {
  return guard([&] { *n_out = kern::attn_tl_dump(out, max_ctas); });
}

int pcb_debug_kernel_bench(const char* which, int64_t a0, int64_t a1, int64_t a2, int iters, double* us_out) {
  return guard([&] {
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    std::vector<void*> bufs;
    auto alloc = [&](size_t bytes) {
      void* p = nullptr;
      if (cudaMalloc(&p, bytes) != cudaSuccess) throw Error(ErrorCode::CudaError, "bench alloc");
      bufs.push_back(p);
      return p;
    };
    std::function<void()> run;
    float* ws = static_cast<float*>(alloc(64ull << 20));
    int* ctr = static_cast<int*>(alloc(65536 * 4));
    cudaMemset(ctr, 0, 65536 * 4);
    if (std::strcmp(which, "gemm") == 0) {  // a0 = M tokens, a1 = N, a2 = K
      void* X = alloc(a0 * a2 * 2);
      void* W = alloc(a1 * a2 * 2);
      float* R = static_cast<float*>(alloc(a0 * a1 * 4));
      kern::init_uniform(kern::BF16, X, a0 * a2, 1, 1.0f, s);
      kern::init_uniform(kern::BF16, W, a1 * a2, 2, 0.02f, s);
      kern::Epilogue e;
      e.kind = std::getenv("PCB_GEMM_EPI_NONE") ? kern::EPI_NONE : kern::EPI_RESID;
      e.resid = R;
      run = [=] { kern::gemm_tc(X, W, a0, static_cast<int>(a1), static_cast<int>(a2), e, ws, 64ull << 20, ctr, s); };
    } else if (std::strcmp(which, "attn") == 0) {  // a0 = n queries, a1 = P past, a2 = heads (hd 128)
      const int H = static_cast<int>(a2), d = H * 128;
      const int64_t tot = a0 + a1;
      void* q = alloc(a0 * d * 2);
      void* k = alloc(tot * d * 2);
      void* v = alloc(tot * d * 2);
      void* o = alloc(a0 * d * 2);
      kern::init_uniform(kern::BF16, q, a0 * d, 3, 1.0f, s);
      kern::init_uniform(kern::BF16, k, tot * d, 4, 1.0f, s);
      kern::init_uniform(kern::BF16, v, tot * d, 5, 1.0f, s);
      kern::AttnArgs a;
      a.q = q;
      a.k = k;
      a.v = v;
      a.out = o;
      a.n = a0;
      a.P = a1;
      a.H = H;
      a.hd = 128;
      a.d = d;
      a.counters = ctr + 8192;
      run = [=] { kern::attention_tc(a, ws, 64ull << 20, s); };
    } else {
      throw Error(ErrorCode::InvalidConfig, "unknown kernel bench");
    }
    for (int i = 0; i < 3; ++i) run();
    cudaEventRecord(e0, s);
    for (int i = 0; i < iters; ++i) run();
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    *us_out = ms * 1000.0 / iters;
    cudaError_t err = cudaGetLastError();
    for (void* p : bufs) cudaFree(p);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    if (err != cudaSuccess) throw Error(ErrorCode::CudaError, cudaGetErrorString(err));
  });
}

// ---- KV ----
int64_t pcb_kv_rows(const pcb_kv* kv) { return kv->kv->rows; }
int pcb_kv_positions(const pcb_kv* kv, int64_t* out) {
  std::memcpy(out, kv->kv->positions.data(), kv->kv->positions.size() * 8);
  return PCB_OK;
}
int pcb_kv_read(const pcb_kv* kvh, int layer, int which, float* out) {
  return guard([&] {
    const model::KVBlock& kv = *kvh->kv;
    if (layer < 0 || layer >= kv.n_layers || which < 0 || which > 1) throw Error(ErrorCode::ShapeMismatch, "bad plane");
    const uint64_t cnt = static_cast<uint64_t>(kv.rows) * kv.hidden;
    if (!cnt) return;
    const void* src = kv.plane(layer, which);
    if (kv.dtype == model::F32) {
      if (cudaMemcpy(out, src, cnt * 4, kv.host ? cudaMemcpyHostToHost : cudaMemcpyDeviceToHost) != cudaSuccess)
        throw Error(ErrorCode::CudaError, "kv read");
      return;
    }
    void* stage = nullptr;
    float* f = nullptr;
    cudaMalloc(&stage, cnt * 2);
    cudaMalloc(&f, cnt * 4);
    cudaMemcpy(stage, src, cnt * 2, kv.host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice);
    kern::convert(kern::BF16, stage, kern::F32, f, cnt, nullptr);
    cudaError_t e = cudaMemcpy(out, f, cnt * 4, cudaMemcpyDeviceToHost);
    cudaFree(stage);
    cudaFree(f);
    if (e != cudaSuccess) throw Error(ErrorCode::CudaError, cudaGetErrorString(e));
  });
}
int pcb_kv_upload(pcb_model* m, const float* k, const float* v, const int64_t* pos, int64_t rows, pcb_kv** out) {
  return guard([&] {
    model::Model& mm = *m->m;
    CK(cudaSetDevice(mm.device()));
    if (rows < 0) throw Error(ErrorCode::ShapeMismatch, "negative row count");
    model::KVPtr kv = mm.alloc_kv(rows);
    const int L = mm.config().n_layers, d = mm.kv_width();
    const uint64_t cnt = static_cast<uint64_t>(rows) * d;
    DeviceBuffer f(cnt * 4);
    for (int l = 0; l < L && cnt; ++l)
      for (int w = 0; w < 2; ++w) {
        CK(cudaMemcpyAsync(f.get(), (w ? v : k) + l * cnt, cnt * 4, cudaMemcpyHostToDevice, mm.stream()));
        kern::convert(kern::F32, f.get(), mm.dtype(), kv->plane(l, w), cnt, mm.stream());
        CK(cudaGetLastError());
      }
    CK(cudaStreamSynchronize(mm.stream()));
    kv->rows = rows;
    kv->positions.assign(pos, pos + rows);
    *out = new pcb_kv{kv};
  });
}
int pcb_kv_concat(pcb_model* m, const pcb_kv* const* kvs, int n, pcb_kv** out) {
  return guard([&] {
    std::vector<cache::EntryPtr> es;
    for (int i = 0; i < n; ++i) {
      auto e = std::make_shared<cache::CacheEntry>();
      e->kv = kvs[i]->kv;
      e->token_len = kvs[i]->kv->rows;
      es.push_back(e);
    }
    *out = new pcb_kv{engine::concat_kv(*m->m, es)};
  });
}
void pcb_kv_destroy(pcb_kv* kv) { delete kv; }

// ---- store ----
static cache::Tier tier_of(int t) { return t == PCB_TIER_SLOW ? cache::Tier::Slow : cache::Tier::Fast; }
int pcb_store_create(pcb_model* m, pcb_store** out) {
  return guard([&] { *out = new pcb_store{std::make_unique<cache::ModuleStore>(*m->m)}; });
}
void pcb_store_destroy(pcb_store* s) { delete s; }
int pcb_store_set_capacity(pcb_store* s, int tier, int64_t bytes) {
  return guard([&] { s->s->set_capacity(tier_of(tier), bytes); });
}
int pcb_store_encode_module(pcb_store* s, const pcb_schema* sc, const char* name, int tier) {
  return guard([&] { s->s->insert(cache::encode_module(s->s->model(), sc->P().plan, name, tier_of(tier))); });
}
int pcb_store_encode_schema(pcb_store* s, const pcb_schema* sc, int tier, int* count) {
  return guard([&] {
    int c = cache::encode_schema(s->s->model(), sc->P().plan, *s->s, tier_of(tier));
    if (count) *count = c;
  });
}
int pcb_store_encode_scaffold(pcb_store* s, const pcb_schema* sc, const char* members_json, int tier) {
  return guard([&] {
    std::vector<std::string> members = nlohmann::json::parse(members_json);
    s->s->insert(cache::encode_scaffold(s->s->model(), sc->P().plan, members, tier_of(tier)));
  });
}
int pcb_store_lookup(pcb_store* s, const char* schema, const char* name, pcb_kv** out) {
  return guard([&] {
    cache::EntryPtr e = s->s->lookup(schema, name);
    *out = e ? new pcb_kv{e->kv} : nullptr;
  });
}
int pcb_store_put_kv(pcb_store* s, const pcb_schema* sc, const char* module, const pcb_kv* kv, int tier) {
  return guard([&] {
    if (!kv) throw Error(ErrorCode::ShapeMismatch, "null KV block");
    s->s->insert(cache::install_module(s->s->model(), sc->P().plan, module, kv->kv, tier_of(tier)));
  });
}
int64_t pcb_store_size(const pcb_store* s) { return static_cast<int64_t>(s->s->size()); }
char* pcb_store_stats_json(const pcb_store* s) { return guard_str([&] { return s->s->stats_json(); }); }
int pcb_store_save(const pcb_store* s, const char* path) { return guard([&] { s->s->save(path); }); }
int pcb_store_load(pcb_store* s, const char* path) { return guard([&] { s->s->load(path); }); }

// ---- engine ----
int pcb_serve(pcb_store* s, const pcb_schema* sc, const pcb_prompt* p, int max_new, int use_cache, int use_scaffolds,
              pcb_response** out) {
  return guard([&] {
    engine::ServeRequest req;
    req.prompt = p->p;
    req.max_new_tokens = max_new;
    req.use_cache = use_cache != 0;
    req.use_scaffolds = use_scaffolds != 0;
    *out = new pcb_response{engine::serve(req, sc->P(), *s->s)};
  });
}
int pcb_serve_batch(pcb_store* s, const pcb_schema* sc, const pcb_prompt* const* prompts, int n, int micro_batch,
                    pcb_response** out) {
  return guard([&] {
    std::vector<engine::ServeRequest> reqs(n);
    for (int i = 0; i < n; ++i) {
      reqs[i].prompt = prompts[i]->p;
      reqs[i].max_new_tokens = 1;
    }
    std::vector<engine::ServeResponse> r = engine::serve_batch(reqs, sc->P(), *s->s, micro_batch);
    for (int i = 0; i < n; ++i) out[i] = new pcb_response{std::move(r[i])};
  });
}
int pcb_oracle_serve(pcb_model* m, const pcb_schema* sc, const pcb_prompt* p, int max_new, pcb_response** out) {
  return guard([&] {
    engine::ServeRequest req;
    req.prompt = p->p;
    req.max_new_tokens = max_new;
    *out = new pcb_response{engine::oracle_serve(req, sc->P(), *m->m)};
  });
}
char* pcb_response_json(const pcb_response* r) { return guard_str([&] { return r->r.to_json(); }); }
int pcb_response_tokens(const pcb_response* r, int32_t* out, int cap) {
  int n = static_cast<int>(r->r.output_tokens.size());
  for (int i = 0; i < n && i < cap; ++i) out[i] = r->r.output_tokens[i];
  return n;
}
int pcb_response_first_logits(const pcb_response* r, float* out, int cap) {
  int n = static_cast<int>(r->r.first_token_logits.size());
  for (int i = 0; i < n && i < cap; ++i) out[i] = r->r.first_token_logits[i];
  return n;
}
void pcb_response_destroy(pcb_response* r) { delete r; }

}  // extern "C"

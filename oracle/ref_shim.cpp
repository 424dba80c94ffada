// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI shim over the UNMODIFIED reference library (pc::*), compiled from the
// sources where they lie under /root/reference/proj/core by oracle/Makefile
// into oracle/_ref/libpcref_<isa>.so.  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference leg load it, as the checker
// and as the reference CPU arm.  Nothing here re-implements reference logic:
// every entry point forwards to the reference function cited beside it.
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.hpp"  // /root/reference/proj/tests/common.hpp (random_case, random_ast)
#include "json.hpp"
#include "promptcache/bench.hpp"
#include "promptcache/cache.hpp"
#include "promptcache/engine.hpp"
#include "promptcache/layout.hpp"
#include "promptcache/model.hpp"
#include "promptcache/pml.hpp"

using nlohmann::json;
using namespace pc;

namespace {

thread_local std::string g_err;
thread_local int g_err_code = 0;

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    g_err_code = static_cast<int>(e.code()) + 1;
    return g_err_code;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_err_code = 1000;
    return g_err_code;
  }
}

// ---- AST <-> JSON (interchange format shared with the product's host layer) ----

json node_to_json(const pml::SchemaNode& n) {
  json j;
  switch (n.kind) {
    case pml::NodeKind::Text: j["k"] = "text"; j["t"] = n.text; return j;
    case pml::NodeKind::Module: j["k"] = "module"; j["name"] = n.name; j["anon"] = n.anonymous; break;
    case pml::NodeKind::Union: j["k"] = "union"; break;
    case pml::NodeKind::Param: j["k"] = "param"; j["name"] = n.name; j["len"] = n.param_len; return j;
    case pml::NodeKind::Chat: j["k"] = "chat"; j["role"] = n.role; break;
  }
  j["ch"] = json::array();
  for (auto& c : n.children) j["ch"].push_back(node_to_json(c));
  return j;
}

pml::SchemaNode node_from_json(const json& j) {
  pml::SchemaNode n;
  std::string k = j.at("k");
  if (k == "text") { n.kind = pml::NodeKind::Text; n.text = j.at("t"); return n; }
  if (k == "param") { n.kind = pml::NodeKind::Param; n.name = j.at("name"); n.param_len = j.at("len"); return n; }
  if (k == "module") { n.kind = pml::NodeKind::Module; n.name = j.at("name"); n.anonymous = j.value("anon", false); }
  else if (k == "union") n.kind = pml::NodeKind::Union;
  else if (k == "chat") { n.kind = pml::NodeKind::Chat; n.role = j.at("role"); }
  else throw Error(ErrorCode::Internal, "bad node kind " + k);
  for (auto& c : j.at("ch")) n.children.push_back(node_from_json(c));
  return n;
}

json schema_to_json(const pml::SchemaDoc& d) {
  json j;
  j["name"] = d.name;
  j["root"] = json::array();
  for (auto& n : d.root) j["root"].push_back(node_to_json(n));
  return j;
}

pml::SchemaDoc schema_from_json(const json& j) {
  pml::SchemaDoc d;
  d.name = j.at("name");
  for (auto& n : j.at("root")) d.root.push_back(node_from_json(n));
  return d;
}

json item_to_json(const pml::PromptItem& it) {
  json j;
  if (it.kind == pml::PromptItem::Kind::Text) { j["k"] = "text"; j["t"] = it.text; return j; }
  j["k"] = "import";
  j["name"] = it.import.name;
  j["args"] = json::array();
  for (auto& [k, v] : it.import.args) j["args"].push_back(json::array({k, v}));
  j["ch"] = json::array();
  for (auto& c : it.import.children) j["ch"].push_back(item_to_json(c));
  return j;
}

pml::PromptItem item_from_json(const json& j) {
  if (j.at("k") == "text") return pml::PromptItem::make_text(j.at("t"));
  pml::ModuleImport imp;
  imp.name = j.at("name");
  for (auto& a : j.at("args")) imp.args.emplace_back(a.at(0), a.at(1));
  for (auto& c : j.at("ch")) imp.children.push_back(item_from_json(c));
  return pml::PromptItem::make_import(std::move(imp));
}

json prompt_to_json(const pml::PromptDoc& d) {
  json j;
  j["schema"] = d.schema_name;
  j["items"] = json::array();
  for (auto& it : d.items) j["items"].push_back(item_to_json(it));
  return j;
}

pml::PromptDoc prompt_from_json(const json& j) {
  pml::PromptDoc d;
  d.schema_name = j.at("schema");
  for (auto& it : j.at("items")) d.items.push_back(item_from_json(it));
  return d;
}

json plan_to_json(const layout::LayoutPlan& p) {
  json j;
  j["schema"] = p.schema_name;
  j["total_len"] = p.total_len;
  j["order"] = p.order;
  j["entries"] = json::object();
  for (auto& [name, m] : p.entries) {
    json e;
    e["start"] = m.start_pos;
    e["len"] = m.token_len;
    e["own_tokens"] = m.own_tokens;
    e["own_positions"] = m.own_positions;
    e["parent"] = m.parent;
    e["order"] = m.order;
    e["anon"] = m.anonymous;
    e["union_group"] = m.union_group;
    e["params"] = json::array();
    for (auto& s : m.param_slots)
      e["params"].push_back({{"name", s.param_name}, {"start", s.slot_start}, {"len", s.slot_len}});
    j["entries"][name] = e;
  }
  j["unions"] = json::array();
  for (auto& g : p.union_groups)
    j["unions"].push_back({{"members", g.members}, {"start", g.start_pos}, {"len", g.group_len}});
  return j;
}

json seg_to_json(const layout::Segment& s) {
  return {{"tokens", s.tokens}, {"positions", s.position_ids}};
}

json resolved_to_json(const layout::ResolvedPrompt& r) {
  json j;
  j["cached_imports"] = r.cached_imports;
  j["suffix_start"] = r.suffix_start;
  j["uncached"] = json::array();
  for (auto& u : r.uncached) {
    if (u.is_arg)
      j["uncached"].push_back({{"arg", true}, {"module", u.arg.module}, {"param", u.arg.param},
                               {"seg", seg_to_json(u.arg.seg)}});
    else
      j["uncached"].push_back({{"arg", false}, {"seg", seg_to_json(u.free_text)}});
  }
  return j;
}

pml::SchemaDoc load_schema(const char* text, int is_ast) {
  if (is_ast) return schema_from_json(json::parse(text));
  return pml::expand_chat_tags(pml::parse_schema(text), pml::ChatTemplate::llama2());
}

pml::PromptDoc load_prompt(const char* text, int is_ast) {
  if (is_ast) return prompt_from_json(json::parse(text));
  return pml::parse_prompt(text);
}

struct KV {
  model::KVState s;
};

}  // namespace

extern "C" {

const char* pcref_last_error() { return g_err.c_str(); }
void pcref_free(void* p) { std::free(p); }

// ---- model (model.hpp:59-91) ----
void* pcref_model_create(const char* cfg_json) {
  model::Model* m = nullptr;
  if (guard([&] { m = new model::Model(model::ModelConfig::from_json(cfg_json)); })) return nullptr;
  return m;
}
void pcref_model_destroy(void* m) { delete static_cast<model::Model*>(m); }

int pcref_config_hash(const char* cfg_json, uint64_t* out) {
  return guard([&] { *out = model::ModelConfig::from_json(cfg_json).hash(); });
}
char* pcref_config_canonical(const char* cfg_json) {
  char* r = nullptr;
  guard([&] { r = dup(model::ModelConfig::from_json(cfg_json).to_json()); });
  return r;
}

int pcref_weight_checksum(void* m, const char* name, uint64_t* out) {
  return guard([&] { *out = static_cast<model::Model*>(m)->weight_checksum(name); });
}

// Model::forward (model.cpp:445-449) / forward_masked (451-455)
int pcref_forward(void* m, const int32_t* tokens, const int64_t* pos, int64_t n, void* past,
                  const uint8_t* mask, float* logits_out, void** new_kv_out) {
  return guard([&] {
    auto* mm = static_cast<model::Model*>(m);
    std::vector<int> t(tokens, tokens + n);
    std::vector<long> p(pos, pos + n);
    model::ForwardOutput o;
    if (mask) {
      std::vector<uint8_t> mk(mask, mask + n * n);
      o = mm->forward_masked(t, p, mk);
    } else {
      o = mm->forward(t, p, past ? &static_cast<KV*>(past)->s : nullptr);
    }
    if (logits_out) std::memcpy(logits_out, o.logits.data(), o.logits.size() * sizeof(float));
    if (new_kv_out) *new_kv_out = new KV{std::move(o.new_kv)};
  });
}

int pcref_generate(void* m, void* kv, int last_token, int64_t last_pos, int n_steps, int32_t* out) {
  return guard([&] {
    auto r = static_cast<model::Model*>(m)->generate(static_cast<KV*>(kv)->s, last_token, last_pos, n_steps);
    for (size_t i = 0; i < r.size(); ++i) out[i] = r[i];
  });
}

int64_t pcref_forward_tokens(void* m) { return static_cast<model::Model*>(m)->forward_tokens.load(); }

// ---- KV states (model.hpp:34-44) ----
void pcref_kv_destroy(void* kv) { delete static_cast<KV*>(kv); }
int64_t pcref_kv_rows(void* kv) { return static_cast<KV*>(kv)->s.seq_len(); }
int pcref_kv_positions(void* kv, int64_t* out) {
  auto& s = static_cast<KV*>(kv)->s;
  for (long i = 0; i < s.seq_len(); ++i) out[i] = s.position_ids[i];
  return 0;
}
int pcref_kv_layer(void* kv, int layer, int which, float* out) {
  auto& s = static_cast<KV*>(kv)->s;
  auto& v = which ? s.v[layer] : s.k[layer];
  std::memcpy(out, v.data(), v.size() * sizeof(float));
  return 0;
}
// Synthetic past rows for timing the reference at 7B shape.
void* pcref_kv_synthetic(int n_layers, int hidden, int64_t rows, uint64_t seed) {
  auto* kv = new KV;
  kv->s.n_layers = n_layers;
  kv->s.hidden = hidden;
  kv->s.k.resize(n_layers);
  kv->s.v.resize(n_layers);
  model::Pcg32 rng(seed);
  for (long r = 0; r < rows; ++r) kv->s.position_ids.push_back(r);
  for (int l = 0; l < n_layers; ++l) {
    kv->s.k[l].resize(rows * hidden);
    kv->s.v[l].resize(rows * hidden);
    for (auto& x : kv->s.k[l]) x = rng.symmetric(1.0f);
    for (auto& x : kv->s.v[l]) x = rng.symmetric(1.0f);
  }
  return kv;
}

// A KVState from caller arrays k/v [n_layers][rows][hidden] + positions (test fixtures:
// the same synthetic past is uploaded to the device model and handed to the reference).
void* pcref_kv_from_arrays(int n_layers, int hidden, int64_t rows, const float* k, const float* v,
                           const int64_t* pos) {
  auto* kv = new KV;
  kv->s.n_layers = n_layers;
  kv->s.hidden = hidden;
  kv->s.k.resize(n_layers);
  kv->s.v.resize(n_layers);
  for (long r = 0; r < rows; ++r) kv->s.position_ids.push_back(pos[r]);
  const size_t cnt = static_cast<size_t>(rows) * hidden;
  for (int l = 0; l < n_layers; ++l) {
    kv->s.k[l].assign(k + l * cnt, k + (l + 1) * cnt);
    kv->s.v[l].assign(v + l * cnt, v + (l + 1) * cnt);
  }
  return kv;
}

// engine::concat_kv (engine.cpp:174-185) over bare KV states wrapped as entries.
void* pcref_kv_concat(void** kvs, int n) {
  KV* out = nullptr;
  guard([&] {
    std::vector<cache::CacheEntry> entries(n);
    std::vector<const cache::CacheEntry*> ptrs;
    for (int i = 0; i < n; ++i) {
      entries[i].kv = static_cast<KV*>(kvs[i])->s;
      entries[i].token_len = entries[i].kv.seq_len();
      ptrs.push_back(&entries[i]);
    }
    out = new KV{engine::concat_kv(ptrs)};
  });
  return out;
}

// ---- PML (pml.hpp:142-155) ----
char* pcref_parse_schema(const char* text, int expand) {
  char* r = nullptr;
  guard([&] {
    auto d = pml::parse_schema(text);
    if (expand) d = pml::expand_chat_tags(d, pml::ChatTemplate::llama2());
    r = dup(schema_to_json(d).dump());
  });
  return r;
}
char* pcref_parse_prompt(const char* text) {
  char* r = nullptr;
  guard([&] { r = dup(prompt_to_json(pml::parse_prompt(text)).dump()); });
  return r;
}
char* pcref_serialize_schema(const char* ast) {
  char* r = nullptr;
  guard([&] { r = dup(pml::serialize(schema_from_json(json::parse(ast)))); });
  return r;
}
char* pcref_serialize_prompt(const char* ast) {
  char* r = nullptr;
  guard([&] { r = dup(pml::serialize(prompt_from_json(json::parse(ast)))); });
  return r;
}
char* pcref_validate(const char* prompt, int prompt_ast, const char* schema, int schema_ast) {
  char* r = nullptr;
  guard([&] {
    r = dup(pml::validate_prompt(load_prompt(prompt, prompt_ast), load_schema(schema, schema_ast)).to_json());
  });
  return r;
}

// ---- layout (layout.cpp:120-257) ----
char* pcref_plan(const char* schema, int is_ast) {
  char* r = nullptr;
  guard([&] { r = dup(plan_to_json(layout::plan_layout(load_schema(schema, is_ast))).dump()); });
  return r;
}
char* pcref_resolve(const char* schema, int schema_ast, const char* prompt, int prompt_ast) {
  char* r = nullptr;
  guard([&] {
    auto plan = layout::plan_layout(load_schema(schema, schema_ast));
    r = dup(resolved_to_json(layout::resolve_prompt(load_prompt(prompt, prompt_ast), plan)).dump());
  });
  return r;
}

// ---- test-fixture generators (tests/common.hpp:75-233; bench.cpp:22-31) ----
char* pcref_random_case(uint32_t seed) {
  auto rc = pctest::random_case(seed);
  json j;
  j["schema"] = schema_to_json(rc.schema);
  j["prompt"] = prompt_to_json(rc.prompt);
  return dup(j.dump());
}
char* pcref_random_ast(uint32_t seed) { return dup(schema_to_json(pctest::random_ast(seed)).dump()); }
char* pcref_synthetic_text(int64_t n, uint64_t seed) {
  static const char alphabet[] = "abcdefghijklmnopqrstuvwxyz ABCDEFGHIJKLMNOPQRSTUVWXYZ.,";
  model::Pcg32 rng(model::splitmix64(seed));
  std::string s;
  for (long i = 0; i < n; ++i) s.push_back(alphabet[rng.next() % (sizeof(alphabet) - 1)]);
  return dup(s);
}

// ---- cache / engine (cache.cpp:288-349; engine.cpp:187-334) ----
// Encodes one module (encode_module) and returns its KV as a handle.
void* pcref_encode_module(void* m, const char* schema, int is_ast, const char* name) {
  KV* out = nullptr;
  guard([&] {
    auto plan = layout::plan_layout(load_schema(schema, is_ast));
    out = new KV{cache::encode_module(*static_cast<model::Model*>(m), plan, name).kv};
  });
  return out;
}
void* pcref_encode_scaffold(void* m, const char* schema, int is_ast, const char* members_json) {
  KV* out = nullptr;
  guard([&] {
    auto plan = layout::plan_layout(load_schema(schema, is_ast));
    std::vector<std::string> members = json::parse(members_json);
    out = new KV{cache::encode_scaffold(*static_cast<model::Model*>(m), plan, members).kv};
  });
  return out;
}

// mode: 0 = serve (cached), 1 = serve baseline (use_cache=false), 2 = oracle_serve.
// scaffold_json: "" or a JSON list of members to encode as a scaffold (used with use_scaffolds).
char* pcref_serve(void* m, const char* schema, int schema_ast, const char* prompt, int prompt_ast,
                  int max_new, int mode, const char* scaffold_json, int tier_slow) {
  char* r = nullptr;
  guard([&] {
    auto& mm = *static_cast<model::Model*>(m);
    auto sd = load_schema(schema, schema_ast);
    auto plan = layout::plan_layout(sd);
    engine::ServeRequest req;
    req.prompt = load_prompt(prompt, prompt_ast);
    req.max_new_tokens = max_new;
    req.use_cache = mode != 1;
    engine::ServeResponse resp;
    if (mode == 2) {
      resp = engine::oracle_serve(req, sd, plan, mm);
    } else {
      cache::ModuleStore store(mm.config());
      cache::encode_schema(mm, plan, store, tier_slow ? cache::Tier::Slow : cache::Tier::Fast);
      if (scaffold_json && *scaffold_json) {
        std::vector<std::string> members = json::parse(scaffold_json);
        store.insert(cache::encode_scaffold(mm, plan, members));
        req.use_scaffolds = true;
      }
      resp = engine::serve(req, sd, plan, store, mm);
    }
    json j = json::parse(resp.to_json());
    j["first_token_logits"] = resp.first_token_logits;
    r = dup(j.dump());
  });
  return r;
}

// Times Model::forward of n suffix tokens over a `past` KV (the reference's cached
// prefill, engine.cpp:245-246) and engine::concat_kv of `past` (engine.cpp:236).
// Returns seconds via out params. Used by bench.py's reference arm.
int pcref_time_cached_step(void* m, void* past, int64_t n, int64_t first_pos, double* t_forward,
                           double* t_concat) {
  return guard([&] {
    auto& mm = *static_cast<model::Model*>(m);
    auto& ps = static_cast<KV*>(past)->s;
    std::vector<int> toks(n);
    std::vector<long> pos(n);
    for (long i = 0; i < n; ++i) { toks[i] = 'a' + static_cast<int>(i % 26); pos[i] = first_pos + i; }
    cache::CacheEntry e;
    e.kv = ps;
    e.token_len = ps.seq_len();
    auto t0 = std::chrono::steady_clock::now();
    model::KVState cat = engine::concat_kv({&e});
    auto t1 = std::chrono::steady_clock::now();
    auto o = mm.forward(toks, pos, &cat);
    auto t2 = std::chrono::steady_clock::now();
    *t_concat = std::chrono::duration<double>(t1 - t0).count();
    *t_forward = std::chrono::duration<double>(t2 - t1).count();
    if (o.logits.empty()) throw Error(ErrorCode::Internal, "no logits");
  });
}

// Store persistence (cache.cpp:178-271): encodes the schema (plus optional slow scaffold)
// and saves a PCST file; used to generate golden PCST fixtures.
int pcref_store_save(void* m, const char* schema, int is_ast, const char* scaffold_json,
                     const char* path) {
  return guard([&] {
    auto& mm = *static_cast<model::Model*>(m);
    auto plan = layout::plan_layout(load_schema(schema, is_ast));
    cache::ModuleStore store(mm.config());
    cache::encode_schema(mm, plan, store);
    if (scaffold_json && *scaffold_json) {
      std::vector<std::string> members = json::parse(scaffold_json);
      store.insert(cache::encode_scaffold(mm, plan, members, cache::Tier::Slow));
    }
    store.save(path);
  });
}

int64_t pcref_per_token_bytes(const char* cfg_json) {
  int64_t r = -1;
  guard([&] { r = cache::per_token_bytes(model::ModelConfig::from_json(cfg_json)); });
  return r;
}

}  // extern "C"

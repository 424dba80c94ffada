// Module store bookkeeping (reference cache.cpp:36-128 semantics) and module
// precompute on the device.  PCST persistence keeps the reference's byte format
// (cache.cpp:131-271) so stores written by either implementation load in both.
#include "cache.hpp"

#include <algorithm>
#include <cstring>
#include <fstream>
#include <set>

#include "../kernels/kernels.cuh"
#include "cuda_check.hpp"
#include "json.hpp"

namespace pcb::cache {

static std::string key_of(const std::string& schema, const std::string& name) { return schema + '\x1f' + name; }

int64_t per_token_bytes(const model::ModelConfig& c) {
  return 2LL * c.n_layers * c.hidden * c.bytes_per_element;
}
int64_t entry_bytes(const CacheEntry& e, const model::ModelConfig& c) { return e.token_len * per_token_bytes(c); }

std::string scaffold_id(const std::vector<std::string>& members) {
  std::vector<std::string> s = members;
  std::sort(s.begin(), s.end());
  std::string id = "scaffold:";
  for (size_t i = 0; i < s.size(); ++i) id += (i ? "+" : "") + s[i];
  return id;
}

void ModuleStore::evict_lru(Tier t, int64_t needed) {
  std::lock_guard<std::recursive_mutex> g(mu_);
  evict_locked(t, needed);
}

void ModuleStore::evict_locked(Tier t, int64_t needed) {
  const int64_t cap = capacity(t);
  if (cap < 0) return;
  while (used(t) + needed > cap) {
    auto victim = entries_.end();
    for (auto it = entries_.begin(); it != entries_.end(); ++it)
      if (it->second->tier == t && (victim == entries_.end() || it->second->last_used < victim->second->last_used))
        victim = it;
    if (victim == entries_.end())
      throw Error(ErrorCode::CapacityExceeded, "cannot free " + std::to_string(needed) + " bytes in tier");
    used(t) -= entry_bytes(*victim->second, model_->config());
    entries_.erase(victim);
  }
}

void ModuleStore::insert(CacheEntry e) {
  std::lock_guard<std::recursive_mutex> g(mu_);
  const int64_t bytes = entry_bytes(e, model_->config());
  const int64_t cap = capacity(e.tier);
  if (cap >= 0 && bytes > cap)
    throw Error(ErrorCode::CapacityExceeded,
                "entry of " + std::to_string(bytes) + " bytes exceeds tier capacity " + std::to_string(cap));
  const std::string key = key_of(e.schema, e.name);
  auto old = entries_.find(key);
  if (old != entries_.end()) {
    used(old->second->tier) -= entry_bytes(*old->second, model_->config());
    entries_.erase(old);
  }
  evict_locked(e.tier, bytes);
  e.created_at = ++clock_;
  e.last_used = e.created_at;
  used(e.tier) += bytes;
  entries_.emplace(key, std::make_shared<CacheEntry>(std::move(e)));
}

EntryPtr ModuleStore::lookup(const std::string& schema, const std::string& name) {
  std::lock_guard<std::recursive_mutex> g(mu_);
  auto it = entries_.find(key_of(schema, name));
  if (it == entries_.end()) {
    ++stats_.misses;
    return nullptr;
  }
  ++stats_.hits;
  it->second->last_used = ++clock_;
  return it->second;
}

EntryPtr ModuleStore::lookup_scaffold(const std::string& schema, const std::vector<std::string>& members) {
  std::lock_guard<std::recursive_mutex> g(mu_);
  auto it = entries_.find(key_of(schema, scaffold_id(members)));
  if (it == entries_.end()) return nullptr;
  ++stats_.hits;
  it->second->last_used = ++clock_;
  return it->second;
}

void ModuleStore::touch(const std::string& schema, const std::string& name) {
  std::lock_guard<std::recursive_mutex> g(mu_);
  auto it = entries_.find(key_of(schema, name));
  if (it != entries_.end()) it->second->last_used = ++clock_;
}

std::vector<std::shared_ptr<const CacheEntry>> ModuleStore::snapshot() const {
  std::lock_guard<std::recursive_mutex> g(mu_);
  std::vector<std::shared_ptr<const CacheEntry>> out;
  for (const auto& kv : entries_) out.push_back(kv.second);
  return out;
}

std::string ModuleStore::stats_json() const {
  std::lock_guard<std::recursive_mutex> g(mu_);
  nlohmann::json j;
  j["entries"] = entries_.size();
  j["bytes_used"] = {{"fast", stats_.bytes_fast}, {"slow", stats_.bytes_slow}};
  j["hits"] = stats_.hits;
  j["misses"] = stats_.misses;
  return j.dump();
}

// ---------------------------------------------------------------------------
// Precompute
// ---------------------------------------------------------------------------
static CacheEntry finish_entry(model::Model& m, const std::string& schema, const std::string& name,
                               model::KVPtr kv, std::vector<int> tokens, std::vector<layout::ParamSlot> slots,
                               Tier tier) {
  CacheEntry e;
  e.schema = schema;
  e.name = name;
  e.tokens = std::move(tokens);
  e.token_len = static_cast<int64_t>(e.tokens.size());
  e.param_slots = std::move(slots);
  e.tier = tier;
  e.kv = tier == Tier::Slow ? m.to_host(*kv) : kv;
  return e;
}

CacheEntry encode_module(model::Model& m, const layout::LayoutPlan& plan, const std::string& name, Tier tier) {
  const layout::ModuleLayout& ml = plan.at(name);
  const int64_t n = static_cast<int64_t>(ml.own_tokens.size());
  model::KVPtr kv = m.alloc_kv(n);
  std::vector<int32_t> t32(ml.own_tokens.begin(), ml.own_tokens.end());
  m.run(t32.data(), ml.own_positions.data(), n, *kv, nullptr, nullptr, /*logit_rows=*/0);
  return finish_entry(m, plan.schema_name, name, kv, ml.own_tokens, ml.param_slots, tier);
}

CacheEntry install_module(model::Model& m, const layout::LayoutPlan& plan, const std::string& name, model::KVPtr kv,
                          Tier tier) {
  auto it = plan.entries.find(name);
  if (it == plan.entries.end()) throw Error(ErrorCode::UnknownModule, "no module \"" + name + "\" in the schema");
  const layout::ModuleLayout& ml = it->second;
  if (!kv || kv->host || kv->n_layers != m.config().n_layers || kv->hidden != m.kv_width() || kv->dtype != m.dtype())
    throw Error(ErrorCode::ShapeMismatch, "install_module: KV block does not belong to this model");
  if (kv->rows != static_cast<int64_t>(ml.own_tokens.size()) || kv->positions != ml.own_positions)
    throw Error(ErrorCode::ShapeMismatch, "install_module: KV rows/positions differ from module \"" + name + "\"'s span");
  return finish_entry(m, plan.schema_name, name, std::move(kv), ml.own_tokens, ml.param_slots, tier);
}

int encode_schema(model::Model& m, const layout::LayoutPlan& plan, ModuleStore& store, Tier tier) {
  int count = 0;
  for (const std::string& name : plan.order) {
    store.insert(encode_module(m, plan, name, tier));
    ++count;
  }
  cudaStreamSynchronize(m.stream());
  return count;
}

CacheEntry encode_scaffold(model::Model& m, const layout::LayoutPlan& plan, const std::vector<std::string>& modules,
                           Tier tier) {
  std::vector<std::string> ordered = modules;
  std::sort(ordered.begin(), ordered.end(),
            [&](const std::string& a, const std::string& b) { return plan.at(a).order < plan.at(b).order; });
  std::vector<int> tokens;
  std::vector<int64_t> positions;
  std::vector<layout::ParamSlot> slots;
  std::set<int64_t> seen;
  for (const std::string& nm : ordered) {
    const layout::ModuleLayout& ml = plan.at(nm);
    tokens.insert(tokens.end(), ml.own_tokens.begin(), ml.own_tokens.end());
    for (int64_t p : ml.own_positions) {
      if (!seen.insert(p).second)
        throw Error(ErrorCode::PositionOverlap, "scaffold members overlap at position " + std::to_string(p));
      positions.push_back(p);
    }
    slots.insert(slots.end(), ml.param_slots.begin(), ml.param_slots.end());
  }
  const int64_t n = static_cast<int64_t>(tokens.size());
  model::KVPtr kv = m.alloc_kv(n);
  std::vector<int32_t> t32(tokens.begin(), tokens.end());
  m.run(t32.data(), positions.data(), n, *kv, nullptr, nullptr, 0);
  CacheEntry e = finish_entry(m, plan.schema_name, scaffold_id(modules), kv, tokens, slots, tier);
  e.scaffold = true;
  e.members = modules;
  std::sort(e.members.begin(), e.members.end());
  cudaStreamSynchronize(m.stream());
  return e;
}

// ---------------------------------------------------------------------------
// PCST v1: "PCST", u32 version, u64 config hash, u32 count, entries sorted by key.
// ---------------------------------------------------------------------------
namespace {
constexpr char kMagic[4] = {'P', 'C', 'S', 'T'};
constexpr uint32_t kVersion = 1;

struct Out {
  std::ofstream f;
  explicit Out(const std::string& p) : f(p, std::ios::binary) {
    if (!f) throw Error(ErrorCode::IoError, "cannot open \"" + p + "\" for write");
  }
  void raw(const void* p, size_t n) {
    f.write(static_cast<const char*>(p), static_cast<std::streamsize>(n));
    if (!f) throw Error(ErrorCode::IoError, "write failed");
  }
  template <typename T>
  void put(T v) { raw(&v, sizeof v); }
  void str(const std::string& s) {
    put<uint32_t>(static_cast<uint32_t>(s.size()));
    raw(s.data(), s.size());
  }
};

struct In {
  std::ifstream f;
  size_t off = 0;
  explicit In(const std::string& p) : f(p, std::ios::binary) {
    if (!f) throw Error(ErrorCode::IoError, "cannot open \"" + p + "\"");
  }
  void raw(void* p, size_t n) {
    f.read(static_cast<char*>(p), static_cast<std::streamsize>(n));
    if (static_cast<size_t>(f.gcount()) != n)
      throw Error(ErrorCode::IoError, "truncated store file at offset " + std::to_string(off));
    off += n;
  }
  template <typename T>
  T get() {
    T v;
    raw(&v, sizeof v);
    return v;
  }
  std::string str() {
    uint32_t n = get<uint32_t>();
    std::string s(n, '\0');
    if (n) raw(s.data(), n);
    return s;
  }
};
}  // namespace

// Header hash: the config hash (reference format, so files move between implementations);
// a tensor-parallel shard mixes its (rank, size) in, so a shard never loads into another
// rank's model (its K/V columns are a different head range).
static uint64_t file_hash(const model::Model& m) {
  uint64_t h = m.config().hash();
  if (m.tp_size() > 1)
    h ^= model::splitmix64((static_cast<uint64_t>(m.tp_rank()) << 32) | static_cast<uint32_t>(m.tp_size()));
  return h;
}

void ModuleStore::save(const std::string& path) const {
  model::Model& m = *model_;
  CK(cudaSetDevice(m.device()));
  Out w(path);
  w.raw(kMagic, 4);
  w.put<uint32_t>(kVersion);
  w.put<uint64_t>(file_hash(m));
  const auto all = snapshot();
  w.put<uint32_t>(static_cast<uint32_t>(all.size()));
  const int L = m.config().n_layers, d = m.kv_width();
  DeviceBuffer f32, stage;  // fp32 conversion target; device copy of a pinned-host plane
  std::vector<float> buf;
  for (const auto& ep : all) {  // std::map order = the reference's sorted-key order
    const CacheEntry& e = *ep;
    w.str(e.schema);
    w.str(e.name);
    w.put<uint8_t>(e.scaffold ? 1 : 0);
    w.put<uint32_t>(static_cast<uint32_t>(e.members.size()));
    for (auto& s : e.members) w.str(s);
    w.put<uint8_t>(e.tier == Tier::Slow ? 1 : 0);
    w.put<int64_t>(e.token_len);
    w.put<uint32_t>(static_cast<uint32_t>(e.tokens.size()));
    w.raw(e.tokens.data(), e.tokens.size() * sizeof(int));
    w.put<uint32_t>(static_cast<uint32_t>(e.param_slots.size()));
    for (auto& s : e.param_slots) {
      w.str(s.param_name);
      w.put<int64_t>(s.slot_start);
      w.put<int32_t>(s.slot_len);
    }
    w.put<uint32_t>(static_cast<uint32_t>(e.kv->positions.size()));
    for (int64_t p : e.kv->positions) w.put<int64_t>(p);
    w.put<uint32_t>(static_cast<uint32_t>(L));
    const uint64_t cnt = static_cast<uint64_t>(e.kv->rows) * d;
    buf.resize(cnt);
    if (cnt && f32.bytes() < cnt * 4) f32.reset(cnt * 4);
    if (cnt && e.kv->host && stage.bytes() < cnt * e.kv->elem()) stage.reset(cnt * e.kv->elem());
    for (int l = 0; l < L; ++l)
      for (int which = 0; which < 2; ++which) {
        if (cnt) {
          const void* src = e.kv->plane(l, which);
          if (e.kv->host) {
            CK(cudaMemcpyAsync(stage.get(), src, cnt * e.kv->elem(), cudaMemcpyHostToDevice, m.stream()));
            src = stage.get();
          }
          kern::convert(e.kv->dtype, src, kern::F32, f32.get(), cnt, m.stream());
          CK(cudaGetLastError());
          CK(cudaMemcpyAsync(buf.data(), f32.get(), cnt * 4, cudaMemcpyDeviceToHost, m.stream()));
          CK(cudaStreamSynchronize(m.stream()));
        }
        w.put<uint64_t>(cnt);
        w.raw(buf.data(), cnt * 4);
      }
  }
}

void ModuleStore::load(const std::string& path) {
  model::Model& m = *model_;
  CK(cudaSetDevice(m.device()));
  In r(path);
  char magic[4];
  r.raw(magic, 4);
  if (std::memcmp(magic, kMagic, 4) != 0) throw Error(ErrorCode::IoError, "\"" + path + "\" is not a module store file");
  uint32_t version = r.get<uint32_t>();
  if (version != kVersion)
    throw Error(ErrorCode::VersionMismatch,
                "store version " + std::to_string(version) + ", expected " + std::to_string(kVersion));
  if (r.get<uint64_t>() != file_hash(m))
    throw Error(ErrorCode::ConfigHashMismatch,
                m.tp_size() > 1 ? "store was built with a different model config or tensor-parallel shard"
                                : "store was built with a different model config");
  const int d = m.kv_width();
  uint32_t count = r.get<uint32_t>();
  std::vector<CacheEntry> loaded;
  DeviceBuffer f32;
  std::vector<float> buf;
  for (uint32_t i = 0; i < count; ++i) {
    CacheEntry e;
    e.schema = r.str();
    e.name = r.str();
    e.scaffold = r.get<uint8_t>() != 0;
    uint32_t nm = r.get<uint32_t>();
    for (uint32_t k = 0; k < nm; ++k) e.members.push_back(r.str());
    e.tier = r.get<uint8_t>() ? Tier::Slow : Tier::Fast;
    e.token_len = r.get<int64_t>();
    uint32_t nt = r.get<uint32_t>();
    e.tokens.resize(nt);
    if (nt) r.raw(e.tokens.data(), nt * sizeof(int));
    uint32_t ns = r.get<uint32_t>();
    for (uint32_t k = 0; k < ns; ++k) {
      layout::ParamSlot s;
      s.param_name = r.str();
      s.slot_start = r.get<int64_t>();
      s.slot_len = r.get<int32_t>();
      e.param_slots.push_back(std::move(s));
    }
    uint32_t np = r.get<uint32_t>();
    std::vector<int64_t> pos(np);
    for (uint32_t k = 0; k < np; ++k) pos[k] = r.get<int64_t>();
    uint32_t L = r.get<uint32_t>();
    if (static_cast<int>(L) != m.config().n_layers) throw Error(ErrorCode::ConfigHashMismatch, "layer count mismatch");
    model::KVPtr kv = m.alloc_kv(np);
    kv->rows = np;
    kv->positions = pos;
    const uint64_t want = static_cast<uint64_t>(np) * d;
    buf.resize(want);
    if (want && f32.bytes() < want * 4) f32.reset(want * 4);
    for (uint32_t l = 0; l < L; ++l)
      for (int which = 0; which < 2; ++which) {
        uint64_t cnt = r.get<uint64_t>();
        if (cnt != want) throw Error(ErrorCode::IoError, "bad KV plane size in store file");
        if (!cnt) continue;
        r.raw(buf.data(), cnt * 4);
        CK(cudaMemcpyAsync(f32.get(), buf.data(), cnt * 4, cudaMemcpyHostToDevice, m.stream()));
        kern::convert(kern::F32, f32.get(), kv->dtype, kv->plane(l, which), cnt, m.stream());
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(m.stream()));  // buf is reused by the next plane
      }
    e.kv = e.tier == Tier::Slow ? m.to_host(*kv) : kv;
    loaded.push_back(std::move(e));
  }
  std::lock_guard<std::recursive_mutex> g(mu_);
  for (auto& e : loaded) insert(std::move(e));
  stats_.hits = 0;
  stats_.misses = 0;
}

}  // namespace pcb::cache

// Cached serving on the device.  Control flow follows the reference's serve
// (engine.cpp:187-258), serve_baseline (128-170) and oracle_serve (260-334);
// the data path is: store blocks --(assembly kernel / H2D)--> request cache
// --(suffix prefill writes its K/V rows in place)--> last-row logits -> argmax.
#include "engine.hpp"

#include <chrono>
#include <cstring>
#include <map>
#include <algorithm>
#include <cstdio>
#include <set>

#include "../kernels/kernels.cuh"
#include "cuda_check.hpp"
#include "json.hpp"


namespace pcb::engine {

namespace {

using Clock = std::chrono::steady_clock;
double us_since(Clock::time_point t0) { return std::chrono::duration<double, std::micro>(Clock::now() - t0).count(); }

// Uncached tokens of one request (reference UncachedPass, engine.cpp:23-63).
struct UncachedPass {
  std::vector<int32_t> tokens;
  std::vector<int64_t> positions;
  std::map<int64_t, int64_t> arg_row_by_pos;
  std::set<int64_t> drop_positions;
  std::vector<int64_t> free_rows;
  int64_t prompt_token_count = 0;
};

UncachedPass build_uncached(const layout::ResolvedPrompt& r, const layout::LayoutPlan& plan, bool need_probe) {
  UncachedPass up;
  for (const auto& u : r.uncached) {
    for (size_t i = 0; i < u.seg.tokens.size(); ++i) {
      const int64_t row = static_cast<int64_t>(up.tokens.size());
      up.tokens.push_back(u.seg.tokens[i]);
      up.positions.push_back(u.seg.position_ids[i]);
      if (u.is_arg) up.arg_row_by_pos[u.seg.position_ids[i]] = row;
      else up.free_rows.push_back(row);
    }
    if (u.is_arg)
      for (const layout::ParamSlot& slot : plan.at(u.module).param_slots)
        if (slot.param_name == u.param)
          for (int64_t p = slot.slot_start + static_cast<int64_t>(u.seg.tokens.size());
               p < slot.slot_start + slot.slot_len; ++p)
            up.drop_positions.insert(p);
  }
  up.prompt_token_count = static_cast<int64_t>(up.tokens.size());
  if (need_probe && up.tokens.empty()) {
    up.free_rows.push_back(0);
    up.tokens.push_back(pml::tok::kBos);
    up.positions.push_back(r.suffix_start);
  }
  return up;
}

void require_valid(const pml::PromptDoc& p, const pml::SchemaDoc& s) {
  pml::ValidationReport rep = pml::validate_prompt(p, s);
  if (!rep.ok) {
    std::string codes;
    for (auto& i : rep.issues)
      if (i.severity == pml::Severity::Error) codes += (codes.empty() ? "" : ", ") + i.code;
    throw Error(ErrorCode::ValidationFailed, codes);
  }
}

// Descriptor tables for the assembly kernel (pinned host + device), grow-only.
struct AsmScratch {
  int cap = 0;
  kern::CopySeg* h_segs = nullptr;
  uint64_t* h_first = nullptr;
  kern::CopySeg* d_segs = nullptr;
  uint64_t* d_first = nullptr;
  int32_t* h_map = nullptr;
  int32_t* d_map = nullptr;
  int64_t map_cap = 0;
  int32_t* h_tok = nullptr;  // first token
  float* h_logits = nullptr;
  int64_t logit_cap = 0;
  cudaEvent_t ev[4] = {};
  // slow tier: pinned-host module blocks stream in on a side stream, one event per layer,
  // so the suffix prefill of layer l only waits for layer l's rows (engine.cpp:229-234)
  cudaStream_t side = nullptr;
  cudaEvent_t side_start = nullptr;
  std::vector<cudaEvent_t> layer_ev;
  struct SlowCopy {
    const model::KVBlock* src;
    model::KVBlock* dst;
    int64_t row;
  };
  std::vector<SlowCopy> slow;
  ~AsmScratch() {
    for (auto& e : layer_ev) cudaEventDestroy(e);
    if (side_start) cudaEventDestroy(side_start);
    if (side) cudaStreamDestroy(side);
    if (h_segs) cudaFreeHost(h_segs);
    if (h_first) cudaFreeHost(h_first);
    if (d_segs) cudaFree(d_segs);
    if (d_first) cudaFree(d_first);
    if (h_map) cudaFreeHost(h_map);
    if (d_map) cudaFree(d_map);
    if (h_tok) cudaFreeHost(h_tok);
    if (h_logits) cudaFreeHost(h_logits);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
  void ensure(int n_segs, int64_t map_rows, int64_t V) {
    if (!ev[0])
      for (auto& e : ev) CK(cudaEventCreate(&e));
    if (n_segs > cap) {
      int c = std::max(n_segs, 2 * cap);
      c = std::max(c, 256);
      kern::CopySeg* old = h_segs;
      h_segs = nullptr;
      if (old) {
        kern::CopySeg* fresh = nullptr;
        CK(cudaMallocHost(&fresh, c * sizeof(kern::CopySeg)));
        std::memcpy(fresh, old, cap * sizeof(kern::CopySeg));  // queued segments survive growth
        cudaFreeHost(old);
        h_segs = fresh;
      }
      if (h_first) cudaFreeHost(h_first);
      if (d_segs) cudaFree(d_segs);
      if (d_first) cudaFree(d_first);
      if (!h_segs) CK(cudaMallocHost(&h_segs, c * sizeof(kern::CopySeg)));
      CK(cudaMallocHost(&h_first, c * sizeof(uint64_t)));
      CK(cudaMalloc(&d_segs, c * sizeof(kern::CopySeg)));
      CK(cudaMalloc(&d_first, c * sizeof(uint64_t)));
      cap = c;
    }
    if (map_rows > map_cap) {
      int64_t c = std::max<int64_t>(map_rows, 1024);
      if (h_map) cudaFreeHost(h_map);
      if (d_map) cudaFree(d_map);
      CK(cudaMallocHost(&h_map, c * 4));
      CK(cudaMalloc(&d_map, c * 4));
      map_cap = c;
    }
    if (!h_tok) CK(cudaMallocHost(&h_tok, 4096 * 4));
    if (V > logit_cap) {
      if (h_logits) cudaFreeHost(h_logits);
      CK(cudaMallocHost(&h_logits, V * 4));
      logit_cap = V;
    }
  }
};

// serve_batch's two pipelined result slots (pinned logits / tokens, events)
struct BatchSlot {
  float* h_logits = nullptr;
  int32_t* h_tok = nullptr;
  size_t cap = 0;
  cudaEvent_t ev[3] = {};
  cudaEvent_t segs_used = nullptr;  // the assembly's segment list left host memory
  cudaEvent_t done = nullptr;       // logits and tokens are in this slot's host buffers
};
struct BatchSlots {
  BatchSlot s[2];
  ~BatchSlots() {
    for (BatchSlot& sl : s) {
      if (sl.done) cudaEventSynchronize(sl.done);
      if (sl.h_logits) cudaFreeHost(sl.h_logits);
      if (sl.h_tok) cudaFreeHost(sl.h_tok);
      for (auto& e : sl.ev)
        if (e) cudaEventDestroy(e);
      if (sl.segs_used) cudaEventDestroy(sl.segs_used);
      if (sl.done) cudaEventDestroy(sl.done);
    }
  }
};
BatchSlots& batch_slots_of(cache::ModuleStore& store) {
  if (!store.batch_slots) store.batch_slots = std::make_shared<BatchSlots>();
  return *static_cast<BatchSlots*>(store.batch_slots.get());
}

AsmScratch& scratch_of(cache::ModuleStore& store) {
  if (!store.assembly_scratch) store.assembly_scratch = std::make_shared<AsmScratch>();
  return *static_cast<AsmScratch*>(store.assembly_scratch.get());
}

// Position-disjointness check of concat_kv (engine.cpp:176-181).
// PositionOverlap unless the entries' position sets are pairwise disjoint (reference
// concat_kv, engine.cpp:179-181).  Module positions are normally increasing runs in
// disjoint ranges, which is checked in O(rows); anything else sorts every position.
void check_disjoint(const std::vector<cache::EntryPtr>& entries) {
  std::vector<std::pair<int64_t, int64_t>> ranges;
  bool runs = true;
  size_t total = 0;
  for (auto& e : entries) {
    const std::vector<int64_t>& p = e->kv->positions;
    total += p.size();
    if (p.empty()) continue;
    for (size_t i = 1; i < p.size() && runs; ++i) runs = p[i] > p[i - 1];
    ranges.emplace_back(p.front(), p.back());
  }
  if (runs) {
    std::sort(ranges.begin(), ranges.end());
    bool apart = true;
    for (size_t i = 1; i < ranges.size() && apart; ++i) apart = ranges[i].first > ranges[i - 1].second;
    if (apart) return;
  }
  std::vector<int64_t> all;
  all.reserve(total);
  for (auto& e : entries) all.insert(all.end(), e->kv->positions.begin(), e->kv->positions.end());
  std::sort(all.begin(), all.end());
  auto dup = std::adjacent_find(all.begin(), all.end());
  if (dup != all.end())
    throw Error(ErrorCode::PositionOverlap, "cache entries overlap at position " + std::to_string(*dup));
}

// Gathers the entries' KV rows into `dst` rows [0, sum) — one assembly-kernel
// launch for every device-resident (fast tier) block; slow-tier blocks are
// H2D copies issued on the same stream.  Returns #slow entries.
int append_segments(model::Model& m, const std::vector<cache::EntryPtr>& entries, model::KVBlock& dst, AsmScratch& sc,
                    int& n_segs) {
  const int L = m.config().n_layers;
  const size_t rb = dst.row_bytes();
  int slow = 0;
  sc.ensure(n_segs + static_cast<int>(entries.size()) * 2 * L, 0, 0);
  int64_t row = 0;
  for (auto& e : entries) {
    const model::KVBlock& b = *e->kv;
    if (b.rows) {
      if (b.host) {
        ++slow;
        sc.slow.push_back({&b, &dst, row});  // issued layer by layer on the side stream
      } else if (rb % 16 == 0) {
        for (int l = 0; l < L; ++l)
          for (int w = 0; w < 2; ++w)
            sc.h_segs[n_segs++] = kern::CopySeg{b.plane(l, w), dst.plane(l, w) + row * rb, b.rows * rb};
      } else {
        CK(cudaMemcpy2DAsync(dst.plane(0, 0) + row * rb, dst.plane_bytes(), b.plane(0, 0), b.plane_bytes(),
                             b.rows * rb, 2 * L, cudaMemcpyDeviceToDevice, m.stream()));
      }
    }
    dst.positions.insert(dst.positions.end(), b.positions.begin(), b.positions.end());
    row += b.rows;
  }
  dst.rows = row;
  return slow;
}

// Slow-tier rows: per layer, the K and V planes of every pinned-host block H2D on the
// side stream, then that layer's event; the model waits for layer l right before its
// attention (Model::set_layer_events), so the suffix GEMMs run under the upload.
void launch_slow(model::Model& m, AsmScratch& sc) {
  if (sc.slow.empty()) return;
  const int L = m.config().n_layers;
  if (!sc.side) {
    CK(cudaStreamCreateWithFlags(&sc.side, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&sc.side_start, cudaEventDisableTiming));
  }
  while (static_cast<int>(sc.layer_ev.size()) < L) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    sc.layer_ev.push_back(e);
  }
  CK(cudaEventRecord(sc.side_start, m.stream()));  // the destination cache is free
  CK(cudaStreamWaitEvent(sc.side, sc.side_start, 0));
  for (int l = 0; l < L; ++l) {
    for (const auto& c : sc.slow) {
      const size_t rb = c.dst->row_bytes();
      CK(cudaMemcpy2DAsync(c.dst->plane(l, 0) + c.row * rb, c.dst->plane_bytes(), c.src->plane(l, 0),
                           c.src->plane_bytes(), c.src->rows * rb, 2, cudaMemcpyHostToDevice, sc.side));
    }
    CK(cudaEventRecord(sc.layer_ev[l], sc.side));
  }
  m.set_layer_events(sc.layer_ev.data(), L);
  sc.slow.clear();
}

// One assembly-kernel launch for every queued device segment.
void launch_segments(model::Model& m, AsmScratch& sc, int n_segs) {
  if (n_segs) {
    const uint64_t chunks = kern::assemble_plan(sc.h_segs, n_segs, sc.h_first);
    CK(cudaMemcpyAsync(sc.d_segs, sc.h_segs, n_segs * sizeof(kern::CopySeg), cudaMemcpyHostToDevice, m.stream()));
    CK(cudaMemcpyAsync(sc.d_first, sc.h_first, n_segs * sizeof(uint64_t), cudaMemcpyHostToDevice, m.stream()));
    double bytes = 0;
    for (int i = 0; i < n_segs; ++i) bytes += 2.0 * sc.h_segs[i].bytes;  // read + write
    m.prof_begin();
    kern::assemble(sc.d_segs, sc.d_first, n_segs, chunks, m.stream());
    m.prof_end(model::Model::PROF_ASM, bytes, 0);
  }
}

// Gathers the entries' KV rows into `dst` rows [0, sum) with one assembly launch;
// returns #slow entries.
int assemble(model::Model& m, const std::vector<cache::EntryPtr>& entries, model::KVBlock& dst, AsmScratch& sc) {
  int n_segs = 0;
  const int slow = append_segments(m, entries, dst, sc, n_segs);
  launch_segments(m, sc, n_segs);
  launch_slow(m, sc);
  return slow;
}

model::KVBlock& arena_of(cache::ModuleStore& store, int64_t cap) {
  model::Model& m = store.model();
  if (!store.arena || store.arena->cap < cap) {
    store.arena.reset();
    store.arena = m.alloc_kv(std::max<int64_t>(cap, 64));
  }
  store.arena->rows = 0;
  store.arena->positions.clear();
  return *store.arena;
}

// Decode working cache (reference assemble_working, engine.cpp:78-97): cached
// rows with supplied <unk> slots replaced by argument rows (unfilled tails
// dropped), then free-text rows.  When nothing is replaced it IS the request
// cache, so no copy is made.
model::KVBlock* make_working(model::Model& m, model::KVBlock& work, int64_t n_cached, const UncachedPass& up,
                             int extra, AsmScratch& sc, model::KVPtr& holder) {
  if (up.arg_row_by_pos.empty() && up.drop_positions.empty()) return &work;
  std::vector<int32_t> map;
  std::vector<int64_t> pos;
  for (int64_t r = 0; r < n_cached; ++r) {
    const int64_t p = work.positions[r];
    auto a = up.arg_row_by_pos.find(p);
    if (a != up.arg_row_by_pos.end()) {
      map.push_back(static_cast<int32_t>(n_cached + a->second));
      pos.push_back(work.positions[n_cached + a->second]);
    } else if (!up.drop_positions.count(p)) {
      map.push_back(static_cast<int32_t>(r));
      pos.push_back(p);
    }
  }
  for (int64_t row : up.free_rows) {
    map.push_back(static_cast<int32_t>(n_cached + row));
    pos.push_back(work.positions[n_cached + row]);
  }
  const int64_t rows = static_cast<int64_t>(map.size());
  holder = m.alloc_kv(rows + extra);
  sc.ensure(0, rows, 0);
  std::memcpy(sc.h_map, map.data(), rows * 4);
  CK(cudaMemcpyAsync(sc.d_map, sc.h_map, rows * 4, cudaMemcpyHostToDevice, m.stream()));
  kern::gather_map(work.data, work.cap, holder->data, holder->cap, sc.d_map, rows,
                   static_cast<int64_t>(work.row_bytes()), 2 * m.config().n_layers, m.stream());
  holder->rows = rows;
  holder->positions = pos;
  return holder.get();
}

// Suffix forward + first token (reference finish_decode, engine.cpp:110-126).
void prefill_and_decode(ServeResponse& resp, model::Model& m, model::KVBlock& work, int64_t n_cached,
                        const UncachedPass& up, int64_t first_pos, int max_new, AsmScratch& sc, Clock::time_point t0,
                        cudaEvent_t ev_start) {
  const int V = m.config().vocab_size;
  const int64_t n = static_cast<int64_t>(up.tokens.size());
  m.run(up.tokens.data(), up.positions.data(), n, work, nullptr, nullptr, max_new > 0 ? 1 : 0);
  if (max_new > 0) {
    m.argmax_last(1);
    CK(cudaEventRecord(sc.ev[2], m.stream()));
    CK(cudaMemcpyAsync(sc.h_logits, m.device_logits(), V * 4, cudaMemcpyDeviceToHost, m.stream()));
    CK(cudaMemcpyAsync(sc.h_tok, m.device_argmax(), 4, cudaMemcpyDeviceToHost, m.stream()));
  } else {
    CK(cudaEventRecord(sc.ev[2], m.stream()));
  }
  CK(cudaStreamSynchronize(m.stream()));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, ev_start, sc.ev[2]));
  resp.timings.prefill_device_us = ms * 1000.0;
  resp.timings.uncached_prefill_us = ms * 1000.0;
  resp.timings.ttft_us = us_since(t0);
  if (max_new <= 0) return;
  resp.first_token_logits.assign(sc.h_logits, sc.h_logits + V);
  const int t1 = sc.h_tok[0];
  resp.output_tokens.push_back(t1);
  resp.timings.ttft_us = us_since(t0);
  if (max_new > 1) {
    auto td = Clock::now();
    model::KVPtr holder;
    model::KVBlock* wk = make_working(m, work, n_cached, up, max_new - 1, sc, holder);
    std::vector<int> rest = m.generate(*wk, t1, first_pos, max_new - 1);
    resp.output_tokens.insert(resp.output_tokens.end(), rest.begin(), rest.end());
    resp.timings.decode_us_per_token = us_since(td) / (max_new - 1);
  }
  resp.output_text = pml::tok::detokenize(resp.output_tokens);
}

ServeResponse serve_baseline(const ServeRequest& req, const layout::ResolvedPrompt& r, const layout::LayoutPlan& plan,
                             cache::ModuleStore& store, Clock::time_point t0) {
  model::Model& m = store.model();
  std::map<int64_t, int> by_pos;
  for (const std::string& name : r.cached_imports) {
    const layout::ModuleLayout& ml = plan.at(name);
    for (size_t i = 0; i < ml.own_tokens.size(); ++i) by_pos[ml.own_positions[i]] = ml.own_tokens[i];
  }
  UncachedPass full = build_uncached(r, plan, false);
  for (size_t i = 0; i < full.tokens.size(); ++i) by_pos[full.positions[i]] = full.tokens[i];
  for (int64_t p : full.drop_positions) by_pos.erase(p);
  UncachedPass up;  // the whole prompt, renumbered 0..n-1, every row free
  for (auto& [p, t] : by_pos) {
    up.free_rows.push_back(static_cast<int64_t>(up.tokens.size()));
    up.positions.push_back(static_cast<int64_t>(up.tokens.size()));
    up.tokens.push_back(t);
  }
  if (up.tokens.empty()) {
    up.tokens.push_back(pml::tok::kBos);
    up.positions.push_back(0);
    up.free_rows.push_back(0);
  }
  ServeResponse resp;
  resp.cache_report.uncached_token_count = static_cast<int64_t>(by_pos.size());
  const int64_t n = static_cast<int64_t>(up.tokens.size());
  AsmScratch& sc = scratch_of(store);
  sc.ensure(0, 0, m.config().vocab_size);
  model::KVBlock& work = arena_of(store, n + std::max(0, req.max_new_tokens - 1));
  CK(cudaEventRecord(sc.ev[1], m.stream()));
  prefill_and_decode(resp, m, work, 0, up, n, req.max_new_tokens, sc, t0, sc.ev[1]);
  return resp;
}

}  // namespace

model::KVPtr concat_kv(model::Model& m, const std::vector<cache::EntryPtr>& entries, int64_t extra_cap) {
  check_disjoint(entries);
  int64_t rows = 0;
  for (auto& e : entries) rows += e->kv->rows;
  model::KVPtr out = m.alloc_kv(rows + extra_cap);
  AsmScratch sc;
  assemble(m, entries, *out, sc);
  CK(cudaStreamSynchronize(m.stream()));
  if (sc.side) CK(cudaStreamSynchronize(sc.side));  // slow-tier rows landed; no forward consumes the events
  m.set_layer_events(nullptr, 0);
  return out;
}

namespace {
ServeResponse serve_unlocked(const ServeRequest& req, const Schema& schema, cache::ModuleStore& store) {
  auto t0 = Clock::now();
  model::Model& m = store.model();
  CK(cudaSetDevice(m.device()));
  require_valid(req.prompt, schema.doc);
  const layout::LayoutPlan& plan = schema.plan;
  layout::ResolvedPrompt resolved = layout::resolve_prompt(req.prompt, plan);
  if (!req.use_cache) return serve_baseline(req, resolved, plan, store, t0);

  ServeResponse resp;
  resp.timings.parse_us = us_since(t0);

  auto tl = Clock::now();
  std::vector<cache::EntryPtr> selected;  // pinned for the whole request
  if (req.use_scaffolds) {
    cache::EntryPtr sc = store.lookup_scaffold(schema.doc.name, resolved.cached_imports);
    if (sc) {
      selected.push_back(sc);
      resp.cache_report.used_scaffold = true;
      ++resp.cache_report.modules_hit;
    }
  }
  if (selected.empty()) {
    for (const std::string& name : resolved.cached_imports) {
      cache::EntryPtr e = store.lookup(schema.doc.name, name);
      const layout::ModuleLayout& ml = plan.at(name);
      const bool stale = e && (e->token_len != static_cast<int64_t>(ml.own_tokens.size()) ||
                               e->kv->positions != ml.own_positions);
      if (!e || stale) {
        ++resp.cache_report.modules_missed;
        store.insert(cache::encode_module(m, plan, name));
        e = store.lookup(schema.doc.name, name);
      } else {
        ++resp.cache_report.modules_hit;
      }
      selected.push_back(e);
    }
  }
  resp.timings.lookup_us = us_since(tl);

  check_disjoint(selected);
  int64_t n_cached = 0;
  for (auto& e : selected) {
    n_cached += e->kv->rows;
    resp.cache_report.cached_token_count += e->token_len;
  }
  UncachedPass up = build_uncached(resolved, plan, req.max_new_tokens > 0);
  resp.cache_report.uncached_token_count = up.prompt_token_count;

  AsmScratch& sc = scratch_of(store);
  sc.ensure(0, 0, m.config().vocab_size);
  const int64_t n = static_cast<int64_t>(up.tokens.size());
  model::KVBlock& work = arena_of(store, n_cached + n + std::max(0, req.max_new_tokens - 1));
  // Zero-copy assembly: when every forward of this request runs the chain's attention phase
  // (few suffix tokens, bf16) and no cached row is replaced for decoding, the modules' K/V
  // are read in place from the store and the request cache holds only the new rows -- the
  // assembly copy (2 x the cached bytes through HBM) disappears.  Otherwise concat_kv's copy.
  bool zc = m.zero_copy && !selected.empty() && static_cast<int>(selected.size()) < kern::ChainStep::kMaxSeg &&
            n > 0 && m.fused_attention_ok(n) && (req.max_new_tokens <= 1 || m.fused_attention_ok(1)) &&
            up.arg_row_by_pos.empty() && up.drop_positions.empty();
  for (auto& e : selected) zc = zc && !e->kv->host;
  struct PrefixGuard {
    model::Model& m;
    ~PrefixGuard() { m.clear_kv_prefix(); }
  } prefix_guard{m};
  CK(cudaEventRecord(sc.ev[0], m.stream()));
  int slow = 0;
  if (zc) {
    std::vector<const model::KVBlock*> blocks;
    for (auto& e : selected) {
      blocks.push_back(e->kv.get());
      work.positions.insert(work.positions.end(), e->kv->positions.begin(), e->kv->positions.end());
    }
    work.rows = n_cached;  // logical rows; [0, n_cached) live in the store blocks
    m.set_kv_prefix(blocks);
  } else {
    slow = assemble(m, selected, work, sc);
  }
  CK(cudaEventRecord(sc.ev[1], m.stream()));
  if (up.tokens.empty()) {
    // no forward consumes the slow tier's per-layer events: the side stream's uploads into
    // the arena must land before the next request reuses it, and the events are dropped
    if (slow) CK(cudaStreamWaitEvent(m.stream(), sc.layer_ev[m.config().n_layers - 1], 0));
    m.set_layer_events(nullptr, 0);
    CK(cudaStreamSynchronize(m.stream()));
    resp.timings.ttft_us = us_since(t0);
    return resp;
  }
  const int64_t first_pos = std::max(resolved.suffix_start, up.positions.back() + 1);
  prefill_and_decode(resp, m, work, n_cached, up, first_pos, req.max_new_tokens, sc, t0, sc.ev[1]);
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, sc.ev[0], sc.ev[1]));
  resp.timings.assemble_us = ms * 1000.0;
  resp.timings.copy_us = slow ? ms * 1000.0 : 0.0;
  return resp;
}
}  // namespace

ServeResponse serve(const ServeRequest& req, const Schema& schema, cache::ModuleStore& store) {
  std::lock_guard<std::mutex> g(store.serve_mutex());
  return serve_unlocked(req, schema, store);
}

std::vector<ServeResponse> serve_batch(const std::vector<ServeRequest>& reqs, const Schema& schema,
                                       cache::ModuleStore& store, int micro_batch) {
  std::lock_guard<std::mutex> g(store.serve_mutex());
  model::Model& m = store.model();
  CK(cudaSetDevice(m.device()));
  const int V = m.config().vocab_size;
  const layout::LayoutPlan& plan = schema.plan;
  micro_batch = std::max(1, std::min(micro_batch, 1024));
  std::vector<ServeResponse> out(reqs.size());
  struct Item {
    size_t idx;
    std::vector<cache::EntryPtr> sel;
    UncachedPass up;
    int64_t n_cached = 0;
  };
  struct Batch {
    Clock::time_point t0;
    std::vector<Item> items;
  };
  cudaEvent_t segs_busy = nullptr;  // the last launch's assembly segment list, until its H2D ran
  // host side of micro-batch [b0, b1): resolve, store lookups (misses encode), uncached passes
  auto prep = [&](size_t b0) {
    Batch bt;
    bt.t0 = Clock::now();
    const size_t b1 = std::min(reqs.size(), b0 + micro_batch);
    for (size_t i = b0; i < b1; ++i) {
      const ServeRequest& req = reqs[i];
      // decode past the first token, baselines, scaffolds and ALiBi models (per-request key
      // positions in the attention) take the single-request path
      if (!req.use_cache || req.use_scaffolds || req.max_new_tokens != 1 ||
          m.config().pos_encoding == model::PosEncoding::Alibi) {
        if (segs_busy) CK(cudaEventSynchronize(segs_busy));  // serve() reuses the segment list
        out[i] = serve_unlocked(req, schema, store);
        continue;
      }
      require_valid(req.prompt, schema.doc);
      layout::ResolvedPrompt resolved = layout::resolve_prompt(req.prompt, plan);
      Item it;
      it.idx = i;
      ServeResponse& resp = out[i];
      resp.timings.parse_us = us_since(bt.t0);
      for (const std::string& name : resolved.cached_imports) {
        cache::EntryPtr e = store.lookup(schema.doc.name, name);
        const layout::ModuleLayout& ml = plan.at(name);
        if (!e || e->token_len != static_cast<int64_t>(ml.own_tokens.size()) || e->kv->positions != ml.own_positions) {
          ++resp.cache_report.modules_missed;
          store.insert(cache::encode_module(m, plan, name));
          e = store.lookup(schema.doc.name, name);
        } else {
          ++resp.cache_report.modules_hit;
        }
        it.sel.push_back(e);
      }
      check_disjoint(it.sel);
      for (auto& e : it.sel) {
        it.n_cached += e->kv->rows;
        resp.cache_report.cached_token_count += e->token_len;
      }
      it.up = build_uncached(resolved, plan, true);
      resp.cache_report.uncached_token_count = it.up.prompt_token_count;
      bt.items.push_back(std::move(it));
    }
    return bt;
  };
  // Per-slot host buffers and events (store-owned, reused across calls: pinned allocations
  // and frees synchronise the device): micro-batch k+1 is launched (queued behind k on the
  // stream) before k's results are collected, so the device never waits for the host's
  // resolve/lookup of the next micro-batch (it did: ~20% idle per 32-request micro-batch).
  BatchSlots& bs = batch_slots_of(store);
  BatchSlot* slots = bs.s;
  AsmScratch& sc = scratch_of(store);
  sc.ensure(0, 0, V);
  auto launch = [&](Batch& bt, BatchSlot& sl) {
    const size_t B = bt.items.size();
    if (sl.cap < B) {
      if (sl.h_logits) cudaFreeHost(sl.h_logits);
      if (sl.h_tok) cudaFreeHost(sl.h_tok);
      CK(cudaMallocHost(&sl.h_logits, B * V * sizeof(float)));
      CK(cudaMallocHost(&sl.h_tok, B * sizeof(int32_t)));
      sl.cap = B;
    }
    if (!sl.ev[0]) {
      for (auto& e : sl.ev) CK(cudaEventCreate(&e));
      CK(cudaEventCreateWithFlags(&sl.segs_used, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    }
    // one request cache per item, equal capacity (run_batch addresses them by offset)
    int64_t cap = 0;
    for (auto& it : bt.items) cap = std::max<int64_t>(cap, it.n_cached + static_cast<int64_t>(it.up.tokens.size()));
    if (store.batch_arenas.size() < B || (!store.batch_arenas.empty() && store.batch_arenas[0]->cap < cap)) {
      // one allocation, request caches at a uniform stride (one batched attention launch)
      const int64_t c = std::max<int64_t>(cap, store.batch_arenas.empty() ? 64 : store.batch_arenas[0]->cap);
      const size_t nreq = std::max<size_t>(B, micro_batch);
      CK(cudaStreamSynchronize(m.stream()));  // the previous micro-batch still reads the old arenas
      store.batch_arenas.clear();
      store.batch_raw.reset();
      model::KVPtr probe = m.alloc_kv(0);
      const size_t req_bytes = static_cast<size_t>(c) * probe->row_bytes() * 2 * probe->n_layers;
      void* raw = nullptr;
      CK(cudaMalloc(&raw, req_bytes * nreq));
      store.batch_raw = std::shared_ptr<void>(raw, [](void* p) { cudaFree(p); });
      for (size_t k = 0; k < nreq; ++k) {
        auto v = std::make_shared<model::KVBlock>();
        v->dtype = probe->dtype;
        v->n_layers = probe->n_layers;
        v->hidden = probe->hidden;
        v->cap = c;
        v->view = true;
        v->data = static_cast<char*>(raw) + k * req_bytes;
        store.batch_arenas.push_back(v);
      }
    }
    if (segs_busy) CK(cudaEventSynchronize(segs_busy));  // sc's pinned segment list is reused
    // zero-copy micro-batch: every request's modules read in place by the batched attention
    // (device-resident blocks, <= 15 per request, <= 128 suffix tokens); else one assembly launch
    bool zc = B > 1 && m.batched_zero_copy_ok();
    for (auto& it : bt.items) {
      zc = zc && static_cast<int>(it.sel.size()) < kern::kAttnMaxSeg && it.up.tokens.size() <= 128;
      for (auto& e : it.sel) zc = zc && !e->kv->host;
    }
    CK(cudaEventRecord(sl.ev[0], m.stream()));
    int n_segs = 0;
    std::vector<model::Model::BatchItem> bi;
    std::vector<std::vector<const model::KVBlock*>> prefixes;
    for (size_t k = 0; k < B; ++k) {
      model::KVBlock& a = *store.batch_arenas[k];
      a.rows = 0;
      a.positions.clear();
      if (zc) {
        std::vector<const model::KVBlock*> blocks;
        for (auto& e : bt.items[k].sel) {
          blocks.push_back(e->kv.get());
          a.positions.insert(a.positions.end(), e->kv->positions.begin(), e->kv->positions.end());
          a.rows += e->kv->rows;  // logical rows: the blocks, read in place
        }
        prefixes.push_back(std::move(blocks));
      } else {
        append_segments(m, bt.items[k].sel, a, sc, n_segs);
      }
      bi.push_back({bt.items[k].up.tokens.data(), bt.items[k].up.positions.data(),
                    static_cast<int64_t>(bt.items[k].up.tokens.size()), &a});
    }
    launch_segments(m, sc, n_segs);
    CK(cudaEventRecord(sl.segs_used, m.stream()));
    segs_busy = sl.segs_used;
    launch_slow(m, sc);
    CK(cudaEventRecord(sl.ev[1], m.stream()));
    if (zc) {
      m.set_kv_prefix_batch(prefixes);
      try {
        m.run_batch(bi, true);
      } catch (...) {
        m.clear_kv_prefix();
        throw;
      }
      m.clear_kv_prefix();
    } else {
      m.run_batch(bi, true);
    }
    m.argmax_last(static_cast<int64_t>(B));
    CK(cudaEventRecord(sl.ev[2], m.stream()));
    CK(cudaMemcpyAsync(sl.h_logits, m.device_logits(), B * V * sizeof(float), cudaMemcpyDeviceToHost, m.stream()));
    CK(cudaMemcpyAsync(sl.h_tok, m.device_argmax(), B * sizeof(int32_t), cudaMemcpyDeviceToHost, m.stream()));
    CK(cudaEventRecord(sl.done, m.stream()));
  };
  auto finish = [&](Batch& bt, BatchSlot& sl) {
    CK(cudaEventSynchronize(sl.done));
    float ms_asm = 0, ms_pre = 0;
    CK(cudaEventElapsedTime(&ms_asm, sl.ev[0], sl.ev[1]));
    CK(cudaEventElapsedTime(&ms_pre, sl.ev[1], sl.ev[2]));
    const double ttft = us_since(bt.t0);
    for (size_t k = 0; k < bt.items.size(); ++k) {
      ServeResponse& resp = out[bt.items[k].idx];
      resp.first_token_logits.assign(sl.h_logits + k * V, sl.h_logits + (k + 1) * V);
      resp.output_tokens.push_back(sl.h_tok[k]);
      resp.output_text = pml::tok::detokenize(resp.output_tokens);
      resp.timings.assemble_us = ms_asm * 1000.0;
      resp.timings.prefill_device_us = ms_pre * 1000.0;
      resp.timings.uncached_prefill_us = ms_pre * 1000.0;
      resp.timings.ttft_us = ttft;
    }
  };
  static const bool trace = std::getenv("PCB_BATCH_TRACE") != nullptr;  // host-side phase times (debug)
  auto stamp = [&](const char* what, Clock::time_point t) {
    if (trace) std::fprintf(stderr, "[serve_batch] %-8s %9.3f ms\n", what, us_since(t) / 1e3);
  };
  try {
    auto t = Clock::now();
    Batch cur = prep(0);
    stamp("prep", t);
    int slot = 0;
    t = Clock::now();
    if (!cur.items.empty()) launch(cur, slots[slot]);
    stamp("launch", t);
    for (size_t b0 = 0; b0 < reqs.size(); b0 += micro_batch) {
      Batch nxt;
      if (b0 + micro_batch < reqs.size()) {
        t = Clock::now();
        nxt = prep(b0 + micro_batch);
        stamp("prep", t);
        t = Clock::now();
        if (!nxt.items.empty()) launch(nxt, slots[slot ^ 1]);
        stamp("launch", t);
      }
      t = Clock::now();
      if (!cur.items.empty()) finish(cur, slots[slot]);
      stamp("finish", t);
      cur = std::move(nxt);
      slot ^= 1;
    }
  } catch (...) {
    cudaStreamSynchronize(m.stream());
    throw;
  }
  return out;
}

ServeResponse oracle_serve(const ServeRequest& req, const Schema& schema, model::Model& m) {
  auto t0 = Clock::now();
  CK(cudaSetDevice(m.device()));
  require_valid(req.prompt, schema.doc);
  const layout::LayoutPlan& plan = schema.plan;
  layout::ResolvedPrompt resolved = layout::resolve_prompt(req.prompt, plan);
  ServeResponse resp;
  resp.timings.parse_us = us_since(t0);
  std::vector<int32_t> tokens;
  std::vector<int64_t> positions;
  std::vector<int32_t> block;
  int bid = 0;
  for (const std::string& name : resolved.cached_imports) {
    const layout::ModuleLayout& ml = plan.at(name);
    for (size_t i = 0; i < ml.own_tokens.size(); ++i) {
      tokens.push_back(ml.own_tokens[i]);
      positions.push_back(ml.own_positions[i]);
      block.push_back(bid);
    }
    ++bid;
    resp.cache_report.cached_token_count += static_cast<int64_t>(ml.own_tokens.size());
  }
  const int64_t n_cached = static_cast<int64_t>(tokens.size());
  UncachedPass up = build_uncached(resolved, plan, req.max_new_tokens > 0);
  resp.cache_report.uncached_token_count = up.prompt_token_count;
  for (size_t i = 0; i < up.tokens.size(); ++i) {
    tokens.push_back(up.tokens[i]);
    positions.push_back(up.positions[i]);
    block.push_back(-1);
  }
  const int64_t n = static_cast<int64_t>(tokens.size());
  if (n == 0) {
    resp.timings.ttft_us = us_since(t0);
    return resp;
  }
  // Block-causal mask as block ids: a cached row sees earlier rows of its own
  // module; an uncached row sees every earlier row (engine.cpp:300-307).
  model::KVPtr kv = m.alloc_kv(n + std::max(0, req.max_new_tokens - 1));
  AsmScratch sc;
  sc.ensure(0, 0, m.config().vocab_size);
  CK(cudaEventRecord(sc.ev[1], m.stream()));
  if (up.tokens.empty()) {
    m.run(tokens.data(), positions.data(), n, *kv, nullptr, block.data(), 0);
    CK(cudaStreamSynchronize(m.stream()));
    resp.timings.ttft_us = us_since(t0);
    return resp;
  }
  // prefill_and_decode runs the uncached rows; here the whole sequence is the
  // "suffix" of an empty cache with block ids, so run it directly.
  const int V = m.config().vocab_size;
  m.run(tokens.data(), positions.data(), n, *kv, nullptr, block.data(), 1);
  m.argmax_last(1);
  CK(cudaMemcpyAsync(sc.h_logits, m.device_logits(), V * 4, cudaMemcpyDeviceToHost, m.stream()));
  CK(cudaMemcpyAsync(sc.h_tok, m.device_argmax(), 4, cudaMemcpyDeviceToHost, m.stream()));
  CK(cudaStreamSynchronize(m.stream()));
  resp.timings.uncached_prefill_us = us_since(t0);
  resp.timings.ttft_us = us_since(t0);
  const int max_new = req.max_new_tokens;
  if (max_new <= 0) return resp;
  resp.first_token_logits.assign(sc.h_logits, sc.h_logits + V);
  const int t1 = sc.h_tok[0];
  resp.output_tokens.push_back(t1);
  const int64_t first_pos = std::max(resolved.suffix_start, positions.back() + 1);
  if (max_new > 1) {
    auto td = Clock::now();
    model::KVPtr holder;
    model::KVBlock* wk = make_working(m, *kv, n_cached, up, max_new - 1, sc, holder);
    std::vector<int> rest = m.generate(*wk, t1, first_pos, max_new - 1);
    resp.output_tokens.insert(resp.output_tokens.end(), rest.begin(), rest.end());
    resp.timings.decode_us_per_token = us_since(td) / (max_new - 1);
  }
  resp.output_text = pml::tok::detokenize(resp.output_tokens);
  return resp;
}

std::string ServeResponse::to_json() const {
  nlohmann::json j;
  j["output_tokens"] = output_tokens;
  j["output_text"] = output_text;
  j["timings"] = {{"parse_us", timings.parse_us},
                  {"lookup_us", timings.lookup_us},
                  {"copy_us", timings.copy_us},
                  {"uncached_prefill_us", timings.uncached_prefill_us},
                  {"ttft_us", timings.ttft_us},
                  {"decode_us_per_token", timings.decode_us_per_token},
                  {"assemble_us", timings.assemble_us},
                  {"prefill_device_us", timings.prefill_device_us}};
  j["cache_report"] = {{"modules_hit", cache_report.modules_hit},
                       {"modules_missed", cache_report.modules_missed},
                       {"cached_token_count", cache_report.cached_token_count},
                       {"uncached_token_count", cache_report.uncached_token_count},
                       {"used_scaffold", cache_report.used_scaffold}};
  return j.dump(-1, ' ', false, nlohmann::json::error_handler_t::replace);
}

}  // namespace pcb::engine

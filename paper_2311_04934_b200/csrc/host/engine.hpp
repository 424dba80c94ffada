// Cached serving: the north-star hot path (reference engine.hpp:13-62 /
// engine.cpp:187-258).  serve() resolves the prompt on the host, pins the
// selected store entries, gathers their KV blocks into the request cache with
// one assembly kernel launch (slow-tier blocks stream in by cudaMemcpyAsync),
// prefills the uncached suffix on top, and returns the first token.
#pragma once

#include <string>
#include <vector>

#include "cache.hpp"
#include "layout.hpp"
#include "model.hpp"
#include "pml.hpp"

namespace pcb::engine {

struct ServeRequest {
  pml::PromptDoc prompt;
  int max_new_tokens = 16;
  bool use_cache = true;
  bool use_scaffolds = false;
};

struct Timings {
  double parse_us = 0, lookup_us = 0, copy_us = 0, uncached_prefill_us = 0, ttft_us = 0, decode_us_per_token = 0;
  // device-side (CUDA events) breakdown of the TTFT window, new here
  double assemble_us = 0, prefill_device_us = 0;
};

struct CacheReport {
  int modules_hit = 0, modules_missed = 0;
  int64_t cached_token_count = 0, uncached_token_count = 0;
  bool used_scaffold = false;
};

struct ServeResponse {
  std::vector<int> output_tokens;
  std::string output_text;
  std::vector<float> first_token_logits;
  Timings timings;
  CacheReport cache_report;
  std::string to_json() const;
};

// Schema bundle: parsed (+chat-expanded) schema with its layout plan.
struct Schema {
  pml::SchemaDoc doc;
  layout::LayoutPlan plan;
};

// Pure concatenation (reference engine.cpp:174-185): duplicate positions raise
// PositionOverlap; returns a device block with rows in entry order.
model::KVPtr concat_kv(model::Model& m, const std::vector<cache::EntryPtr>& entries, int64_t extra_cap = 0);

ServeResponse serve(const ServeRequest& req, const Schema& schema, cache::ModuleStore& store);
// Micro-batched cached serving: requests of one micro-batch are
// assembled with one kernel launch into their own caches and their uncached suffixes
// prefilled together (one weight stream per micro-batch, attention per request).
// First token only (max_new_tokens == 1); other requests take serve().
std::vector<ServeResponse> serve_batch(const std::vector<ServeRequest>& reqs, const Schema& schema,
                                       cache::ModuleStore& store, int micro_batch);
// Block-causal exact reference (engine.cpp:260-334) run on the device.
ServeResponse oracle_serve(const ServeRequest& req, const Schema& schema, model::Model& m);

}  // namespace pcb::engine

// Schema layout and prompt resolution: the bit-exact integer contract of the
// hot path (module selection, gather offsets, position IDs).  Types mirror the
// reference's layout.hpp:11-94; implementation written from scratch.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "pml.hpp"

namespace pcb::layout {

struct ParamSlot {
  std::string param_name;
  int64_t slot_start = 0;
  int slot_len = 0;
  bool operator==(const ParamSlot&) const = default;
};

struct ModuleLayout {
  std::string module;
  int64_t start_pos = 0;
  int64_t token_len = 0;  // full span incl. nested children
  std::vector<int> own_tokens;
  std::vector<int64_t> own_positions;
  std::vector<ParamSlot> param_slots;
  std::string parent;
  int order = 0;
  bool anonymous = false;
  int union_group = -1;
};

struct UnionGroup {
  std::vector<std::string> members;
  int64_t start_pos = 0;
  int64_t group_len = 0;
};

struct LayoutPlan {
  std::string schema_name;
  std::map<std::string, ModuleLayout> entries;
  std::vector<std::string> order;
  std::vector<UnionGroup> union_groups;
  int64_t total_len = 0;

  const ModuleLayout& at(const std::string& name) const;
  std::string to_json() const;  // full plan (all fields), for parity fixtures
};

struct Segment {
  std::vector<int> tokens;
  std::vector<int64_t> position_ids;
};

struct ResolvedPrompt {
  std::vector<std::string> cached_imports;  // schema order
  struct Uncached {
    bool is_arg = false;
    std::string module, param;  // is_arg
    Segment seg;
  };
  std::vector<Uncached> uncached;  // prompt document order
  int64_t suffix_start = 0;

  std::string to_json() const;
};

LayoutPlan plan_layout(const pml::SchemaDoc& schema);
ResolvedPrompt resolve_prompt(const pml::PromptDoc& prompt, const LayoutPlan& plan);

}  // namespace pcb::layout

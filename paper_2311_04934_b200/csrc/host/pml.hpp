// PML schema / prompt ASTs and their operations — the API surface the north star
// keeps.  Semantics follow the reference's pml.hpp:15-155 (parse, serialize,
// validate, chat-tag expansion); the implementation here is written from scratch.
#pragma once

#include <map>
#include <string>
#include <utility>
#include <vector>

#include "errors.hpp"

namespace pcb::pml {

enum class NodeKind { Text, Module, Union, Param, Chat };

struct SchemaNode {
  NodeKind kind = NodeKind::Text;
  std::string text;        // Text
  std::string name;        // Module, Param
  int param_len = 0;       // Param
  std::string role;        // Chat
  bool anonymous = false;  // Module wrapping bare schema-level text
  std::vector<SchemaNode> children;

  bool operator==(const SchemaNode&) const = default;
};

struct SchemaDoc {
  std::string name;
  std::vector<SchemaNode> root;
  bool operator==(const SchemaDoc&) const = default;
};

struct PromptItem;

struct ModuleImport {
  std::string name;
  std::vector<std::pair<std::string, std::string>> args;  // document order
  std::vector<PromptItem> children;                       // nested imports
  bool operator==(const ModuleImport&) const;
};

struct PromptItem {
  enum class Kind { Import, Text };
  Kind kind = Kind::Text;
  ModuleImport import;
  std::string text;
  bool operator==(const PromptItem&) const;
};

struct PromptDoc {
  std::string schema_name;
  std::vector<PromptItem> items;
  bool operator==(const PromptDoc&) const = default;
};

enum class Severity { Warning, Error };

struct Issue {
  Severity severity = Severity::Error;
  std::string code;
  std::string message;
};

struct ValidationReport {
  bool ok = true;
  std::vector<Issue> issues;
  void add(Severity s, const std::string& code, const std::string& msg);
  std::string to_json() const;
};

struct ChatTemplate {
  struct Role {
    std::string prefix, suffix;
  };
  std::map<std::string, Role> roles;
  static ChatTemplate llama2();
};

SchemaDoc parse_schema(const std::string& text);
PromptDoc parse_prompt(const std::string& text);
std::string serialize(const SchemaDoc& doc);
std::string serialize(const PromptDoc& doc);
ValidationReport validate_prompt(const PromptDoc& prompt, const SchemaDoc& schema);
SchemaDoc expand_chat_tags(const SchemaDoc& doc, const ChatTemplate& tpl);

// AST interchange (JSON), shared with the test harness so in-memory ASTs built by
// the reference's fixture generators can be replayed bit-for-bit.
std::string schema_to_ast_json(const SchemaDoc& doc);
SchemaDoc schema_from_ast_json(const std::string& json);
std::string prompt_to_ast_json(const PromptDoc& doc);
PromptDoc prompt_from_ast_json(const std::string& json);

// Byte tokenizer (reference tokenizer.cpp:5-20): token = byte, specials 256..258.
namespace tok {
constexpr int kUnk = 256, kBos = 257, kEos = 258, kMinVocab = 259;
std::vector<int> tokenize(const std::string& s);
std::string detokenize(const std::vector<int>& t);
}  // namespace tok

}  // namespace pcb::pml

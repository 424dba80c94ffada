// PML front end (SPEC.md [MODULE] pml): schema / prompt parsing, serialization,
// validation and chat-template expansion.  Host-only.
//
// Design: a pull lexer turns the source into markup events (open / self-close / close
// tag, text run) and each document is built in one pass by a stack of frames -- there
// is no intermediate element tree.  Lexical errors abort at once; structural errors
// found while building are deferred until the source has lexed to its end, so a
// malformed document reports SyntaxError before any semantic code (MissingSchemaAttr),
// the precedence of the reference's read-then-build parser (pml.cpp:424-473).
// Validation issue codes and messages are the reference's output contract
// (pml.cpp:556-701) and are reproduced exactly; parse-error wording is our own.
#include "pml.hpp"

#include <algorithm>
#include <cctype>
#include <optional>
#include <set>

#include "json.hpp"

namespace pcb {

const char* error_code_name(ErrorCode c) {
  static const char* names[] = {
      "SyntaxError",       "MissingSchemaAttr",  "UnknownRole",     "TokenizerFailure",
      "FREE_TEXT_OVERFLOW", "ARG_TOO_LONG",      "InvalidConfig",   "PositionOutOfRange",
      "ShapeMismatch",     "UnknownModule",      "CapacityExceeded", "IoError",
      "VersionMismatch",   "ConfigHashMismatch", "ValidationFailed", "PositionOverlap",
      "UnknownCall",       "RecursionDetected",  "DuplicateName",   "InvalidProgram",
      "Internal",          "CudaError"};
  int i = static_cast<int>(c);
  return (i >= 0 && i < static_cast<int>(sizeof(names) / sizeof(names[0]))) ? names[i] : "Unknown";
}

namespace pml {

namespace tok {
std::vector<int> tokenize(const std::string& s) {
  std::vector<int> t;
  t.reserve(s.size());
  for (unsigned char c : s) t.push_back(c);
  return t;
}
std::string detokenize(const std::vector<int>& t) {
  std::string s;
  for (int x : t)
    if (x >= 0 && x < 256) s.push_back(static_cast<char>(x));
  return s;
}
}  // namespace tok

bool ModuleImport::operator==(const ModuleImport& o) const {
  return name == o.name && args == o.args && children == o.children;
}
bool PromptItem::operator==(const PromptItem& o) const {
  return kind == o.kind && (kind == Kind::Text ? text == o.text : import == o.import);
}

namespace {

using Attrs = std::vector<std::pair<std::string, std::string>>;

// ---------------------------------------------------------------------------
// Lexer: XML subset -- elements, quoted attributes, self-closing tags, text with the
// entities lt/gt/amp/quot/apos.  No comments, processing instructions, CDATA or
// numeric character references.
// ---------------------------------------------------------------------------
struct Event {
  enum Kind { Open, SelfClose, Close, Text, End } kind = End;
  std::string name;  // tag name (Open / SelfClose / Close)
  Attrs attrs;       // Open / SelfClose
  std::string text;  // Text: entities decoded, never empty
  int line = 1, col = 1;
};

class Lexer {
 public:
  explicit Lexer(const std::string& src) : src_(src) {}

  Event next() {
    Event ev;
    ev.line = line_;
    ev.col = col_;
    if (at_end()) return ev;
    if (peek() != '<') {
      ev.kind = Event::Text;
      while (!at_end() && peek() != '<') {
        if (peek() == '&') {
          advance();
          ev.text += entity();
        } else {
          ev.text.push_back(advance());
        }
      }
      return ev;
    }
    advance();  // '<'
    if (!at_end() && peek() == '/') {
      advance();
      ev.kind = Event::Close;
      ev.name = ident("closing tag");
      skip_space();
      expect('>', "'>' to end </" + ev.name);
      return ev;
    }
    ev.name = ident("tag");
    for (;;) {
      skip_space();
      if (at_end()) fail("tag <" + ev.name + "> is not terminated");
      if (peek() == '>') {
        advance();
        ev.kind = Event::Open;
        return ev;
      }
      if (peek() == '/') {
        advance();
        expect('>', "'>' right after '/' in <" + ev.name + "/>");
        ev.kind = Event::SelfClose;
        return ev;
      }
      std::string key = ident("attribute");
      skip_space();
      expect('=', "'=' after attribute " + key);
      skip_space();
      std::string value = quoted();
      if (std::any_of(ev.attrs.begin(), ev.attrs.end(), [&](const auto& a) { return a.first == key; }))
        fail("attribute " + key + " given twice on <" + ev.name + ">");
      ev.attrs.emplace_back(std::move(key), std::move(value));
    }
  }

  void skip_space() {
    while (!at_end() && std::isspace(static_cast<unsigned char>(peek()))) advance();
  }
  bool at_end() const { return pos_ >= src_.size(); }
  [[noreturn]] void fail(const std::string& what) const { throw Error(ErrorCode::SyntaxError, what, line_, col_); }

 private:
  char peek() const { return src_[pos_]; }
  char advance() {
    const char c = src_[pos_++];
    if (c == '\n') {
      ++line_;
      col_ = 1;
    } else {
      ++col_;
    }
    return c;
  }
  void expect(char c, const std::string& what) {
    if (at_end() || peek() != c) fail("expected " + what);
    advance();
  }
  std::string ident(const char* what) {
    auto head = [](char c) { return std::isalpha(static_cast<unsigned char>(c)) || c == '_'; };
    auto tail = [](char c) { return std::isalnum(static_cast<unsigned char>(c)) || c == '_' || c == '-' || c == '.'; };
    if (at_end() || !head(peek())) fail(std::string("expected a ") + what + " name");
    std::string s;
    while (!at_end() && tail(peek())) s.push_back(advance());
    return s;
  }
  // after '&': a named entity up to ';' (names of more than 8 characters are rejected)
  std::string entity() {
    std::string nm;
    while (!at_end() && peek() != ';' && nm.size() < 8) nm.push_back(advance());
    if (at_end() || peek() != ';') fail("entity &" + nm + " is not terminated by ';'");
    advance();
    if (nm == "lt") return "<";
    if (nm == "gt") return ">";
    if (nm == "amp") return "&";
    if (nm == "quot") return "\"";
    if (nm == "apos") return "'";
    fail("unsupported entity &" + nm + ";");
  }
  std::string quoted() {
    if (at_end() || (peek() != '"' && peek() != '\'')) fail("attribute value must be quoted");
    const char q = advance();
    std::string v;
    for (;;) {
      if (at_end()) fail("attribute value runs to the end of input");
      const char c = peek();
      if (c == q) break;
      if (c == '<') fail("'<' inside an attribute value");
      if (c == '&') {
        advance();
        v += entity();
      } else {
        v.push_back(advance());
      }
    }
    advance();
    return v;
  }

  const std::string& src_;
  size_t pos_ = 0;
  int line_ = 1, col_ = 1;
};

bool is_space_only(const std::string& s) {
  return std::all_of(s.begin(), s.end(), [](unsigned char c) { return std::isspace(c) != 0; });
}

std::string trim(const std::string& s) {
  size_t b = 0, e = s.size();
  while (b < e && std::isspace(static_cast<unsigned char>(s[b]))) ++b;
  while (e > b && std::isspace(static_cast<unsigned char>(s[e - 1]))) --e;
  return s.substr(b, e - b);
}

std::optional<std::string> attr_of(const Attrs& a, const char* key) {
  for (const auto& kv : a)
    if (kv.first == key) return kv.second;
  return std::nullopt;
}

bool is_chat_role(const std::string& t) { return t == "system" || t == "user" || t == "assistant"; }

bool is_reserved(const std::string& t) {
  return t == "schema" || t == "module" || t == "union" || t == "param" || t == "prompt" || is_chat_role(t);
}

SchemaNode make_text(std::string t) {
  SchemaNode n;
  n.kind = NodeKind::Text;
  n.text = std::move(t);
  return n;
}

// Param.len: decimal int with optional leading blanks and sign, nothing after the
// digits (what std::stoi accepts when it consumes the whole string); 0 = not an int.
int decimal_len(const std::string& s) {
  size_t i = 0;
  while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  int sign = 1;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) sign = s[i++] == '-' ? -1 : 1;
  if (i == s.size()) return 0;
  long long v = 0;
  for (; i < s.size(); ++i) {
    if (!std::isdigit(static_cast<unsigned char>(s[i]))) return 0;
    v = v * 10 + (s[i] - '0');
    if (v > 2147483648LL) return 0;
  }
  v *= sign;
  return (v > 2147483647LL || v < -2147483648LL) ? 0 : static_cast<int>(v);
}

// The first structural error in document order, raised once the source lexed cleanly.
struct Deferred {
  std::optional<Error> first;
  void note(const std::string& msg, int line, int col) {
    if (!first) first.emplace(ErrorCode::SyntaxError, msg, line, col);
  }
  void raise() const {
    if (first) throw *first;
  }
};

// Lexes a whole document: `on_root` gets the root's start tag, `body` every event
// strictly inside the root.  Tag balance and "nothing after the root" are checked here.
template <typename Body>
Event scan_document(const std::string& text, Body&& body) {
  Lexer lx(text);
  lx.skip_space();
  if (lx.at_end()) lx.fail("document has no root element");
  Event root = lx.next();
  if (root.kind != Event::Open && root.kind != Event::SelfClose) lx.fail("document must start with its root element");
  if (root.kind == Event::Open) {
    std::vector<std::string> open{root.name};
    for (;;) {
      Event ev = lx.next();
      if (ev.kind == Event::End) lx.fail("<" + open.back() + "> is never closed");
      if (ev.kind == Event::Close) {
        if (ev.name != open.back()) lx.fail("</" + ev.name + "> does not close <" + open.back() + ">");
        open.pop_back();
        if (open.empty()) break;
      } else if (ev.kind == Event::Open) {
        open.push_back(ev.name);
      }
      body(ev);
    }
  }
  lx.skip_space();
  if (!lx.at_end()) lx.fail("content after the root element");
  return root;
}

// ---------------------------------------------------------------------------
// Schema builder: one frame per open element; a frame whose element is invalid (or
// sits where nothing is allowed) swallows its subtree.
// ---------------------------------------------------------------------------
class SchemaBuilder {
 public:
  explicit SchemaBuilder(Deferred& d) : err_(d) { stack_.emplace_back(); }

  void feed(const Event& ev) {
    if (ev.kind == Event::Text) return on_text(ev);
    if (ev.kind == Event::Close) return pop();
    push(ev);
    if (ev.kind == Event::SelfClose) pop();
  }
  std::vector<SchemaNode> root() { return std::move(stack_.front().node.children); }

 private:
  enum class Role { Root, Node, Union, Param, Dead };
  struct Frame {
    Role role = Role::Root;
    SchemaNode node;
    bool param_content = false;
    int line = 0, col = 0;
  };

  void on_text(const Event& ev) {
    Frame& f = stack_.back();
    switch (f.role) {
      case Role::Root:  // schema-level text becomes an always-included anonymous module
        if (!is_space_only(ev.text)) {
          SchemaNode anon;
          anon.kind = NodeKind::Module;
          anon.anonymous = true;
          anon.name = "__anon_" + std::to_string(anon_next_++);
          anon.children.push_back(make_text(trim(ev.text)));
          f.node.children.push_back(std::move(anon));
        }
        break;
      case Role::Union:
        if (!is_space_only(ev.text)) err_.note("text directly inside <union>", ev.line, ev.col);
        break;
      case Role::Param:
        f.param_content = true;
        break;
      case Role::Node:
        f.node.children.push_back(make_text(ev.text));
        break;
      case Role::Dead:
        break;
    }
  }

  void push(const Event& ev) {
    Frame& parent = stack_.back();
    Frame f;
    f.role = Role::Dead;
    f.line = ev.line;
    f.col = ev.col;
    if (parent.role == Role::Param) parent.param_content = true;
    if (parent.role == Role::Dead || parent.role == Role::Param) {
      // inside an invalid element or a param: already reported (or will be)
    } else if (parent.role == Role::Union && ev.name != "module") {
      err_.note("<union> may only contain <module> elements, found <" + ev.name + ">", ev.line, ev.col);
    } else if (ev.name == "module") {
      auto nm = attr_of(ev.attrs, "name");
      if (nm && !nm->empty()) {
        f.role = Role::Node;
        f.node.kind = NodeKind::Module;
        f.node.name = *nm;
      } else {
        err_.note("<module> needs a non-empty name", ev.line, ev.col);
      }
    } else if (ev.name == "union") {
      f.role = Role::Union;
      f.node.kind = NodeKind::Union;
    } else if (ev.name == "param") {
      auto nm = attr_of(ev.attrs, "name");
      auto len = attr_of(ev.attrs, "len");
      if (!nm || nm->empty()) {
        err_.note("<param> needs a non-empty name", ev.line, ev.col);
      } else if (!len) {
        err_.note("<param> needs a len", ev.line, ev.col);
      } else if (decimal_len(*len) < 1) {
        err_.note("<param len=\"" + *len + "\"> is not a positive integer", ev.line, ev.col);
      } else {
        f.role = Role::Param;
        f.node.kind = NodeKind::Param;
        f.node.name = *nm;
        f.node.param_len = decimal_len(*len);
      }
    } else if (is_chat_role(ev.name)) {
      f.role = Role::Node;
      f.node.kind = NodeKind::Chat;
      f.node.role = ev.name;
    } else {
      err_.note("<" + ev.name + "> is not a schema element", ev.line, ev.col);
    }
    stack_.push_back(std::move(f));
  }

  void pop() {
    Frame f = std::move(stack_.back());
    stack_.pop_back();
    if (f.role == Role::Dead) return;
    if (f.role == Role::Param && f.param_content) {
      err_.note("<param> must be an empty element", f.line, f.col);
      return;
    }
    stack_.back().node.children.push_back(std::move(f.node));
  }

  Deferred& err_;
  std::vector<Frame> stack_;
  int anon_next_ = 0;
};

// ---------------------------------------------------------------------------
// Prompt builder.  Under an import, a child element is an argument when it has no
// attributes, no element children and non-empty text; otherwise it is a nested import.
// That is only known at its end tag, so every element frame collects both readings.
// ---------------------------------------------------------------------------
class PromptBuilder {
 public:
  explicit PromptBuilder(Deferred& d) : err_(d) { stack_.emplace_back(); }

  void feed(const Event& ev) {
    if (ev.kind == Event::Text) return on_text(ev);
    if (ev.kind == Event::Close) return pop();
    Frame f;
    f.name = ev.name;
    f.attrs = ev.attrs;
    f.line = ev.line;
    f.col = ev.col;
    if (stack_.size() > 1) stack_.back().has_elements = true;
    stack_.push_back(std::move(f));
    if (ev.kind == Event::SelfClose) pop();
  }
  std::vector<PromptItem> items() { return std::move(stack_.front().items); }

 private:
  struct Frame {  // stack_[0] is the <prompt> root
    std::string name;
    Attrs attrs;
    std::string text;                 // concatenated text runs
    bool has_elements = false;
    std::optional<Event> stray_text;  // first non-blank text run (an error if this is an import)
    std::vector<std::pair<std::string, std::string>> args;
    std::vector<PromptItem> items;    // nested imports (root: every item)
    int line = 0, col = 0;
  };

  void on_text(const Event& ev) {
    Frame& f = stack_.back();
    if (stack_.size() == 1) {  // prompt-level text: new uncached text
      if (!is_space_only(ev.text)) {
        PromptItem it;
        it.kind = PromptItem::Kind::Text;
        it.text = trim(ev.text);
        f.items.push_back(std::move(it));
      }
      return;
    }
    f.text += ev.text;
    if (!f.stray_text && !is_space_only(ev.text)) f.stray_text = ev;
  }

  void pop() {
    Frame f = std::move(stack_.back());
    stack_.pop_back();
    Frame& parent = stack_.back();
    const bool under_import = stack_.size() > 1;
    if (under_import && f.attrs.empty() && !f.has_elements && !f.text.empty()) {
      parent.args.emplace_back(f.name, f.text);
      return;
    }
    if (is_reserved(f.name)) {
      err_.note("<" + f.name + "> is a reserved tag, not a module import", f.line, f.col);
      return;
    }
    if (f.stray_text) err_.note("text inside the import <" + f.name + ">", f.stray_text->line, f.stray_text->col);
    PromptItem it;
    it.kind = PromptItem::Kind::Import;
    it.import.name = f.name;
    it.import.args = std::move(f.attrs);  // attribute arguments first, then element arguments
    for (auto& a : f.args) it.import.args.push_back(std::move(a));
    it.import.children = std::move(f.items);
    parent.items.push_back(std::move(it));
  }

  Deferred& err_;
  std::vector<Frame> stack_;
};

// ---------------------------------------------------------------------------
// Serialization
// ---------------------------------------------------------------------------
void put_escaped(std::string& out, const std::string& s, bool in_attr) {
  for (char c : s) switch (c) {
      case '<': out += "&lt;"; break;
      case '>': out += "&gt;"; break;
      case '&': out += "&amp;"; break;
      case '"':
        if (in_attr) {
          out += "&quot;";
          break;
        }
        [[fallthrough]];
      default: out.push_back(c);
    }
}

void write_nodes(std::string& out, const std::vector<SchemaNode>& nodes);

void write_node(std::string& out, const SchemaNode& n) {
  switch (n.kind) {
    case NodeKind::Text:
      put_escaped(out, n.text, false);
      break;
    case NodeKind::Param:
      out += "<param name=\"";
      put_escaped(out, n.name, true);
      out += "\" len=\"";
      out += std::to_string(n.param_len);
      out += "\"/>";
      break;
    case NodeKind::Module:
      if (n.anonymous) {  // anonymous modules are bare schema text
        write_nodes(out, n.children);
        break;
      }
      out += "<module name=\"";
      put_escaped(out, n.name, true);
      out += "\">";
      write_nodes(out, n.children);
      out += "</module>";
      break;
    case NodeKind::Union:
    case NodeKind::Chat: {
      const std::string tag = n.kind == NodeKind::Union ? std::string("union") : n.role;
      out += "<" + tag + ">";
      write_nodes(out, n.children);
      out += "</" + tag + ">";
      break;
    }
  }
}

void write_nodes(std::string& out, const std::vector<SchemaNode>& nodes) {
  for (const SchemaNode& n : nodes) write_node(out, n);
}

void write_items(std::string& out, const std::vector<PromptItem>& items) {
  for (const PromptItem& it : items) {
    if (it.kind == PromptItem::Kind::Text) {
      put_escaped(out, it.text, false);
      continue;
    }
    const ModuleImport& imp = it.import;
    if (imp.args.empty() && imp.children.empty()) {
      out += "<" + imp.name + "/>";
      continue;
    }
    out += "<" + imp.name + ">";
    for (const auto& [param, value] : imp.args) {  // arguments always as child elements
      out += "<" + param + ">";
      put_escaped(out, value, false);
      out += "</" + param + ">";
    }
    write_items(out, imp.children);
    out += "</" + imp.name + ">";
  }
}

}  // namespace

SchemaDoc parse_schema(const std::string& text) {
  Deferred err;
  SchemaBuilder b(err);
  const Event root = scan_document(text, [&](const Event& ev) { b.feed(ev); });
  if (root.name != "schema") throw Error(ErrorCode::SyntaxError, "the root element is <" + root.name + ">, not <schema>",
                                         root.line, root.col);
  auto name = attr_of(root.attrs, "name");
  if (!name || name->empty())
    throw Error(ErrorCode::SyntaxError, "<schema> needs a non-empty name", root.line, root.col);
  err.raise();
  SchemaDoc doc;
  doc.name = *name;
  doc.root = b.root();
  // params only inside modules (a chat or union between them and the module is fine);
  // module names unique over the whole tree
  std::set<std::string> names;
  std::vector<std::pair<const SchemaNode*, bool>> todo;  // (node, inside a module)
  for (auto it = doc.root.rbegin(); it != doc.root.rend(); ++it) todo.emplace_back(&*it, false);
  std::vector<std::string> in_order;
  while (!todo.empty()) {
    auto [n, in_module] = todo.back();
    todo.pop_back();
    if (n->kind == NodeKind::Param && !in_module)
      throw Error(ErrorCode::SyntaxError, "<param " + n->name + "> outside any module");
    if (n->kind == NodeKind::Module) in_order.push_back(n->name);
    const bool child_in_module = in_module || n->kind == NodeKind::Module;
    for (auto it = n->children.rbegin(); it != n->children.rend(); ++it) todo.emplace_back(&*it, child_in_module);
  }
  for (const std::string& nm : in_order)
    if (!names.insert(nm).second) throw Error(ErrorCode::SyntaxError, "module name \"" + nm + "\" is used twice");
  return doc;
}

PromptDoc parse_prompt(const std::string& text) {
  Deferred err;
  PromptBuilder b(err);
  const Event root = scan_document(text, [&](const Event& ev) { b.feed(ev); });
  if (root.name != "prompt") throw Error(ErrorCode::SyntaxError, "the root element is <" + root.name + ">, not <prompt>",
                                         root.line, root.col);
  auto schema = attr_of(root.attrs, "schema");
  if (!schema || schema->empty())
    throw Error(ErrorCode::MissingSchemaAttr, "<prompt> needs a schema attribute", root.line, root.col);
  err.raise();
  PromptDoc doc;
  doc.schema_name = *schema;
  doc.items = b.items();
  return doc;
}

std::string serialize(const SchemaDoc& doc) {
  std::string out = "<schema name=\"";
  put_escaped(out, doc.name, true);
  out += "\">";
  write_nodes(out, doc.root);
  out += "</schema>";
  return out;
}

std::string serialize(const PromptDoc& doc) {
  std::string out = "<prompt schema=\"";
  put_escaped(out, doc.schema_name, true);
  out += "\">";
  write_items(out, doc.items);
  out += "</prompt>";
  return out;
}

// ---------------------------------------------------------------------------
// Validation
// ---------------------------------------------------------------------------

void ValidationReport::add(Severity s, const std::string& code, const std::string& msg) {
  if (s == Severity::Error) ok = false;
  issues.push_back({s, code, msg});
}

std::string ValidationReport::to_json() const {
  nlohmann::json arr = nlohmann::json::array();
  for (const Issue& i : issues)
    arr.push_back({{"severity", i.severity == Severity::Error ? "error" : "warning"},
                   {"code", i.code},
                   {"message", i.message},
                   {"line", 0},
                   {"col", 0}});
  nlohmann::json j;
  j["ok"] = ok;
  j["issues"] = std::move(arr);
  return j.dump();
}

namespace {

// What validation needs to know about one schema module.
struct ModuleFacts {
  std::string parent;  // enclosing module ("" at top level); chat tags are transparent
  int union_id = -1;   // union it is an arm of (pre-order numbering), -1 = none
  std::map<std::string, int> params;  // its own params, including those inside its chat tags
};

// Schema facts by an explicit-stack walk.  A union's arms (directly, or through chat
// tags) carry its pre-order number; a module's own params are its param children and
// params reached from it through chat tags only.
std::map<std::string, ModuleFacts> schema_facts(const SchemaDoc& schema) {
  std::map<std::string, ModuleFacts> facts;
  struct Item {
    const SchemaNode* n;
    std::string parent;
    int union_id;
    ModuleFacts* owner;  // module whose params a param here belongs to (through chats)
  };
  int unions = 0;
  std::vector<Item> todo;
  for (auto it = schema.root.rbegin(); it != schema.root.rend(); ++it) todo.push_back({&*it, "", -1, nullptr});
  while (!todo.empty()) {
    Item cur = todo.back();
    todo.pop_back();
    const SchemaNode& n = *cur.n;
    std::vector<Item> kids;
    if (n.kind == NodeKind::Module) {
      ModuleFacts& f = facts[n.name];
      f = ModuleFacts{cur.parent, cur.union_id, {}};
      for (const SchemaNode& c : n.children) kids.push_back({&c, n.name, -1, &f});
    } else if (n.kind == NodeKind::Union) {
      const int id = unions++;
      for (const SchemaNode& c : n.children) kids.push_back({&c, cur.parent, id, nullptr});
    } else if (n.kind == NodeKind::Chat) {
      for (const SchemaNode& c : n.children) kids.push_back({&c, cur.parent, cur.union_id, cur.owner});
    } else if (n.kind == NodeKind::Param && cur.owner) {
      cur.owner->params[n.name] = n.param_len;
    }
    for (auto it = kids.rbegin(); it != kids.rend(); ++it) todo.push_back(*it);
  }
  return facts;
}

}  // namespace

ValidationReport validate_prompt(const PromptDoc& prompt, const SchemaDoc& schema) {
  ValidationReport rep;
  if (prompt.schema_name != schema.name) {
    rep.add(Severity::Error, "UNKNOWN_SCHEMA",
            "prompt references schema \"" + prompt.schema_name + "\", validated against \"" + schema.name + "\"");
    return rep;
  }
  const std::map<std::string, ModuleFacts> facts = schema_facts(schema);
  std::map<std::string, int> times_imported;
  std::map<int, std::vector<std::string>> union_members;

  // imports in document order, depth first; an unknown module's children are not visited
  struct Visit {
    const ModuleImport* imp;
    std::string enclosing;
  };
  std::vector<Visit> todo;
  auto push_items = [&](const std::vector<PromptItem>& items, const std::string& enclosing) {
    for (auto it = items.rbegin(); it != items.rend(); ++it)
      if (it->kind == PromptItem::Kind::Import) todo.push_back({&it->import, enclosing});
  };
  push_items(prompt.items, "");
  while (!todo.empty()) {
    const Visit v = todo.back();
    todo.pop_back();
    const ModuleImport& imp = *v.imp;
    auto fi = facts.find(imp.name);
    if (fi == facts.end()) {
      rep.add(Severity::Error, "UNKNOWN_MODULE", "unknown module \"" + imp.name + "\"");
      continue;
    }
    const ModuleFacts& f = fi->second;
    if (f.parent != v.enclosing)
      rep.add(Severity::Error, "PARENT_NOT_IMPORTED",
              "module \"" + imp.name + "\" must be imported inside \"" +
                  (f.parent.empty() ? std::string("<top level>") : f.parent) + "\"");
    if (++times_imported[imp.name] > 1)
      rep.add(Severity::Error, "DUPLICATE_IMPORT", "module \"" + imp.name + "\" imported more than once");
    if (f.union_id >= 0) union_members[f.union_id].push_back(imp.name);
    std::set<std::string> supplied;
    for (const auto& [param, value] : imp.args) {
      supplied.insert(param);
      auto p = f.params.find(param);
      if (p == f.params.end()) {
        rep.add(Severity::Error, "UNKNOWN_PARAM", "module \"" + imp.name + "\" has no parameter \"" + param + "\"");
      } else if (static_cast<int>(tok::tokenize(value).size()) > p->second) {
        rep.add(Severity::Error, "ARG_TOO_LONG",
                "argument for \"" + param + "\" is " + std::to_string(tok::tokenize(value).size()) +
                    " tokens, parameter len is " + std::to_string(p->second));
      }
    }
    for (const auto& [param, len] : f.params)
      if (!supplied.count(param))
        rep.add(Severity::Warning, "UNUSED_PARAM",
                "parameter \"" + param + "\" of module \"" + imp.name + "\" not supplied");
    push_items(imp.children, imp.name);
  }
  for (const auto& [id, members] : union_members) {
    if (members.size() < 2) continue;
    std::string list = members.front();
    for (size_t i = 1; i < members.size(); ++i) list += ", " + members[i];
    rep.add(Severity::Error, "UNION_CONFLICT", "modules from the same union imported together: " + list);
  }
  return rep;
}

// ---------------------------------------------------------------------------
// Chat-template expansion
// ---------------------------------------------------------------------------

ChatTemplate ChatTemplate::llama2() {
  ChatTemplate t;
  t.roles["system"] = {"<<SYS>>\n", "\n<</SYS>>\n\n"};
  t.roles["user"] = {"[INST] ", " [/INST]"};
  t.roles["assistant"] = {" ", " </s>"};
  return t;
}

namespace {

// Replaces every chat tag by (prefix text, its expanded children, suffix text).
std::vector<SchemaNode> without_chat(const std::vector<SchemaNode>& in, const ChatTemplate& tpl) {
  std::vector<SchemaNode> out;
  for (const SchemaNode& n : in) {
    if (n.kind != NodeKind::Chat) {
      SchemaNode c = n;
      c.children = without_chat(n.children, tpl);
      out.push_back(std::move(c));
      continue;
    }
    auto role = tpl.roles.find(n.role);
    if (role == tpl.roles.end()) throw Error(ErrorCode::UnknownRole, "the chat template has no role \"" + n.role + "\"");
    if (!role->second.prefix.empty()) out.push_back(make_text(role->second.prefix));
    for (SchemaNode& c : without_chat(n.children, tpl)) out.push_back(std::move(c));
    if (!role->second.suffix.empty()) out.push_back(make_text(role->second.suffix));
  }
  return out;
}

// Largest N over anonymous modules named "__anon_<N...>" anywhere in the tree (the
// number is read like std::stoi: leading blanks, sign, digits, rest ignored); -1 if none.
int max_anon_index(const std::vector<SchemaNode>& nodes) {
  int best = -1;
  std::vector<const SchemaNode*> todo;
  for (const SchemaNode& n : nodes) todo.push_back(&n);
  while (!todo.empty()) {
    const SchemaNode* n = todo.back();
    todo.pop_back();
    for (const SchemaNode& c : n->children) todo.push_back(&c);
    if (n->kind != NodeKind::Module || !n->anonymous || n->name.compare(0, 7, "__anon_") != 0) continue;
    const char* p = n->name.c_str() + 7;
    while (std::isspace(static_cast<unsigned char>(*p))) ++p;
    const bool neg = *p == '-';
    if (*p == '+' || *p == '-') ++p;
    if (!std::isdigit(static_cast<unsigned char>(*p))) continue;
    long long v = 0;
    while (std::isdigit(static_cast<unsigned char>(*p)) && v < 2147483648LL) v = v * 10 + (*p++ - '0');
    if (v <= 2147483647LL) best = std::max(best, static_cast<int>(neg ? -v : v));
  }
  return best;
}

}  // namespace

SchemaDoc expand_chat_tags(const SchemaDoc& doc, const ChatTemplate& tpl) {
  std::vector<SchemaNode> flat = without_chat(doc.root, tpl);
  int next_anon = max_anon_index(flat) + 1;
  SchemaDoc out;
  out.name = doc.name;
  // runs of schema-level text (template prefixes/suffixes) become new anonymous modules
  for (size_t i = 0; i < flat.size();) {
    if (flat[i].kind != NodeKind::Text) {
      out.root.push_back(std::move(flat[i++]));
      continue;
    }
    std::string run;
    while (i < flat.size() && flat[i].kind == NodeKind::Text) run += flat[i++].text;
    if (run.empty()) continue;
    SchemaNode anon;
    anon.kind = NodeKind::Module;
    anon.anonymous = true;
    anon.name = "__anon_" + std::to_string(next_anon++);
    anon.children.push_back(make_text(std::move(run)));
    out.root.push_back(std::move(anon));
  }
  return out;
}

// ---------------------------------------------------------------------------
// AST JSON interchange (test fixtures replay the reference's in-memory ASTs)
// ---------------------------------------------------------------------------

namespace {
using nlohmann::json;

json node_json(const SchemaNode& n) {
  json j;
  switch (n.kind) {
    case NodeKind::Text: return {{"k", "text"}, {"t", n.text}};
    case NodeKind::Param: return {{"k", "param"}, {"name", n.name}, {"len", n.param_len}};
    case NodeKind::Module: j = {{"k", "module"}, {"name", n.name}, {"anon", n.anonymous}}; break;
    case NodeKind::Union: j = {{"k", "union"}}; break;
    case NodeKind::Chat: j = {{"k", "chat"}, {"role", n.role}}; break;
  }
  j["ch"] = json::array();
  for (auto& c : n.children) j["ch"].push_back(node_json(c));
  return j;
}

SchemaNode node_from(const json& j) {
  SchemaNode n;
  const std::string k = j.at("k");
  if (k == "text") return make_text(j.at("t"));
  if (k == "param") {
    n.kind = NodeKind::Param;
    n.name = j.at("name");
    n.param_len = j.at("len");
    return n;
  }
  if (k == "module") {
    n.kind = NodeKind::Module;
    n.name = j.at("name");
    n.anonymous = j.value("anon", false);
  } else if (k == "union") {
    n.kind = NodeKind::Union;
  } else if (k == "chat") {
    n.kind = NodeKind::Chat;
    n.role = j.at("role");
  } else {
    throw Error(ErrorCode::SyntaxError, "unknown AST node kind \"" + k + "\"");
  }
  for (auto& c : j.at("ch")) n.children.push_back(node_from(c));
  return n;
}

json item_json(const PromptItem& it) {
  if (it.kind == PromptItem::Kind::Text) return {{"k", "text"}, {"t", it.text}};
  json j = {{"k", "import"}, {"name", it.import.name}};
  j["args"] = json::array();
  for (auto& [a, b] : it.import.args) j["args"].push_back(json::array({a, b}));
  j["ch"] = json::array();
  for (auto& c : it.import.children) j["ch"].push_back(item_json(c));
  return j;
}

PromptItem item_from(const json& j) {
  PromptItem it;
  if (j.at("k") == "text") {
    it.kind = PromptItem::Kind::Text;
    it.text = j.at("t");
    return it;
  }
  it.kind = PromptItem::Kind::Import;
  it.import.name = j.at("name");
  for (auto& a : j.at("args")) it.import.args.emplace_back(a.at(0), a.at(1));
  for (auto& c : j.at("ch")) it.import.children.push_back(item_from(c));
  return it;
}

json parse_json(const std::string& s) {
  try {
    return json::parse(s);
  } catch (const std::exception& e) {
    throw Error(ErrorCode::SyntaxError, std::string("bad AST JSON: ") + e.what());
  }
}
}  // namespace

std::string schema_to_ast_json(const SchemaDoc& d) {
  json j = {{"name", d.name}, {"root", json::array()}};
  for (auto& n : d.root) j["root"].push_back(node_json(n));
  return j.dump(-1, ' ', false, json::error_handler_t::replace);
}

SchemaDoc schema_from_ast_json(const std::string& s) {
  json j = parse_json(s);
  SchemaDoc d;
  try {
    d.name = j.at("name");
    for (auto& n : j.at("root")) d.root.push_back(node_from(n));
  } catch (const json::exception& e) {
    throw Error(ErrorCode::SyntaxError, std::string("bad schema AST: ") + e.what());
  }
  return d;
}

std::string prompt_to_ast_json(const PromptDoc& d) {
  json j = {{"schema", d.schema_name}, {"items", json::array()}};
  for (auto& it : d.items) j["items"].push_back(item_json(it));
  return j.dump(-1, ' ', false, json::error_handler_t::replace);
}

PromptDoc prompt_from_ast_json(const std::string& s) {
  json j = parse_json(s);
  PromptDoc d;
  try {
    d.schema_name = j.at("schema");
    for (auto& it : j.at("items")) d.items.push_back(item_from(it));
  } catch (const json::exception& e) {
    throw Error(ErrorCode::SyntaxError, std::string("bad prompt AST: ") + e.what());
  }
  return d;
}

}  // namespace pml
}  // namespace pcb

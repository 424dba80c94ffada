// PML front end, written from scratch against the semantics of the reference
// (proj/core/src/pml.cpp): scanner grammar 30-177, schema building 236-324,
// prompt building 374-406, parse 424-473, serialize 477-551, validation
// 556-701, chat expansion 707-786.  Host-only: no device work happens here.
#include "pml.hpp"

#include <algorithm>
#include <cctype>
#include <functional>
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
  std::vector<int> t(s.size());
  for (size_t i = 0; i < s.size(); ++i) t[i] = static_cast<unsigned char>(s[i]);
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
  if (kind != o.kind) return false;
  return kind == Kind::Text ? text == o.text : import == o.import;
}

namespace {

// ---------------------------------------------------------------------------
// Element reader.  Produces a generic element tree; schema / prompt builders
// interpret it.  Grammar: elements with quoted attributes, self-closing tags,
// text with the five predefined entities; no comments, CDATA or numeric refs.
// ---------------------------------------------------------------------------

struct Elem {
  bool text_node = false;
  std::string tag;   // element
  std::string body;  // text node (entities decoded)
  std::vector<std::pair<std::string, std::string>> attrs;
  std::vector<Elem> kids;
  int line = 1, col = 1;
};

class Reader {
 public:
  explicit Reader(const std::string& s) : s_(s) {}

  Elem document() {
    blanks();
    if (done() || cur() != '<') err("expected a root element");
    Elem root = element();
    blanks();
    if (!done()) err("trailing content after root element");
    return root;
  }

 private:
  const std::string& s_;
  size_t i_ = 0;
  int line_ = 1, col_ = 1;

  [[noreturn]] void err(const std::string& m) const {
    throw Error(ErrorCode::SyntaxError, m, line_, col_);
  }
  bool done() const { return i_ >= s_.size(); }
  char cur() const { return s_[i_]; }
  char take() {
    char c = s_[i_++];
    if (c == '\n') {
      ++line_;
      col_ = 1;
    } else {
      ++col_;
    }
    return c;
  }
  void blanks() {
    while (!done() && std::isspace(static_cast<unsigned char>(cur()))) take();
  }
  static bool first_name_char(char c) { return std::isalpha(static_cast<unsigned char>(c)) || c == '_'; }
  static bool name_char(char c) {
    return std::isalnum(static_cast<unsigned char>(c)) || c == '_' || c == '-' || c == '.';
  }
  std::string name() {
    if (done() || !first_name_char(cur())) err("expected a name");
    size_t b = i_;
    while (!done() && name_char(cur())) take();
    return s_.substr(b, i_ - b);
  }
  // positioned after '&'
  std::string entity() {
    std::string e;
    while (!done() && cur() != ';' && e.size() < 8) e.push_back(take());
    if (done() || cur() != ';') err("unterminated entity");
    take();
    static const std::pair<const char*, const char*> table[] = {
        {"lt", "<"}, {"gt", ">"}, {"amp", "&"}, {"quot", "\""}, {"apos", "'"}};
    for (auto& [k, v] : table)
      if (e == k) return v;
    err("unknown entity &" + e + ";");
  }
  std::string quoted() {
    if (done() || (cur() != '"' && cur() != '\'')) err("expected quoted attribute value");
    char q = take();
    std::string v;
    for (;;) {
      if (done()) err("unterminated attribute value");
      char c = cur();
      if (c == q) break;
      if (c == '<') err("'<' in attribute value");
      if (c == '&') {
        take();
        v += entity();
      } else {
        v.push_back(take());
      }
    }
    take();
    return v;
  }
  Elem element() {
    Elem e;
    e.line = line_;
    e.col = col_;
    take();  // '<'
    e.tag = name();
    for (;;) {
      blanks();
      if (done()) err("unterminated tag <" + e.tag + ">");
      if (cur() == '/') {
        take();
        if (done() || cur() != '>') err("malformed self-closing tag");
        take();
        return e;
      }
      if (cur() == '>') {
        take();
        break;
      }
      std::string k = name();
      blanks();
      if (done() || cur() != '=') err("expected '=' after attribute name");
      take();
      blanks();
      std::string v = quoted();
      for (auto& a : e.attrs)
        if (a.first == k) err("duplicate attribute '" + k + "'");
      e.attrs.emplace_back(std::move(k), std::move(v));
    }
    Elem txt;
    txt.text_node = true;
    auto push_text = [&] {
      if (!txt.body.empty()) {
        e.kids.push_back(std::move(txt));
        txt = Elem{};
        txt.text_node = true;
      }
    };
    for (;;) {
      if (done()) err("missing closing tag </" + e.tag + ">");
      char c = cur();
      if (c == '<') {
        push_text();
        if (i_ + 1 < s_.size() && s_[i_ + 1] == '/') {
          take();
          take();
          std::string close = name();
          blanks();
          if (done() || cur() != '>') err("malformed closing tag");
          take();
          if (close != e.tag) err("mismatched closing tag </" + close + ">, expected </" + e.tag + ">");
          return e;
        }
        e.kids.push_back(element());
        continue;
      }
      if (txt.body.empty()) {
        txt.line = line_;
        txt.col = col_;
      }
      if (c == '&') {
        take();
        txt.body += entity();
      } else {
        txt.body.push_back(take());
      }
    }
  }
};

bool blank(const std::string& s) {
  for (unsigned char c : s)
    if (!std::isspace(c)) return false;
  return true;
}

std::string strip(const std::string& s) {
  size_t b = 0, e = s.size();
  while (b < e && std::isspace(static_cast<unsigned char>(s[b]))) ++b;
  while (e > b && std::isspace(static_cast<unsigned char>(s[e - 1]))) --e;
  return s.substr(b, e - b);
}

const std::string* attr(const Elem& e, const char* key) {
  for (auto& a : e.attrs)
    if (a.first == key) return &a.second;
  return nullptr;
}

bool chat_role(const std::string& t) { return t == "system" || t == "user" || t == "assistant"; }

SchemaNode text_node(std::string t) {
  SchemaNode n;
  n.kind = NodeKind::Text;
  n.text = std::move(t);
  return n;
}

// std::stoi-compatible strict parse: optional leading blanks and sign, digits,
// whole string consumed, int range.  Returns 0 on any failure.
int parse_len(const std::string& s) {
  size_t i = 0;
  while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  bool neg = false;
  if (i < s.size() && (s[i] == '+' || s[i] == '-')) neg = s[i++] == '-';
  size_t d0 = i;
  long long v = 0;
  while (i < s.size() && std::isdigit(static_cast<unsigned char>(s[i]))) {
    v = v * 10 + (s[i++] - '0');
    if (v > 2147483648LL) return 0;
  }
  if (i == d0 || i != s.size()) return 0;
  if (neg) v = -v;
  if (v > 2147483647LL || v < -2147483648LL) return 0;
  return static_cast<int>(v);
}

class SchemaMaker {
 public:
  std::vector<SchemaNode> root(const Elem& schema) {
    std::vector<SchemaNode> out;
    for (const Elem& k : schema.kids) {
      if (k.text_node) {
        if (blank(k.body)) continue;
        SchemaNode anon;
        anon.kind = NodeKind::Module;
        anon.name = "__anon_" + std::to_string(anon_++);
        anon.anonymous = true;
        anon.children.push_back(text_node(strip(k.body)));
        out.push_back(std::move(anon));
      } else {
        out.push_back(node(k));
      }
    }
    return out;
  }

 private:
  int anon_ = 0;

  std::vector<SchemaNode> content(const Elem& e) {
    std::vector<SchemaNode> out;
    for (const Elem& k : e.kids) out.push_back(k.text_node ? text_node(k.body) : node(k));
    return out;
  }
  SchemaNode module(const Elem& e) {
    const std::string* nm = attr(e, "name");
    if (!nm || nm->empty())
      throw Error(ErrorCode::SyntaxError, "<module> requires a non-empty name attribute", e.line, e.col);
    SchemaNode n;
    n.kind = NodeKind::Module;
    n.name = *nm;
    n.children = content(e);
    return n;
  }
  SchemaNode node(const Elem& e) {
    if (e.tag == "module") return module(e);
    if (e.tag == "union") {
      SchemaNode u;
      u.kind = NodeKind::Union;
      for (const Elem& k : e.kids) {
        if (k.text_node) {
          if (blank(k.body)) continue;
          throw Error(ErrorCode::SyntaxError, "bare text under <union>", k.line, k.col);
        }
        if (k.tag != "module")
          throw Error(ErrorCode::SyntaxError, "non-module child <" + k.tag + "> of <union>", k.line, k.col);
        u.children.push_back(module(k));
      }
      return u;
    }
    if (e.tag == "param") {
      const std::string* nm = attr(e, "name");
      if (!nm || nm->empty())
        throw Error(ErrorCode::SyntaxError, "<param> requires a non-empty name attribute", e.line, e.col);
      const std::string* len = attr(e, "len");
      if (!len) throw Error(ErrorCode::SyntaxError, "<param> requires a len attribute", e.line, e.col);
      int v = parse_len(*len);
      if (v < 1)
        throw Error(ErrorCode::SyntaxError, "<param> len must be a positive integer, got \"" + *len + "\"",
                    e.line, e.col);
      if (!e.kids.empty()) throw Error(ErrorCode::SyntaxError, "<param> must be empty", e.line, e.col);
      SchemaNode p;
      p.kind = NodeKind::Param;
      p.name = *nm;
      p.param_len = v;
      return p;
    }
    if (chat_role(e.tag)) {
      SchemaNode c;
      c.kind = NodeKind::Chat;
      c.role = e.tag;
      c.children = content(e);
      return c;
    }
    throw Error(ErrorCode::SyntaxError, "unknown tag <" + e.tag + "> in schema", e.line, e.col);
  }
};

void check_params(const std::vector<SchemaNode>& ns, bool in_module) {
  for (const SchemaNode& n : ns) {
    if (n.kind == NodeKind::Param && !in_module)
      throw Error(ErrorCode::SyntaxError, "<param> must appear inside a <module>");
    if (n.kind == NodeKind::Module) check_params(n.children, true);
    if (n.kind == NodeKind::Union || n.kind == NodeKind::Chat) check_params(n.children, in_module);
  }
}

void module_names(const std::vector<SchemaNode>& ns, std::vector<std::string>& out) {
  for (const SchemaNode& n : ns) {
    if (n.kind == NodeKind::Module) out.push_back(n.name);
    if (n.kind == NodeKind::Module || n.kind == NodeKind::Union || n.kind == NodeKind::Chat)
      module_names(n.children, out);
  }
}

const std::set<std::string>& reserved() {
  static const std::set<std::string> r = {"schema", "module", "union", "param",
                                          "prompt", "system", "user",  "assistant"};
  return r;
}

ModuleImport make_import(const Elem& e) {
  if (reserved().count(e.tag))
    throw Error(ErrorCode::SyntaxError, "reserved tag <" + e.tag + "> cannot be imported", e.line, e.col);
  ModuleImport imp;
  imp.name = e.tag;
  imp.args = e.attrs;
  for (const Elem& k : e.kids) {
    if (k.text_node) {
      if (blank(k.body)) continue;
      throw Error(ErrorCode::SyntaxError, "bare text inside module import <" + e.tag + ">", k.line, k.col);
    }
    // an argument element: no attributes, only text children, non-empty text
    bool is_arg = k.attrs.empty();
    std::string value;
    for (const Elem& t : k.kids) {
      if (!t.text_node) {
        is_arg = false;
        break;
      }
      value += t.body;
    }
    if (is_arg && !value.empty()) {
      imp.args.emplace_back(k.tag, value);
    } else {
      PromptItem child;
      child.kind = PromptItem::Kind::Import;
      child.import = make_import(k);
      imp.children.push_back(std::move(child));
    }
  }
  return imp;
}

void esc(const std::string& s, std::string& out, bool attr_mode) {
  for (char c : s) {
    if (c == '<') out += "&lt;";
    else if (c == '>') out += "&gt;";
    else if (c == '&') out += "&amp;";
    else if (attr_mode && c == '"') out += "&quot;";
    else out.push_back(c);
  }
}

void emit(const SchemaNode& n, std::string& o) {
  switch (n.kind) {
    case NodeKind::Text: esc(n.text, o, false); return;
    case NodeKind::Param:
      o += "<param name=\"";
      esc(n.name, o, true);
      o += "\" len=\"" + std::to_string(n.param_len) + "\"/>";
      return;
    case NodeKind::Module:
      if (n.anonymous) {
        for (auto& c : n.children) emit(c, o);
        return;
      }
      o += "<module name=\"";
      esc(n.name, o, true);
      o += "\">";
      for (auto& c : n.children) emit(c, o);
      o += "</module>";
      return;
    case NodeKind::Union:
      o += "<union>";
      for (auto& c : n.children) emit(c, o);
      o += "</union>";
      return;
    case NodeKind::Chat:
      o += "<" + n.role + ">";
      for (auto& c : n.children) emit(c, o);
      o += "</" + n.role + ">";
      return;
  }
}

void emit(const PromptItem& it, std::string& o) {
  if (it.kind == PromptItem::Kind::Text) {
    esc(it.text, o, false);
    return;
  }
  const ModuleImport& m = it.import;
  o += "<" + m.name;
  if (m.args.empty() && m.children.empty()) {
    o += "/>";
    return;
  }
  o += ">";
  for (auto& [k, v] : m.args) {
    o += "<" + k + ">";
    esc(v, o, false);
    o += "</" + k + ">";
  }
  for (auto& c : m.children) emit(c, o);
  o += "</" + m.name + ">";
}

}  // namespace

SchemaDoc parse_schema(const std::string& text) {
  Reader r(text);
  Elem root = r.document();
  if (root.tag != "schema")
    throw Error(ErrorCode::SyntaxError, "root element must be <schema>, got <" + root.tag + ">", root.line,
                root.col);
  const std::string* nm = attr(root, "name");
  if (!nm || nm->empty())
    throw Error(ErrorCode::SyntaxError, "<schema> requires a non-empty name attribute", root.line, root.col);
  SchemaDoc doc;
  doc.name = *nm;
  SchemaMaker maker;
  doc.root = maker.root(root);
  check_params(doc.root, false);
  std::vector<std::string> names;
  module_names(doc.root, names);
  std::set<std::string> seen;
  for (auto& n : names)
    if (!seen.insert(n).second) throw Error(ErrorCode::SyntaxError, "duplicate module name \"" + n + "\"");
  return doc;
}

PromptDoc parse_prompt(const std::string& text) {
  Reader r(text);
  Elem root = r.document();
  if (root.tag != "prompt")
    throw Error(ErrorCode::SyntaxError, "root element must be <prompt>, got <" + root.tag + ">", root.line,
                root.col);
  const std::string* sc = attr(root, "schema");
  if (!sc || sc->empty())
    throw Error(ErrorCode::MissingSchemaAttr, "<prompt> requires a schema attribute", root.line, root.col);
  PromptDoc doc;
  doc.schema_name = *sc;
  for (const Elem& k : root.kids) {
    PromptItem it;
    if (k.text_node) {
      if (blank(k.body)) continue;
      it.kind = PromptItem::Kind::Text;
      it.text = strip(k.body);
    } else {
      it.kind = PromptItem::Kind::Import;
      it.import = make_import(k);
    }
    doc.items.push_back(std::move(it));
  }
  return doc;
}

std::string serialize(const SchemaDoc& doc) {
  std::string o = "<schema name=\"";
  esc(doc.name, o, true);
  o += "\">";
  for (auto& n : doc.root) emit(n, o);
  return o + "</schema>";
}

std::string serialize(const PromptDoc& doc) {
  std::string o = "<prompt schema=\"";
  esc(doc.schema_name, o, true);
  o += "\">";
  for (auto& it : doc.items) emit(it, o);
  return o + "</prompt>";
}

// ---------------------------------------------------------------------------
// Validation (reference pml.cpp:556-701)
// ---------------------------------------------------------------------------

void ValidationReport::add(Severity s, const std::string& code, const std::string& msg) {
  if (s == Severity::Error) ok = false;
  issues.push_back({s, code, msg});
}

std::string ValidationReport::to_json() const {
  nlohmann::json j;
  j["ok"] = ok;
  j["issues"] = nlohmann::json::array();
  for (auto& i : issues)
    j["issues"].push_back({{"severity", i.severity == Severity::Error ? "error" : "warning"},
                           {"code", i.code},
                           {"message", i.message},
                           {"line", 0},
                           {"col", 0}});
  return j.dump();
}

namespace {

struct ModInfo {
  std::map<std::string, int> params;
  std::string parent;
  int union_group = -1;
};

struct Index {
  std::map<std::string, ModInfo> mods;
  int unions = 0;

  static void chat_params(const std::vector<SchemaNode>& ns, ModInfo& info) {
    for (auto& c : ns)
      if (c.kind == NodeKind::Chat) {
        for (auto& cc : c.children)
          if (cc.kind == NodeKind::Param) info.params[cc.name] = cc.param_len;
        chat_params(c.children, info);
      }
  }

  void walk(const std::vector<SchemaNode>& ns, const std::string& parent, int group) {
    for (auto& n : ns) {
      if (n.kind == NodeKind::Module) {
        ModInfo info;
        info.parent = parent;
        info.union_group = group;
        for (auto& c : n.children)
          if (c.kind == NodeKind::Param) info.params[c.name] = c.param_len;
        chat_params(n.children, info);
        mods[n.name] = std::move(info);
        walk(n.children, n.name, -1);
      } else if (n.kind == NodeKind::Union) {
        walk(n.children, parent, unions++);
      } else if (n.kind == NodeKind::Chat) {
        walk(n.children, parent, group);
      }
    }
  }
};

void check_imports(const std::vector<PromptItem>& items, const std::string& enclosing, const Index& idx,
                   ValidationReport& rep, std::map<std::string, int>& count,
                   std::map<int, std::vector<std::string>>& by_union) {
  for (auto& it : items) {
    if (it.kind != PromptItem::Kind::Import) continue;
    const ModuleImport& imp = it.import;
    auto f = idx.mods.find(imp.name);
    if (f == idx.mods.end()) {
      rep.add(Severity::Error, "UNKNOWN_MODULE", "unknown module \"" + imp.name + "\"");
      continue;
    }
    const ModInfo& info = f->second;
    if (info.parent != enclosing)
      rep.add(Severity::Error, "PARENT_NOT_IMPORTED",
              "module \"" + imp.name + "\" must be imported inside \"" +
                  (info.parent.empty() ? std::string("<top level>") : info.parent) + "\"");
    if (++count[imp.name] > 1)
      rep.add(Severity::Error, "DUPLICATE_IMPORT", "module \"" + imp.name + "\" imported more than once");
    if (info.union_group >= 0) by_union[info.union_group].push_back(imp.name);
    std::set<std::string> given;
    for (auto& [p, v] : imp.args) {
      given.insert(p);
      auto pp = info.params.find(p);
      if (pp == info.params.end()) {
        rep.add(Severity::Error, "UNKNOWN_PARAM", "module \"" + imp.name + "\" has no parameter \"" + p + "\"");
        continue;
      }
      int nt = static_cast<int>(v.size());  // byte tokenizer: one token per byte
      if (nt > pp->second)
        rep.add(Severity::Error, "ARG_TOO_LONG",
                "argument for \"" + p + "\" is " + std::to_string(nt) + " tokens, parameter len is " +
                    std::to_string(pp->second));
    }
    for (auto& [p, len] : info.params)
      if (!given.count(p))
        rep.add(Severity::Warning, "UNUSED_PARAM",
                "parameter \"" + p + "\" of module \"" + imp.name + "\" not supplied");
    check_imports(imp.children, imp.name, idx, rep, count, by_union);
  }
}

}  // namespace

ValidationReport validate_prompt(const PromptDoc& prompt, const SchemaDoc& schema) {
  ValidationReport rep;
  if (prompt.schema_name != schema.name) {
    rep.add(Severity::Error, "UNKNOWN_SCHEMA",
            "prompt references schema \"" + prompt.schema_name + "\", validated against \"" + schema.name + "\"");
    return rep;
  }
  Index idx;
  idx.walk(schema.root, "", -1);
  std::map<std::string, int> count;
  std::map<int, std::vector<std::string>> by_union;
  check_imports(prompt.items, "", idx, rep, count, by_union);
  for (auto& [g, names] : by_union)
    if (names.size() > 1) {
      std::string joined;
      for (auto& n : names) joined += (joined.empty() ? "" : ", ") + n;
      rep.add(Severity::Error, "UNION_CONFLICT", "modules from the same union imported together: " + joined);
    }
  return rep;
}

// ---------------------------------------------------------------------------
// Chat expansion (reference pml.cpp:707-786)
// ---------------------------------------------------------------------------

ChatTemplate ChatTemplate::llama2() {
  ChatTemplate t;
  t.roles["system"] = {"<<SYS>>\n", "\n<</SYS>>\n\n"};
  t.roles["user"] = {"[INST] ", " [/INST]"};
  t.roles["assistant"] = {" ", " </s>"};
  return t;
}

namespace {

void expand(const std::vector<SchemaNode>& in, const ChatTemplate& tpl, std::vector<SchemaNode>& out) {
  for (auto& n : in) {
    if (n.kind == NodeKind::Chat) {
      auto r = tpl.roles.find(n.role);
      if (r == tpl.roles.end()) throw Error(ErrorCode::UnknownRole, "no template for role \"" + n.role + "\"");
      if (!r->second.prefix.empty()) out.push_back(text_node(r->second.prefix));
      expand(n.children, tpl, out);
      if (!r->second.suffix.empty()) out.push_back(text_node(r->second.suffix));
      continue;
    }
    SchemaNode c = n;
    if (!c.children.empty()) {
      std::vector<SchemaNode> k;
      expand(n.children, tpl, k);
      c.children = std::move(k);
    }
    out.push_back(std::move(c));
  }
}

int highest_anon(const std::vector<SchemaNode>& ns) {
  int best = -1;
  for (auto& n : ns) {
    if (n.kind == NodeKind::Module && n.anonymous && n.name.rfind("__anon_", 0) == 0) {
      const std::string tail = n.name.substr(7);
      // std::stoi semantics: leading digits only; non-numeric names are ignored
      size_t i = 0;
      while (i < tail.size() && std::isspace(static_cast<unsigned char>(tail[i]))) ++i;
      bool neg = i < tail.size() && tail[i] == '-';
      if (i < tail.size() && (tail[i] == '+' || tail[i] == '-')) ++i;
      long long v = 0;
      size_t d0 = i;
      while (i < tail.size() && std::isdigit(static_cast<unsigned char>(tail[i])) && v < 2147483648LL)
        v = v * 10 + (tail[i++] - '0');
      if (i > d0 && v <= 2147483647LL) best = std::max(best, static_cast<int>(neg ? -v : v));
    }
    best = std::max(best, highest_anon(n.children));
  }
  return best;
}

}  // namespace

SchemaDoc expand_chat_tags(const SchemaDoc& doc, const ChatTemplate& tpl) {
  SchemaDoc out;
  out.name = doc.name;
  std::vector<SchemaNode> flat;
  expand(doc.root, tpl, flat);
  int next = highest_anon(flat) + 1;
  std::string run;
  auto flush = [&] {
    if (run.empty()) return;
    SchemaNode a;
    a.kind = NodeKind::Module;
    a.name = "__anon_" + std::to_string(next++);
    a.anonymous = true;
    a.children.push_back(text_node(std::move(run)));
    out.root.push_back(std::move(a));
    run.clear();
  };
  for (auto& n : flat) {
    if (n.kind == NodeKind::Text) {
      run += n.text;
    } else {
      flush();
      out.root.push_back(std::move(n));
    }
  }
  flush();
  return out;
}

// ---------------------------------------------------------------------------
// AST JSON interchange
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
  if (k == "text") return text_node(j.at("t"));
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

// Native grammar parser: EBNF text -> the int32 prefix IR of front_end.cpp
// (gm_grammar_parse, include/gmask.h).  The C++ form of
// paper_2411_15100_b200/grammar.py (which stays as the executable
// specification: tests/test_frontend.py compares the IR, the rule names,
// the root and every error message / position of the two).
//
// Surface semantics follow the reference exactly because they decide mask
// bits: literals are the UTF-8 of their text,
// \xHH a raw byte, \uXXXX the UTF-8 of a code point, simple escapes
// \n \t \r \" \\ \' (REF grammar.py:290, 326-350, 393-411); classes with
// \] \- \^ \[ escapes, '-' literal first / last, ']' literal only first
// (REF grammar.py:413-443); negated classes ASCII / \x only, complemented
// over bytes (REF grammar.py:576-586); positive classes above U+007F lowered
// to exact UTF-8 byte-range alternations, surrogates excluded (REF
// grammar.py:231-281, 565-594); * + ? {m} {m,} {m,n}; "" = empty string;
// root = `root` else the first rule; undefined references, duplicates, an
// empty grammar and unproductive rules are errors (REF grammar.py:629-656).
// Positions are 1-based (line, column) counted in code points, as Python
// indexes a str.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "gmask.h"

namespace gm {
void set_error(const std::string& msg);
}

namespace {

struct ParseFail {
  std::string msg;
  int line, col;  // 0: no position
};

struct Mask {
  uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  void range(int lo, int hi) {
    for (int b = lo; b <= hi; ++b) w[b >> 5] |= 1u << (b & 31);
  }
  bool empty() const {
    for (uint32_t x : w)
      if (x) return false;
    return true;
  }
};

// AST (the IR tags of front_end.cpp)
enum { E_EPS = 0, E_BYTES = 1, E_LIT = 2, E_SEQ = 3, E_ALT = 4, E_REP = 5, E_REF = 6 };
struct Node {
  int tag = E_EPS;
  Mask mask;                                 // BYTES
  std::string data;                          // LIT bytes / REF name
  std::vector<std::unique_ptr<Node>> items;  // SEQ / ALT / REP (1 item)
  int lo = 0, hi = -1;                       // REP
};
using P = std::unique_ptr<Node>;

P mk(int tag) {
  P n(new Node());
  n->tag = tag;
  return n;
}

std::string hexs(long v) {  // Python f"{v:#x}"
  char b[32];
  std::snprintf(b, sizeof b, "0x%lx", v);
  return b;
}

void put_utf8(std::string& s, uint32_t cp) {
  if (cp < 0x80) {
    s += (char)cp;
  } else if (cp < 0x800) {
    s += (char)(0xC0 | (cp >> 6));
    s += (char)(0x80 | (cp & 0x3F));
  } else if (cp < 0x10000) {
    s += (char)(0xE0 | (cp >> 12));
    s += (char)(0x80 | ((cp >> 6) & 0x3F));
    s += (char)(0x80 | (cp & 0x3F));
  } else {
    s += (char)(0xF0 | (cp >> 18));
    s += (char)(0x80 | ((cp >> 12) & 0x3F));
    s += (char)(0x80 | ((cp >> 6) & 0x3F));
    s += (char)(0x80 | (cp & 0x3F));
  }
}

// Python repr() of a one-character string (the "unexpected character" error)
std::string repr_char(uint32_t c) {
  std::string body;
  char b[16];
  const char q = c == '\'' ? '"' : '\'';
  if (c == '\\') body = "\\\\";
  else if (c == '\n') body = "\\n";
  else if (c == '\r') body = "\\r";
  else if (c == '\t') body = "\\t";
  else if (c < 0x20 || c == 0x7F || (c >= 0x80 && c < 0xA0)) {
    std::snprintf(b, sizeof b, "\\x%02x", c);
    body = b;
  } else if (c >= 0xD800 && c <= 0xDFFF) {
    std::snprintf(b, sizeof b, "\\u%04x", c);
    body = b;
  } else {
    put_utf8(body, c);
  }
  return std::string(1, q) + body + q;
}

// ---------------------------------------------------------------- scanner
enum Kind { K_EOF, K_IDENT, K_DEFINE, K_LIT, K_CLASS, K_LPAREN, K_RPAREN, K_PIPE, K_STAR, K_PLUS, K_QMARK, K_BOUNDS };
const char* kind_name(int k) {
  static const char* n[] = {"EOF", "IDENT", "DEFINE", "LITERAL", "CLASS", "LPAREN", "RPAREN", "PIPE", "STAR", "PLUS",
                            "QMARK", "BOUNDS"};
  return n[k];
}

struct ClassMember {
  uint32_t lo, hi;
  bool raw;
};

struct Tok {
  int kind;
  std::string text;                  // IDENT name / LIT bytes
  std::vector<ClassMember> members;  // CLASS
  bool negated = false;
  int lo = 0, hi = -1;               // BOUNDS (hi -1: open)
  int line, col;
};

struct Scanner {
  std::vector<uint32_t> s;
  size_t i = 0;
  int line = 1, col = 1;

  uint32_t ch(size_t k = 0) const { return i + k < s.size() ? s[i + k] : 0; }
  bool at_end(size_t k = 0) const { return i + k >= s.size(); }
  void bump(int k = 1) {
    for (int j = 0; j < k; ++j) {
      if (i < s.size() && s[i] == '\n') {
        ++line;
        col = 1;
      } else {
        ++col;
      }
      ++i;
    }
  }
  [[noreturn]] void error(const std::string& m) { throw ParseFail{m, line, col}; }

  static int hexval(uint32_t c) {
    if (c >= '0' && c <= '9') return (int)(c - '0');
    if (c >= 'a' && c <= 'f') return (int)(c - 'a' + 10);
    if (c >= 'A' && c <= 'F') return (int)(c - 'A' + 10);
    return -1;
  }

  // after a backslash: (value, denotes a raw byte)
  std::pair<uint32_t, bool> escape(bool in_class) {
    bump();
    if (at_end()) error("unterminated escape");
    const uint32_t c = ch();
    switch (c) {
      case 'n': bump(); return {0x0A, false};
      case 't': bump(); return {0x09, false};
      case 'r': bump(); return {0x0D, false};
      case '"': bump(); return {0x22, false};
      case '\\': bump(); return {0x5C, false};
      case '\'': bump(); return {0x27, false};
    }
    if (in_class && (c == ']' || c == '-' || c == '^' || c == '[')) {
      bump();
      return {c, false};
    }
    if (c == 'x' || c == 'u') {
      const int width = c == 'x' ? 2 : 4;
      uint32_t v = 0;
      bool ok = true;
      for (int k = 0; k < width; ++k) {
        const int h = at_end(1 + k) ? -1 : hexval(ch(1 + k));
        if (h < 0) ok = false;
        else v = v * 16 + (uint32_t)h;
      }
      if (!ok)
        error(std::string("\\") + (char)c + " escape needs " + (width == 2 ? "two" : "four") + " hex digits");
      bump(width + 1);
      return {v, c == 'x'};
    }
    std::string m = "unknown escape \\";
    put_utf8(m, c);
    error(m);
  }

  Tok literal() {
    Tok t;
    t.kind = K_LIT;
    t.line = line;
    t.col = col;
    bump();
    for (;;) {
      if (at_end() || ch() == '\n') throw ParseFail{"unterminated string literal", t.line, t.col};
      const uint32_t c = ch();
      if (c == '"') {
        bump();
        return t;
      }
      if (c == '\\') {
        const auto e = escape(false);
        if (e.second) {
          t.text += (char)(e.first & 0xFF);
        } else {
          if (e.first >= 0xD800 && e.first <= 0xDFFF) {
            char b[64];
            std::snprintf(b, sizeof b, "escape \\u%04X is a lone surrogate", e.first);
            throw ParseFail{b, t.line, t.col};
          }
          put_utf8(t.text, e.first);
        }
      } else {
        put_utf8(t.text, c);
        bump();
      }
    }
  }

  std::pair<uint32_t, bool> class_atom() {
    if (ch() == '\\') return escape(true);
    const uint32_t c = ch();
    bump();
    return {c, false};
  }

  Tok char_class() {
    Tok t;
    t.kind = K_CLASS;
    t.line = line;
    t.col = col;
    bump();
    if (ch() == '^' && !at_end()) {
      t.negated = true;
      bump();
    }
    for (;;) {
      if (at_end() || ch() == '\n') throw ParseFail{"unterminated character class", t.line, t.col};
      if (ch() == ']' && !t.members.empty()) {
        bump();
        return t;
      }
      auto lo = class_atom();
      auto hi = lo;
      if (!at_end() && ch() == '-' && !at_end(1) && ch(1) != ']') {
        bump();
        hi = class_atom();
      }
      if (hi.first < lo.first)
        throw ParseFail{"class range out of order: " + hexs(lo.first) + "-" + hexs(hi.first), t.line, t.col};
      t.members.push_back({lo.first, hi.first, lo.second || hi.second});
    }
  }

  Tok bounds() {
    Tok t;
    t.kind = K_BOUNDS;
    t.line = line;
    t.col = col;
    bump();
    auto number = [&](std::string& d) {
      while (!at_end() && ch() >= '0' && ch() <= '9') {
        d += (char)ch();
        bump();
      }
    };
    std::string lo_s;
    number(lo_s);
    if (lo_s.empty()) error("repeat bounds need a count");
    t.lo = std::stoi(lo_s);
    t.hi = t.lo;
    if (!at_end() && ch() == ',') {
      bump();
      std::string hi_s;
      number(hi_s);
      t.hi = hi_s.empty() ? -1 : std::stoi(hi_s);
    }
    if (at_end() || ch() != '}') error("unterminated repeat bounds");
    bump();
    return t;
  }

  static bool id0(uint32_t c) { return (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || c == '_'; }
  static bool id1(uint32_t c) { return id0(c) || (c >= '0' && c <= '9') || c == '-'; }

  std::vector<Tok> tokens() {
    std::vector<Tok> out;
    for (;;) {
      if (at_end()) {
        Tok t;
        t.kind = K_EOF;
        t.line = line;
        t.col = col;
        out.push_back(t);
        return out;
      }
      const uint32_t c = ch();
      if (c == ' ' || c == '\t' || c == '\r' || c == '\n') {
        bump();
      } else if (c == '#') {
        while (!at_end() && ch() != '\n') bump();
      } else if (id0(c)) {
        Tok t;
        t.kind = K_IDENT;
        t.line = line;
        t.col = col;
        while (!at_end() && id1(ch())) {
          t.text += (char)ch();
          bump();
        }
        out.push_back(std::move(t));
      } else if (c == ':' && ch(1) == ':' && ch(2) == '=' && !at_end(2)) {
        Tok t;
        t.kind = K_DEFINE;
        t.line = line;
        t.col = col;
        out.push_back(t);
        bump(3);
      } else if (c == '"') {
        out.push_back(literal());
      } else if (c == '[') {
        out.push_back(char_class());
      } else if (c == '(' || c == ')' || c == '|' || c == '*' || c == '+' || c == '?') {
        Tok t;
        t.kind = c == '(' ? K_LPAREN : c == ')' ? K_RPAREN : c == '|' ? K_PIPE : c == '*' ? K_STAR
                 : c == '+' ? K_PLUS : K_QMARK;
        t.line = line;
        t.col = col;
        out.push_back(t);
        bump();
      } else if (c == '{') {
        out.push_back(bounds());
      } else {
        error("unexpected character " + repr_char(c));
      }
    }
  }
};

// ---------------------------------------------------------------- UTF-8 ranges
// Byte-range sequences covering every byte string s with lo <= s <= hi
// (same length; grammar.py _cont_split).
typedef std::vector<std::pair<int, int>> Seq;
std::vector<Seq> cont_split(const std::string& lo, const std::string& hi) {
  const size_t n = lo.size();
  const int a = (uint8_t)lo[0], b = (uint8_t)hi[0];
  if (n == 1) return {Seq{{a, b}}};
  std::vector<Seq> out;
  if (a == b) {
    for (auto& rest : cont_split(lo.substr(1), hi.substr(1))) {
      Seq s{{a, a}};
      s.insert(s.end(), rest.begin(), rest.end());
      out.push_back(s);
    }
    return out;
  }
  const std::string tmin(n - 1, (char)0x80), tmax(n - 1, (char)0xBF);
  const bool first_full = lo.substr(1) == tmin, last_full = hi.substr(1) == tmax;
  const int mid_lo = first_full ? a : a + 1, mid_hi = last_full ? b : b - 1;
  if (!first_full)
    for (auto& rest : cont_split(lo.substr(1), tmax)) {
      Seq s{{a, a}};
      s.insert(s.end(), rest.begin(), rest.end());
      out.push_back(s);
    }
  if (mid_lo <= mid_hi) {
    Seq s{{mid_lo, mid_hi}};
    for (size_t k = 1; k < n; ++k) s.push_back({0x80, 0xBF});
    out.push_back(s);
  }
  if (!last_full)
    for (auto& rest : cont_split(tmin, hi.substr(1))) {
      Seq s{{b, b}};
      s.insert(s.end(), rest.begin(), rest.end());
      out.push_back(s);
    }
  return out;
}

std::vector<Seq> utf8_range_sequences(uint32_t lo, uint32_t hi) {
  static const uint32_t lim[4][2] = {{0x00, 0x7F}, {0x80, 0x7FF}, {0x800, 0xFFFF}, {0x10000, 0x10FFFF}};
  std::vector<Seq> pieces;
  const uint32_t parts[2][2] = {{lo, std::min<uint32_t>(hi, 0xD7FF)}, {std::max<uint32_t>(lo, 0xE000), hi}};
  for (auto& pr : parts) {
    if (pr[0] > pr[1]) continue;
    for (auto& l : lim) {
      const uint32_t a = std::max(pr[0], l[0]), b = std::min(pr[1], l[1]);
      if (a <= b) {
        std::string sa, sb;
        put_utf8(sa, a);
        put_utf8(sb, b);
        for (auto& s : cont_split(sa, sb)) pieces.push_back(s);
      }
    }
  }
  return pieces;
}

P bytes_node(int lo, int hi) {
  P n = mk(E_BYTES);
  n->mask.range(lo, hi);
  return n;
}

P lower_class(const Tok& t) {
  Mask byte_mask;
  std::vector<std::pair<uint32_t, uint32_t>> cps;
  for (auto& m : t.members) {
    if (m.raw || m.hi <= 0x7F) {
      if (m.hi > 0xFF) throw ParseFail{"byte escape out of range: " + hexs(m.hi), t.line, t.col};
      byte_mask.range((int)m.lo, (int)m.hi);
    } else {
      cps.push_back({m.lo, m.hi});
    }
  }
  if (t.negated) {
    if (!cps.empty()) throw ParseFail{"negated classes may only contain ASCII or \\xHH members", t.line, t.col};
    P n = mk(E_BYTES);
    for (int k = 0; k < 8; ++k) n->mask.w[k] = ~byte_mask.w[k];
    return n;
  }
  if (cps.empty()) {
    P n = mk(E_BYTES);
    n->mask = byte_mask;
    return n;
  }
  std::vector<P> alts;
  Mask cp_ascii;
  for (auto cp : cps) {
    uint32_t lo = cp.first;
    const uint32_t hi = cp.second;
    if (hi > 0x10FFFF) throw ParseFail{"code point out of range: " + hexs(hi), 0, 0};
    if (lo <= 0x7F) {
      cp_ascii.range((int)lo, 0x7F);
      lo = 0x80;
    }
    for (auto& seq : utf8_range_sequences(lo, hi)) {
      if (seq.size() == 1) {
        alts.push_back(bytes_node(seq[0].first, seq[0].second));
      } else {
        P s = mk(E_SEQ);
        for (auto& r : seq) s->items.push_back(bytes_node(r.first, r.second));
        alts.push_back(std::move(s));
      }
    }
  }
  Mask un = byte_mask;
  for (int k = 0; k < 8; ++k) un.w[k] |= cp_ascii.w[k];
  if (alts.empty() && cp_ascii.empty()) throw ParseFail{"empty character class after lowering", 0, 0};
  if (!un.empty()) {
    P b = mk(E_BYTES);
    b->mask = un;
    alts.insert(alts.begin(), std::move(b));
  }
  if (alts.size() == 1) return std::move(alts[0]);
  P a = mk(E_ALT);
  a->items = std::move(alts);
  return a;
}

// ---------------------------------------------------------------- parser
struct Parser {
  std::vector<Tok> t;
  size_t k = 0;

  const Tok& peek(size_t off = 0) const { return t[std::min(k + off, t.size() - 1)]; }
  const Tok& take() {
    const Tok& tok = t[k];
    if (tok.kind != K_EOF) ++k;
    return tok;
  }
  const Tok& expect(int kind) {
    const Tok& tok = take();
    if (tok.kind != kind)
      throw ParseFail{std::string("expected ") + kind_name(kind) + ", got " + kind_name(tok.kind), tok.line, tok.col};
    return tok;
  }

  P alternation() {
    std::vector<P> alts;
    alts.push_back(sequence());
    while (peek().kind == K_PIPE) {
      take();
      alts.push_back(sequence());
    }
    if (alts.size() == 1) return std::move(alts[0]);
    P a = mk(E_ALT);
    a->items = std::move(alts);
    return a;
  }

  P sequence() {
    std::vector<P> items;
    for (;;) {
      const int kind = peek().kind;
      if (kind == K_PIPE || kind == K_RPAREN || kind == K_EOF || (kind == K_IDENT && peek(1).kind == K_DEFINE)) break;
      items.push_back(postfix());
    }
    if (items.empty()) return mk(E_EPS);
    if (items.size() == 1) return std::move(items[0]);
    P s = mk(E_SEQ);
    s->items = std::move(items);
    return s;
  }

  P postfix() {
    P e = atom();
    for (;;) {
      const Tok& tk = peek();
      int lo, hi;
      if (tk.kind == K_STAR) {
        lo = 0; hi = -1;
      } else if (tk.kind == K_PLUS) {
        lo = 1; hi = -1;
      } else if (tk.kind == K_QMARK) {
        lo = 0; hi = 1;
      } else if (tk.kind == K_BOUNDS) {
        lo = tk.lo; hi = tk.hi;
        if (hi >= 0 && hi < lo)
          throw ParseFail{"bad repeat bounds {" + std::to_string(lo) + "," + std::to_string(hi) + "}", tk.line, tk.col};
      } else {
        return e;
      }
      P r = mk(E_REP);
      r->lo = lo;
      r->hi = hi;
      r->items.push_back(std::move(e));
      e = std::move(r);
      take();
    }
  }

  P atom() {
    const Tok& tk = take();
    switch (tk.kind) {
      case K_LIT: {
        if (tk.text.empty()) return mk(E_EPS);
        P n = mk(E_LIT);
        n->data = tk.text;
        return n;
      }
      case K_CLASS: return lower_class(tk);
      case K_IDENT: {
        P n = mk(E_REF);
        n->data = tk.text;
        return n;
      }
      case K_LPAREN: {
        P e = alternation();
        expect(K_RPAREN);
        return e;
      }
    }
    throw ParseFail{std::string("unexpected ") + kind_name(tk.kind) + " in expression", tk.line, tk.col};
  }
};

void walk(const Node* e, std::vector<const Node*>& out) {  // pre-order (grammar.py _walk)
  out.push_back(e);
  for (auto& it : e->items) walk(it.get(), out);
}

bool derives(const Node* e, const std::set<std::string>& productive) {
  switch (e->tag) {
    case E_BYTES: return !e->mask.empty();
    case E_LIT:
    case E_EPS: return true;
    case E_SEQ:
      for (auto& x : e->items)
        if (!derives(x.get(), productive)) return false;
      return true;
    case E_ALT:
      for (auto& x : e->items)
        if (derives(x.get(), productive)) return true;
      return false;
    case E_REP: return e->lo == 0 || derives(e->items[0].get(), productive);
  }
  return productive.count(e->data) > 0;
}

void emit(const Node* e, const std::map<std::string, int>& rid, std::vector<int32_t>& out) {
  switch (e->tag) {
    case E_EPS: out.push_back(E_EPS); return;
    case E_BYTES:
      out.push_back(E_BYTES);
      for (uint32_t w : e->mask.w) out.push_back((int32_t)w);
      return;
    case E_LIT:
      out.push_back(E_LIT);
      out.push_back((int32_t)e->data.size());
      for (char c : e->data) out.push_back((int32_t)(uint8_t)c);
      return;
    case E_SEQ:
    case E_ALT:
      out.push_back(e->tag);
      out.push_back((int32_t)e->items.size());
      for (auto& x : e->items) emit(x.get(), rid, out);
      return;
    case E_REP:
      out.push_back(E_REP);
      out.push_back(e->lo);
      out.push_back(e->hi);
      emit(e->items[0].get(), rid, out);
      return;
    case E_REF:
      out.push_back(E_REF);
      out.push_back(rid.at(e->data));
      return;
  }
}

std::string quote(const std::string& s) { return "'" + s + "'"; }  // repr() of an identifier

}  // namespace

struct gm_parsed {
  std::vector<int32_t> ir;
  std::string names;  // rule names, '\0'-separated
  std::vector<int64_t> name_off;
  std::string error;
};

extern "C" {

gm_status gm_grammar_parse(const uint8_t* text, int64_t len, const char* root_rule_name, gm_parsed** out,
                           gm_parse_view* view) {
  if (!out || !view || (len > 0 && !text)) {
    gm::set_error("bad parse arguments");
    return GM_ERR_INVALID;
  }
  *out = nullptr;
  std::memset(view, 0, sizeof(*view));
  auto* g = new gm_parsed();
  try {
    Scanner sc;
    // decode UTF-8 (Python encodes the str with surrogatepass)
    for (int64_t i = 0; i < len;) {
      const uint8_t c = text[i];
      uint32_t cp;
      int n;
      if (c < 0x80) { cp = c; n = 1; }
      else if ((c >> 5) == 6) { cp = c & 0x1F; n = 2; }
      else if ((c >> 4) == 14) { cp = c & 0x0F; n = 3; }
      else { cp = c & 0x07; n = 4; }
      for (int k = 1; k < n && i + k < len; ++k) cp = (cp << 6) | (text[i + k] & 0x3F);
      sc.s.push_back(cp);
      i += n;
    }
    Parser ps;
    ps.t = sc.tokens();
    struct Raw {
      std::string name;
      P body;
      int line, col;
    };
    std::vector<Raw> raw;
    while (ps.peek().kind != K_EOF) {
      const Tok& name = ps.expect(K_IDENT);
      Raw r{name.text, nullptr, name.line, name.col};
      ps.expect(K_DEFINE);
      r.body = ps.alternation();
      raw.push_back(std::move(r));
    }
    if (raw.empty()) throw ParseFail{"empty grammar", 0, 0};
    std::map<std::string, int> rid;
    for (auto& r : raw) {
      if (rid.count(r.name)) throw ParseFail{"duplicate rule name " + quote(r.name), r.line, r.col};
      rid.emplace(r.name, (int)rid.size());
    }
    for (auto& r : raw) {
      std::vector<const Node*> nodes;
      walk(r.body.get(), nodes);
      for (const Node* e : nodes)
        if (e->tag == E_REF && !rid.count(e->data))
          throw ParseFail{"undefined rule reference " + quote(e->data) + " in " + quote(r.name), r.line, r.col};
    }
    std::set<std::string> productive;
    for (bool grew = true; grew;) {
      grew = false;
      for (auto& r : raw)
        if (!productive.count(r.name) && derives(r.body.get(), productive)) {
          productive.insert(r.name);
          grew = true;
        }
    }
    std::string dead;
    for (auto& r : raw)
      if (!productive.count(r.name)) dead += (dead.empty() ? "" : ", ") + r.name;
    if (!dead.empty()) throw ParseFail{"rules derive no strings (empty language): " + dead, 0, 0};
    for (auto& r : raw) {
      std::vector<const Node*> nodes;
      walk(r.body.get(), nodes);
      for (const Node* e : nodes)
        if (e->tag == E_BYTES && e->mask.empty()) throw ParseFail{"character class matches no byte", 0, 0};
    }
    int root;
    if (root_rule_name) {
      auto it = rid.find(root_rule_name);
      if (it == rid.end()) throw ParseFail{std::string("root rule ") + quote(root_rule_name) + " is not defined", 0, 0};
      root = it->second;
    } else {
      auto it = rid.find("root");
      root = it != rid.end() ? it->second : 0;
    }
    for (auto& r : raw) {
      emit(r.body.get(), rid, g->ir);
      g->name_off.push_back((int64_t)g->names.size());
      g->names += r.name;
      g->names += '\0';
    }
    g->name_off.push_back((int64_t)g->names.size());
    view->ir = g->ir.data();
    view->ir_len = (int64_t)g->ir.size();
    view->n_rules = (int32_t)raw.size();
    view->root_rule = root;
    view->names = g->names.data();
    view->name_off = g->name_off.data();
    *out = g;
    return GM_OK;
  } catch (const ParseFail& f) {
    g->error = f.msg;
    view->error = g->error.c_str();
    view->err_line = f.line;
    view->err_col = f.col;
    std::string full = f.msg;
    if (f.line) full += " (line " + std::to_string(f.line) + ", column " + std::to_string(f.col) + ")";
    gm::set_error(full);
    *out = g;  // keeps the message alive for the view
    return GM_ERR_GRAMMAR;
  } catch (const std::exception& e) {
    delete g;
    gm::set_error(std::string("grammar parse: ") + e.what());
    return GM_ERR_INVALID;
  }
}

void gm_grammar_parse_release(gm_parsed* g) { delete g; }

}  // extern "C"

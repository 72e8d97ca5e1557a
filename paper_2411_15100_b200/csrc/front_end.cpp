// Native host front end: grammar expression IR -> device automaton tables
// (gm_front_end_build, include/gmask.h).  Replaces the reference's PDA
// construction and optimisation passes (REF pda.py:246-535) and the
// FollowFsa precompute (REF cache.py:241-333) — SURVEY §8f rank 2.
//
// It is the C++ form of paper_2411_15100_b200/automaton.py (the executable
// specification, kept for the CPU tests that compare the two table sets
// array for array): per-rule epsilon-NFA -> subset construction -> Moore
// minimisation (canonical BFS numbering), inlining of small call-free rules
// to fixpoint, the silent-move pre-closure per node, and the follow DFA.
// Every numbering is canonical (sorted symbol order), so the tables are
// identical to the Python specification's.
//
// IR (int32, prefix order): EPS=0 | BYTES=1 m0..m7 (256-bit mask, LSW first)
// | LIT=2 len b... | SEQ=3 k items | ALT=4 k items | REP=5 lo hi(-1: inf) item
// | REF=6 rid.  Rules are consecutive bodies, rule ids = source order.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "gmask.h"

namespace gm {
void set_error(const std::string& msg);
}

namespace {

struct Bits {
  uint64_t w[4] = {0, 0, 0, 0};
  void set(int b) { w[b >> 6] |= 1ull << (b & 63); }
  bool test(int b) const { return (w[b >> 6] >> (b & 63)) & 1; }
  bool any() const { return w[0] | w[1] | w[2] | w[3]; }
  bool operator<(const Bits& o) const {
    for (int i = 3; i >= 0; --i)
      if (w[i] != o.w[i]) return w[i] < o.w[i];
    return false;
  }
  bool operator==(const Bits& o) const { return !std::memcmp(w, o.w, sizeof w); }
};

struct GrammarFail : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CapFail : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- IR
enum { E_EPS = 0, E_BYTES = 1, E_LIT = 2, E_SEQ = 3, E_ALT = 4, E_REP = 5, E_REF = 6 };

struct Ir {
  const int32_t* p;
  int64_t n;
  int64_t skip(int64_t i) const {  // index past the expression at i
    if (i >= n) throw GrammarFail("truncated grammar IR");
    switch (p[i]) {
      case E_EPS: return i + 1;
      case E_BYTES: return i + 9;
      case E_LIT: return i + 2 + p[i + 1];
      case E_SEQ:
      case E_ALT: {
        int64_t j = i + 2;
        for (int k = 0; k < p[i + 1]; ++k) j = skip(j);
        return j;
      }
      case E_REP: return skip(i + 3);
      case E_REF: return i + 2;
    }
    throw GrammarFail("bad grammar IR tag");
  }
};

Bits bytes_mask(const int32_t* m) {
  Bits b;
  for (int i = 0; i < 8; ++i) {
    const uint64_t v = (uint32_t)m[i];
    b.w[i >> 1] |= v << (32 * (i & 1));
  }
  return b;
}

// ---------------------------------------------------------------- automata
struct Nfa {
  std::vector<std::vector<std::pair<Bits, int>>> byte;  // (class set, dst)
  std::vector<std::vector<std::pair<int, int>>> call;   // (rid, dst)
  std::vector<std::vector<int>> eps;
  int start = 0;
  std::vector<int> finals;
  int add() {
    byte.emplace_back();
    call.emplace_back();
    eps.emplace_back();
    return (int)byte.size() - 1;
  }
};

struct Dfa {
  std::vector<std::vector<std::pair<int, int>>> trans;  // (class, dst), ascending class
  std::vector<std::vector<std::pair<int, int>>> calls;  // (rid, dst), ascending rid
  std::vector<char> finals;
  int start = 0;
  int size() const { return (int)trans.size(); }
};

struct Builder {
  const Ir& ir;
  const uint8_t* cls;  // byte -> class
  Nfa a;
  std::map<Bits, Bits> memo;
  Builder(const Ir& ir_, const uint8_t* c) : ir(ir_), cls(c) {}
  Bits cset(const Bits& mask) {
    auto it = memo.find(mask);
    if (it != memo.end()) return it->second;
    Bits out;
    for (int b = 0; b < 256; ++b)
      if (mask.test(b)) out.set(cls[b]);
    memo[mask] = out;
    return out;
  }
  int emit(int64_t i, int s) {
    const int32_t* p = ir.p;
    switch (p[i]) {
      case E_EPS: return s;
      case E_BYTES: {
        const int t = a.add();
        a.byte[s].push_back({cset(bytes_mask(p + i + 1)), t});
        return t;
      }
      case E_LIT: {
        for (int k = 0; k < p[i + 1]; ++k) {
          Bits m;
          m.set(p[i + 2 + k] & 0xFF);
          const int t = a.add();
          a.byte[s].push_back({cset(m), t});
          s = t;
        }
        return s;
      }
      case E_SEQ: {
        int64_t j = i + 2;
        for (int k = 0; k < p[i + 1]; ++k) {
          s = emit(j, s);
          j = ir.skip(j);
        }
        return s;
      }
      case E_ALT: {
        const int join = a.add();
        int64_t j = i + 2;
        for (int k = 0; k < p[i + 1]; ++k) {
          const int head = a.add();
          a.eps[s].push_back(head);
          const int e = emit(j, head);
          a.eps[e].push_back(join);
          j = ir.skip(j);
        }
        return join;
      }
      case E_REP: {
        const int lo = p[i + 1], hi = p[i + 2];
        const int64_t item = i + 3;
        for (int k = 0; k < lo; ++k) {
          const int head = a.add();
          a.eps[s].push_back(head);
          s = emit(item, head);
        }
        if (hi < 0) {
          const int loop = a.add();
          a.eps[s].push_back(loop);
          const int body = a.add();
          a.eps[loop].push_back(body);
          const int e = emit(item, body);
          a.eps[e].push_back(loop);
          return loop;
        }
        const int exit_ = a.add();
        a.eps[s].push_back(exit_);
        for (int k = 0; k < hi - lo; ++k) {
          const int head = a.add();
          a.eps[s].push_back(head);
          s = emit(item, head);
          a.eps[s].push_back(exit_);
        }
        return exit_;
      }
      case E_REF: {
        const int t = a.add();
        a.call[s].push_back({p[i + 1], t});
        return t;
      }
    }
    throw GrammarFail("bad grammar IR tag");
  }
};

struct VecHash {
  size_t operator()(const std::vector<int>& v) const {
    uint64_t h = 1469598103934665603ull;
    for (int x : v) h = (h ^ (uint32_t)x) * 1099511628211ull;
    return (size_t)h;
  }
};

std::vector<int> eps_close(const Nfa& a, std::vector<int> states, std::vector<char>& mark) {
  std::vector<int> work = states;
  for (int u : states) mark[u] = 1;
  while (!work.empty()) {
    const int u = work.back();
    work.pop_back();
    for (int v : a.eps[u])
      if (!mark[v]) {
        mark[v] = 1;
        states.push_back(v);
        work.push_back(v);
      }
  }
  for (int u : states) mark[u] = 0;
  std::sort(states.begin(), states.end());
  return states;
}

// subset construction over max_states states (caught: eps_free fallback)
struct DfaLimit : GrammarFail {
  using GrammarFail::GrammarFail;
};

Dfa determinize(const Nfa& a, int n_classes, int max_states) {
  std::vector<char> mark(a.byte.size(), 0), is_final(a.byte.size(), 0);
  for (int f : a.finals) is_final[f] = 1;
  std::unordered_map<std::vector<int>, int, VecHash> ids;
  std::vector<std::vector<int>> order;
  auto start = eps_close(a, {a.start}, mark);
  ids.emplace(start, 0);
  order.push_back(start);
  Dfa d;
  std::vector<std::vector<int>> by_class(n_classes);
  std::map<int, std::vector<int>> by_rule;
  for (size_t i = 0; i < order.size(); ++i) {
    const std::vector<int> S = order[i];
    for (auto& v : by_class) v.clear();
    by_rule.clear();
    bool fin = false;
    for (int u : S) {
      fin |= is_final[u];
      for (auto& e : a.byte[u])
        for (int c = 0; c < n_classes; ++c)
          if (e.first.test(c)) by_class[c].push_back(e.second);
      for (auto& e : a.call[u]) by_rule[e.first].push_back(e.second);
    }
    auto target = [&](const std::vector<int>& vs) {
      std::vector<int> T = eps_close(a, vs, mark);
      auto it = ids.find(T);
      if (it != ids.end()) return it->second;
      const int id = (int)order.size();
      ids.emplace(T, id);
      order.push_back(std::move(T));
      if ((int)order.size() > max_states)
        throw DfaLimit("rule automaton exceeds " + std::to_string(max_states) +
                       " states after determinisation");
      return id;
    };
    std::vector<std::pair<int, int>> row, crow;
    for (int c = 0; c < n_classes; ++c) {
      if (by_class[c].empty()) continue;
      std::vector<int> vs = by_class[c];
      std::sort(vs.begin(), vs.end());
      vs.erase(std::unique(vs.begin(), vs.end()), vs.end());
      row.push_back({c, target(vs)});
    }
    for (auto& kv : by_rule) {
      std::vector<int> vs = kv.second;
      std::sort(vs.begin(), vs.end());
      vs.erase(std::unique(vs.begin(), vs.end()), vs.end());
      crow.push_back({kv.first, target(vs)});
    }
    d.trans.push_back(std::move(row));
    d.calls.push_back(std::move(crow));
    d.finals.push_back(fin);
  }
  return d;
}

// Fallback when the subset construction of a rule would exceed
// max_dfa_states (e.g. `[ab]* "a" [ab]{20}`, 2^21 subsets): the rule keeps
// an epsilon-free NFA instead.  A node per NFA state reached by a byte or
// call edge (plus the start); its moves are the edges of every state of its
// epsilon closure, so a (node, class) may lead to several targets and the
// walkers carry one stack per live target — what the reference's Thompson
// automaton does at run time (REF pda.py:246-329), bounded by the same
// 4096-stack cap.  The language is unchanged, so masks are too.
Dfa eps_free(const Nfa& a, int n_classes) {
  std::vector<char> mark(a.byte.size(), 0), is_final(a.byte.size(), 0);
  for (int f : a.finals) is_final[f] = 1;
  std::vector<int> id(a.byte.size(), -1), order{a.start};
  id[a.start] = 0;
  auto node = [&](int v) {
    if (id[v] < 0) {
      id[v] = (int)order.size();
      order.push_back(v);
    }
    return id[v];
  };
  Dfa d;
  for (size_t i = 0; i < order.size(); ++i) {
    const std::vector<int> C = eps_close(a, {order[i]}, mark);
    std::vector<std::pair<int, int>> row, crow;
    bool fin = false;
    for (int u : C) {
      fin |= is_final[u];
      for (auto& e : a.byte[u])
        for (int c = 0; c < n_classes; ++c)
          if (e.first.test(c)) row.push_back({c, node(e.second)});
      for (auto& e : a.call[u]) crow.push_back({e.first, node(e.second)});
    }
    std::sort(row.begin(), row.end());
    row.erase(std::unique(row.begin(), row.end()), row.end());
    std::sort(crow.begin(), crow.end());
    crow.erase(std::unique(crow.begin(), crow.end()), crow.end());
    d.trans.push_back(std::move(row));
    d.calls.push_back(std::move(crow));
    d.finals.push_back(fin);
  }
  return d;
}

Dfa det_or_nfa(const Nfa& a, int n_classes, int max_states) {
  try {
    return determinize(a, n_classes, max_states);
  } catch (const DfaLimit&) {
    return eps_free(a, n_classes);
  }
}

Dfa minimize(const Dfa& d) {
  const int n = d.size();
  std::vector<int> block(n), nxt(n);
  {
    std::map<std::vector<int>, int> keys;
    for (int s = 0; s < n; ++s) {
      std::vector<int> k{d.finals[s]};
      k.push_back((int)d.trans[s].size());
      for (auto& e : d.trans[s]) k.push_back(e.first);
      for (auto& e : d.calls[s]) k.push_back(e.first);
      block[s] = keys.emplace(k, (int)keys.size()).first->second;
    }
    int nb = (int)keys.size();
    while (true) {
      std::unordered_map<std::vector<int>, int, VecHash> k2;
      for (int s = 0; s < n; ++s) {
        std::vector<int> k{block[s], (int)d.trans[s].size()};
        for (auto& e : d.trans[s]) { k.push_back(e.first); k.push_back(block[e.second]); }
        for (auto& e : d.calls[s]) { k.push_back(e.first); k.push_back(block[e.second]); }
        nxt[s] = k2.emplace(k, (int)k2.size()).first->second;
      }
      if ((int)k2.size() == nb) break;
      block.swap(nxt);
      nb = (int)k2.size();
    }
  }
  std::vector<int> rep(n, -1);
  for (int s = 0; s < n; ++s)
    if (rep[block[s]] < 0) rep[block[s]] = s;
  std::vector<int> order{block[d.start]};
  std::vector<int> seen(n, -1);
  seen[block[d.start]] = 0;
  for (size_t i = 0; i < order.size(); ++i) {
    const int s = rep[order[i]];
    for (auto& e : d.trans[s])
      if (seen[block[e.second]] < 0) { seen[block[e.second]] = (int)order.size(); order.push_back(block[e.second]); }
    for (auto& e : d.calls[s])
      if (seen[block[e.second]] < 0) { seen[block[e.second]] = (int)order.size(); order.push_back(block[e.second]); }
  }
  Dfa m;
  for (int b : order) {
    const int s = rep[b];
    std::vector<std::pair<int, int>> t, c;
    for (auto& e : d.trans[s]) t.push_back({e.first, seen[block[e.second]]});
    for (auto& e : d.calls[s]) c.push_back({e.first, seen[block[e.second]]});
    m.trans.push_back(std::move(t));
    m.calls.push_back(std::move(c));
    m.finals.push_back(d.finals[s]);
  }
  return m;
}

Nfa dfa_as_nfa(const Dfa& d) {
  Nfa a;
  for (int s = 0; s < d.size(); ++s) a.add();
  for (int s = 0; s < d.size(); ++s) {
    for (auto& e : d.trans[s]) {
      Bits b;
      b.set(e.first);
      a.byte[s].push_back({b, e.second});
    }
    for (auto& e : d.calls[s]) a.call[s].push_back(e);
    if (d.finals[s]) a.finals.push_back(s);
  }
  a.start = d.start;
  return a;
}

Nfa inline_into(const Dfa& host, const std::map<int, const Dfa*>& callees) {
  Nfa a = dfa_as_nfa(host);
  const int base = host.size();
  for (int s = 0; s < base; ++s) {
    std::vector<std::pair<int, int>> keep;
    const auto calls = a.call[s];
    for (auto& e : calls) {
      auto it = callees.find(e.first);
      if (it == callees.end()) {
        keep.push_back(e);
        continue;
      }
      const Dfa& sub = *it->second;
      const int off = a.add();
      for (int q = 1; q < sub.size(); ++q) a.add();
      for (int q = 0; q < sub.size(); ++q) {
        for (auto& te : sub.trans[q]) {
          Bits b;
          b.set(te.first);
          a.byte[off + q].push_back({b, off + te.second});
        }
        for (auto& ce : sub.calls[q]) a.call[off + q].push_back({ce.first, off + ce.second});
        if (sub.finals[q]) a.eps[off + q].push_back(e.second);
      }
      a.eps[s].push_back(off + sub.start);
    }
    a.call[s] = keep;
  }
  return a;
}

bool has_calls(const Dfa& d) {
  for (auto& c : d.calls)
    if (!c.empty()) return true;
  return false;
}

// ---------------------------------------------------------------- result
struct Result {
  int32_t n_nodes = 0, n_rules = 0, n_classes = 0, start_node = 0, root_rule = 0, n_fstates = 0;
  std::vector<uint8_t> byte_class;
  std::vector<int32_t> trans_off, trans, push_pool, node_rule, cache_keys, follow_start, follow_next, kept;
  std::vector<uint8_t> node_flags;
  // the per-rule DFAs before the pre-closure (bundle export): per node
  // (symbol, dst) with symbol >= 0 a byte class, < 0 a call of rule -(sym+1)
  std::vector<int32_t> raw_off, raw, rule_start;
  std::vector<uint8_t> finals;
};

void build(const Ir& ir, int32_t n_rules_in, int32_t root_in, const gm_fe_options& o, Result& R) {
  // rule bodies
  std::vector<int64_t> body(n_rules_in);
  {
    int64_t i = 0;
    for (int r = 0; r < n_rules_in; ++r) {
      body[r] = i;
      i = ir.skip(i);
    }
    if (i != ir.n) throw GrammarFail("grammar IR length mismatch");
  }
  // byte classes: coarsest partition refining every mask
  std::vector<Bits> masks;
  for (int64_t i = 0; i < ir.n;) {
    const int32_t tag = ir.p[i];
    if (tag == E_BYTES) {
      masks.push_back(bytes_mask(ir.p + i + 1));
      i += 9;
    } else if (tag == E_LIT) {
      for (int k = 0; k < ir.p[i + 1]; ++k) {
        Bits b;
        b.set(ir.p[i + 2 + k] & 0xFF);
        masks.push_back(b);
      }
      i += 2 + ir.p[i + 1];
    } else if (tag == E_SEQ || tag == E_ALT) {
      i += 2;
    } else if (tag == E_REP) {
      i += 3;
    } else if (tag == E_REF) {
      i += 2;
    } else if (tag == E_EPS) {
      i += 1;
    } else {
      throw GrammarFail("bad grammar IR tag");
    }
  }
  std::sort(masks.begin(), masks.end());
  masks.erase(std::unique(masks.begin(), masks.end()), masks.end());
  std::vector<int> cls(256, 0);
  for (const Bits& m : masks) {
    std::map<std::pair<int, int>, int> remap;
    std::vector<int> nxt(256);
    for (int b = 0; b < 256; ++b) nxt[b] = remap.emplace(std::make_pair(cls[b], (int)m.test(b)), (int)remap.size()).first->second;
    cls = nxt;
  }
  std::vector<int> first(256, -1);
  int n_classes = 0;
  for (int b = 0; b < 256; ++b)
    if (first[cls[b]] < 0) first[cls[b]] = n_classes++;
  R.byte_class.resize(256);
  for (int b = 0; b < 256; ++b) R.byte_class[b] = (uint8_t)first[cls[b]];
  R.n_classes = n_classes;

  if (!o.determinize) throw GrammarFail("determinize=False is not supported by the device tables");
  std::vector<Dfa> dfas(n_rules_in);
  for (int r = 0; r < n_rules_in; ++r) {
    Builder bld(ir, R.byte_class.data());
    bld.a.start = bld.a.add();
    bld.a.finals = {bld.emit(body[r], bld.a.start)};
    dfas[r] = minimize(det_or_nfa(bld.a, n_classes, o.max_dfa_states));
  }
  if (o.inline_rules) {
    // a host whose inlining was refused (too many states / DFA limit) is not
    // retried while neither it nor any of its targets has changed (version
    // counters): the retry would refuse again
    std::vector<int64_t> version(n_rules_in, 0);
    std::vector<std::vector<int64_t>> refused(n_rules_in);
    for (int pass = 0; pass < 64; ++pass) {
      std::vector<char> inl(n_rules_in, 0);
      std::vector<Dfa> snap(n_rules_in);
      const std::vector<int64_t> snap_version = version;
      for (int r = 0; r < n_rules_in; ++r)
        if (!has_calls(dfas[r]) && dfas[r].size() <= o.inline_max_rule_states) {
          inl[r] = 1;
          snap[r] = dfas[r];
        }
      if (o.inline_calls) {
        // single-live-caller rules with calls (automaton.py build_tables)
        std::vector<std::set<int>> callers(n_rules_in);
        std::vector<char> seen(n_rules_in, 0);
        std::vector<int> work{root_in};
        seen[root_in] = 1;
        while (!work.empty()) {
          const int h = work.back();
          work.pop_back();
          for (auto& cs : dfas[h].calls)
            for (auto& e : cs) {
              callers[e.first].insert(h);
              if (!seen[e.first]) { seen[e.first] = 1; work.push_back(e.first); }
            }
        }
        for (int r = 0; r < n_rules_in; ++r) {
          if (!seen[r] || inl[r] || r == root_in || callers[r].size() != 1 || callers[r].count(r)) continue;
          if (dfas[r].size() <= o.inline_max_result_states) {
            inl[r] = 1;
            snap[r] = dfas[r];
          }
        }
      }
      bool changed = false;
      for (int host = 0; host < n_rules_in; ++host) {
        std::map<int, const Dfa*> targets;
        for (auto& cs : dfas[host].calls)
          for (auto& e : cs)
            if (inl[e.first] && e.first != host) targets[e.first] = &snap[e.first];
        if (targets.empty()) continue;
        std::vector<int64_t> sig{version[host]};
        for (auto& kv : targets) {
          sig.push_back(kv.first);
          sig.push_back(snap_version[kv.first]);
        }
        if (sig == refused[host]) continue;
        Dfa nd;
        try {
          nd = minimize(determinize(inline_into(dfas[host], targets), n_classes, o.max_dfa_states));
        } catch (const DfaLimit&) {
          refused[host] = sig;
          continue;  // inlining here would blow the subset construction up: keep the calls
        }
        if (nd.size() > o.inline_max_result_states) {
          refused[host] = sig;
          continue;
        }
        dfas[host] = std::move(nd);
        ++version[host];
        changed = true;
      }
      if (!changed) break;
    }
  }
  // rules reachable from the root
  std::vector<char> live(n_rules_in, 0);
  std::vector<int> work{root_in};
  live[root_in] = 1;
  while (!work.empty()) {
    const int r = work.back();
    work.pop_back();
    for (auto& cs : dfas[r].calls)
      for (auto& e : cs)
        if (!live[e.first]) { live[e.first] = 1; work.push_back(e.first); }
  }
  std::vector<int> new_rid(n_rules_in, -1), offset(n_rules_in, 0);
  int n_nodes = 0;
  for (int r = 0; r < n_rules_in; ++r)
    if (live[r]) {
      new_rid[r] = (int)R.kept.size();
      R.kept.push_back(r);
      offset[r] = n_nodes;
      n_nodes += dfas[r].size();
    }
  const int n_rules = (int)R.kept.size();
  std::vector<int> node_rule(n_nodes), rule_start(n_rules);
  std::vector<std::vector<std::pair<int, int>>> trans_n(n_nodes), calls_n(n_nodes);
  std::vector<char> final_n(n_nodes);
  for (int r : R.kept) {
    const Dfa& d = dfas[r];
    const int o0 = offset[r];
    rule_start[new_rid[r]] = o0 + d.start;
    for (int s = 0; s < d.size(); ++s) {
      node_rule[o0 + s] = new_rid[r];
      for (auto& e : d.trans[s]) trans_n[o0 + s].push_back({e.first, o0 + e.second});
      for (auto& e : d.calls[s]) calls_n[o0 + s].push_back({new_rid[e.first], o0 + e.second});
      std::sort(calls_n[o0 + s].begin(), calls_n[o0 + s].end());
      final_n[o0 + s] = d.finals[s];
    }
  }
  const int root_n = new_rid[root_in];
  const int start_node = rule_start[root_n];
  R.raw_off.assign(1, 0);
  for (int u = 0; u < n_nodes; ++u) {
    for (auto& e : trans_n[u]) { R.raw.push_back(e.first); R.raw.push_back(e.second); }
    for (auto& e : calls_n[u]) { R.raw.push_back(-(e.first + 1)); R.raw.push_back(e.second); }
    R.raw_off.push_back((int32_t)(R.raw.size() / 2));
    R.finals.push_back((uint8_t)final_n[u]);
  }
  R.rule_start.assign(rule_start.begin(), rule_start.end());
  std::vector<char> dead_end(n_nodes);
  for (int u = 0; u < n_nodes; ++u) dead_end[u] = final_n[u] && trans_n[u].empty() && calls_n[u].empty();

  // silent-move pre-closure per node
  std::vector<char> pop_flag(n_nodes, 0);
  std::map<std::vector<int>, int> push_off;
  push_off[{}] = 0;
  std::vector<int32_t> push_pool;
  std::vector<int64_t> trans_off((size_t)n_nodes * n_classes + 1, 0);
  std::vector<int32_t> trans_flat;
  std::vector<char> is_key(n_nodes, 0);
  is_key[start_node] = 1;
  typedef std::pair<std::vector<int>, int> St;
  std::vector<std::vector<St>> per_class(n_classes);
  for (int u = 0; u < n_nodes; ++u) {
    std::map<St, char> seen;  // ordered: sorted(seen)
    std::vector<St> wk;
    seen[St({}, u)] = 1;
    wk.push_back(St({}, u));
    while (!wk.empty()) {
      St cur = wk.back();
      wk.pop_back();
      const std::vector<int>& P = cur.first;
      const int m = cur.second;
      std::vector<St> nx;
      for (auto& e : calls_n[m]) {
        std::vector<int> PP = P;
        PP.push_back(e.second);
        nx.push_back(St(PP, rule_start[e.first]));
      }
      if (final_n[m]) {
        if (!P.empty()) {
          std::vector<int> PP(P.begin(), P.end() - 1);
          nx.push_back(St(PP, P.back()));
        } else {
          pop_flag[u] = 1;
        }
      }
      for (auto& st : nx)
        if (seen.emplace(st, 1).second) {
          wk.push_back(st);
          if ((int64_t)seen.size() > o.state_cap)
            throw CapFail("branch set exceeded cap of " + std::to_string(o.state_cap));
        }
    }
    for (auto& v : per_class) v.clear();  // reused across nodes (no per-node allocation)
    for (auto& kv : seen) {
      const std::vector<int>& P = kv.first.first;
      const int m = kv.first.second;
      for (auto& e : trans_n[m]) {
        std::vector<int> PP = P;
        int d = e.second;
        while (dead_end[d] && !PP.empty()) {
          d = PP.back();
          PP.pop_back();
        }
        auto& lst = per_class[e.first];
        const St x(PP, d);
        if (std::find(lst.begin(), lst.end(), x) == lst.end()) lst.push_back(x);
      }
    }
    for (int c = 0; c < n_classes; ++c) {
      trans_off[(size_t)u * n_classes + c] = (int64_t)trans_flat.size() / 2;
      auto& lst = per_class[c];
      if (lst.size() > 1)
        std::sort(lst.begin(), lst.end(), [](const St& a, const St& b) {
        if (a.second != b.second) return a.second < b.second;
        return a.first < b.first;
      });
      for (auto& x : lst) {
        if (x.first.size() > 255) throw CapFail("push run longer than 255 frames");
        auto it = push_off.find(x.first);
        int off;
        if (it == push_off.end()) {
          off = (int)push_pool.size();
          push_off.emplace(x.first, off);
          push_pool.insert(push_pool.end(), x.first.begin(), x.first.end());
          if (push_pool.size() >= (1u << 24)) throw CapFail("push pool exceeds 16M entries");
        } else {
          off = it->second;
        }
        trans_flat.push_back(x.second);
        trans_flat.push_back((int32_t)((uint32_t)off | ((uint32_t)x.first.size() << 24)));
        is_key[x.second] = 1;
        for (int q : x.first) is_key[q] = 1;
      }
    }
  }
  trans_off[(size_t)n_nodes * n_classes] = (int64_t)trans_flat.size() / 2;
  if (trans_flat.size() / 2 > (size_t)INT32_MAX) throw CapFail("transition table too large");

  R.n_nodes = n_nodes;
  R.n_rules = n_rules;
  R.start_node = start_node;
  R.root_rule = root_n;
  R.trans_off.assign(trans_off.begin(), trans_off.end());
  R.trans = std::move(trans_flat);
  R.push_pool = push_pool.empty() ? std::vector<int32_t>{0} : push_pool;
  R.node_rule.assign(node_rule.begin(), node_rule.end());
  R.node_flags.resize(n_nodes);
  for (int u = 0; u < n_nodes; ++u)
    R.node_flags[u] = (uint8_t)((pop_flag[u] ? GM_NODE_POP : 0) | (dead_end[u] ? GM_NODE_DEAD_END : 0));
  for (int k = 0; k < n_nodes; ++k)
    if (is_key[k] && !(dead_end[k] && node_rule[k] != root_n)) R.cache_keys.push_back(k);

  // follow automaton (context expansion)
  R.follow_start.assign(n_rules, GM_FOLLOW_ANY);
  if (!o.ctx_expansion) {
    R.follow_next.assign(n_classes, 0);
    R.n_fstates = 0;
    return;
  }
  const int END = -1;
  std::vector<std::vector<int>> seeds(n_rules);
  for (int u = 0; u < n_nodes; ++u)
    for (auto& e : calls_n[u]) seeds[e.first].push_back(e.second);
  for (auto& s : seeds) {
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
  }
  std::vector<char> mark(n_nodes + 1, 0);  // index node + 1 (END = 0)
  auto expand = [&](const std::vector<int>& S, bool& wild) {
    std::vector<int> seen;
    std::vector<int> wk;
    wild = false;
    for (int s : S)
      if (!mark[s + 1]) {
        mark[s + 1] = 1;
        seen.push_back(s);
        if (s != END) wk.push_back(s);
      }
    while (!wk.empty()) {
      const int s = wk.back();
      wk.pop_back();
      if (!calls_n[s].empty()) {
        wild = true;
        continue;
      }
      if (final_n[s]) {
        const int r = node_rule[s];
        for (int t : seeds[r])
          if (!mark[t + 1]) {
            mark[t + 1] = 1;
            seen.push_back(t);
            wk.push_back(t);
          }
        if (r == root_n && !mark[0]) {
          mark[0] = 1;
          seen.push_back(END);
        }
      }
    }
    for (int s : seen) mark[s + 1] = 0;
    std::sort(seen.begin(), seen.end());
    return seen;
  };
  std::map<std::vector<int>, int> fids;
  std::vector<std::vector<int>> forder;
  auto intern = [&](const std::vector<int>& S, bool wild) -> int {
    if (wild) return GM_FOLLOW_ANY;
    if (S.empty()) return GM_FOLLOW_DEAD;
    auto it = fids.find(S);
    if (it != fids.end()) return it->second;
    if ((int)forder.size() >= o.max_follow_states) return GM_FOLLOW_ANY;  // sound over-approximation
    const int id = (int)forder.size();
    fids.emplace(S, id);
    forder.push_back(S);
    return id;
  };
  for (int r = 0; r < n_rules; ++r) {
    std::vector<int> seed = seeds[r];
    if (r == root_n) seed.push_back(END);
    if (seed.empty()) {
      R.follow_start[r] = GM_FOLLOW_ANY;
      continue;
    }
    bool wild;
    const std::vector<int> S = expand(seed, wild);
    R.follow_start[r] = intern(S, wild);
  }
  std::vector<int32_t> rows;
  for (size_t i = 0; i < forder.size(); ++i) {
    const std::vector<int> S = forder[i];
    std::vector<std::vector<int>> by_class(n_classes);
    for (int s : S) {
      if (s == END) continue;
      for (auto& e : trans_n[s]) by_class[e.first].push_back(e.second);
    }
    std::vector<int32_t> row(n_classes, GM_FOLLOW_DEAD);
    for (int c = 0; c < n_classes; ++c) {
      if (by_class[c].empty()) continue;
      bool wild;
      const std::vector<int> T = expand(by_class[c], wild);
      row[c] = intern(T, wild);
    }
    rows.insert(rows.end(), row.begin(), row.end());
  }
  if (rows.empty()) rows.assign(n_classes, GM_FOLLOW_DEAD);
  R.follow_next = std::move(rows);
  R.n_fstates = (int32_t)forder.size();
}

}  // namespace

struct gm_front_end {
  Result r;
};

extern "C" gm_status gm_front_end_build(const int32_t* ir, int64_t ir_len, int32_t n_rules, int32_t root_rule,
                                        const gm_fe_options* opts, gm_front_end** out, gm_fe_tables* view) {
  if (!ir || ir_len <= 0 || n_rules <= 0 || root_rule < 0 || root_rule >= n_rules || !opts || !out || !view) {
    gm::set_error("bad front-end arguments");
    return GM_ERR_INVALID;
  }
  gm_front_end* fe = new gm_front_end();
  try {
    Ir x{ir, ir_len};
    build(x, n_rules, root_rule, *opts, fe->r);
  } catch (const CapFail& e) {
    delete fe;
    gm::set_error(e.what());
    return GM_ERR_STATE_CAP;
  } catch (const GrammarFail& e) {
    delete fe;
    gm::set_error(e.what());
    return GM_ERR_GRAMMAR;
  } catch (const std::exception& e) {
    delete fe;
    gm::set_error(std::string("front end: ") + e.what());
    return GM_ERR_OOM;
  }
  const Result& R = fe->r;
  view->n_nodes = R.n_nodes;
  view->n_rules = R.n_rules;
  view->n_classes = R.n_classes;
  view->start_node = R.start_node;
  view->root_rule = R.root_rule;
  view->n_trans = (int32_t)(R.trans.size() / 2);
  view->n_push = (int32_t)R.push_pool.size();
  view->n_keys = (int32_t)R.cache_keys.size();
  view->n_fstates = R.n_fstates;
  view->byte_class = R.byte_class.data();
  view->trans_off = R.trans_off.data();
  view->trans = R.trans.data();
  view->push_pool = R.push_pool.data();
  view->node_flags = R.node_flags.data();
  view->node_rule = R.node_rule.data();
  view->cache_keys = R.cache_keys.data();
  view->follow_start = R.follow_start.data();
  view->follow_next = R.follow_next.data();
  view->kept_rules = R.kept.data();
  view->raw_off = R.raw_off.data();
  view->raw = R.raw.data();
  view->n_raw = (int32_t)(R.raw.size() / 2);
  view->finals = R.finals.data();
  view->rule_start = R.rule_start.data();
  *out = fe;
  return GM_OK;
}

extern "C" void gm_front_end_release(gm_front_end* fe) { delete fe; }

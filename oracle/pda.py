"""Oracle automaton: restatement of REF pda.py (Thompson construction, node
merging, rule inlining, frozen tables, reachable stack tops) and of the
IR normalisation in REF grammar.py:673-729.  TEST INFRASTRUCTURE ONLY."""

from __future__ import annotations

from typing import Dict, List, Optional, Tuple

from paper_2411_15100_b200.grammar import Alt, Bytes, Eps, Lit, ParsedGrammar, Ref, Rep, Seq

EPS, CHAR, RULE = 0, 1, 2
STATE_CAP = 4096  # REF pda.py:53


class OracleStateLimit(RuntimeError):
    """REF pda.py:56-57 StateLimitError."""


def mask_to_ranges(mask: int) -> tuple:
    out = []
    b = 0
    while b < 256:
        if (mask >> b) & 1:
            e = b
            while e + 1 < 256 and (mask >> (e + 1)) & 1:
                e += 1
            out.append((b, e))
            b = e + 1
        else:
            b += 1
    return tuple(out)


# -- normalisation: REF grammar.py:673-720 -------------------------------------

def normalize(e):
    if isinstance(e, (Bytes, Ref, Eps)):
        return e
    if isinstance(e, Lit):
        return e if e.data else Eps()
    if isinstance(e, Seq):
        flat = []
        for x in map(normalize, e.items):
            if isinstance(x, Eps):
                continue
            flat.extend(x.items if isinstance(x, Seq) else [x])
        return Eps() if not flat else (flat[0] if len(flat) == 1 else Seq(tuple(flat)))
    if isinstance(e, Alt):
        flat = []
        for x in map(normalize, e.items):
            flat.extend(x.items if isinstance(x, Alt) else [x])
        return flat[0] if len(flat) == 1 else Alt(tuple(flat))
    if isinstance(e, Rep):
        inner = normalize(e.item)
        if isinstance(inner, Eps) or e.hi == 0:
            return Eps()
        if e.lo == 1 and e.hi == 1:
            return inner
        if e.hi is None and isinstance(inner, Rep) and inner.hi is None and inner.lo <= 1 and e.lo <= 1:
            return Rep(inner.item, 0 if 0 in (e.lo, inner.lo) else 1, None)
        return Rep(inner, e.lo, e.hi)
    raise TypeError(e)


# -- frozen automaton: REF pda.py:76-177 -----------------------------------------

class OraclePda:
    def __init__(self, node_rule, edges, rule_names, rule_start, rule_finals, root):
        self.node_rule = list(node_rule)
        self.edges = [tuple(e) for e in edges]
        self.rule_names = list(rule_names)
        self.rule_start = list(rule_start)
        self.rule_finals = [frozenset(f) for f in rule_finals]
        self.root = root
        n = len(self.node_rule)
        self.eps_out = [[] for _ in range(n)]
        self.rule_out = [[] for _ in range(n)]
        self.char_out = [[] for _ in range(n)]
        for s, d, k, v in self.edges:
            if k == EPS:
                self.eps_out[s].append(d)
            elif k == RULE:
                self.rule_out[s].append((v, d))
            else:
                self.char_out[s].append((v, d))
        self.is_final = [False] * n
        for fs in self.rule_finals:
            for f in fs:
                self.is_final[f] = True
        self.quiet = [not self.eps_out[i] and not self.rule_out[i] and not self.is_final[i] for i in range(n)]
        self.dead_end = [self.is_final[i] and not self.eps_out[i] and not self.rule_out[i] and not self.char_out[i]
                         for i in range(n)]
        none = ()
        self.byte_targets = []
        self.first_bytes = [0] * n
        for u in range(n):
            row = [none] * 256
            for ranges, d in self.char_out[u]:
                for lo, hi in ranges:
                    self.first_bytes[u] |= ((1 << (hi - lo + 1)) - 1) << lo
                    for b in range(lo, hi + 1):
                        row[b] = row[b] + (d,)
            self.byte_targets.append(row)

    @property
    def node_count(self) -> int:
        return len(self.node_rule)

    def start_node(self) -> int:
        return self.rule_start[self.root]


class _Work:
    """Mutable automaton used by construction and the optimisation passes."""

    def __init__(self):
        self.node_rule: List[int] = []
        self.edges: List[list] = []
        self.names: List[str] = []
        self.start: List[int] = []
        self.finals: List[set] = []
        self.root = 0

    @classmethod
    def of(cls, p: OraclePda) -> "_Work":
        w = cls()
        w.node_rule = list(p.node_rule)
        w.edges = [list(e) for e in p.edges]
        w.names = list(p.rule_names)
        w.start = list(p.rule_start)
        w.finals = [set(f) for f in p.rule_finals]
        w.root = p.root
        return w

    def node(self, rid: int) -> int:
        self.node_rule.append(rid)
        return len(self.node_rule) - 1

    def freeze(self, alive=None) -> OraclePda:
        if alive is None:
            return OraclePda(self.node_rule, self.edges, self.names, self.start, self.finals, self.root)
        remap, rules = {}, []
        for old, a in enumerate(alive):  # REF pda.py:218-239 compacted()
            if a:
                remap[old] = len(rules)
                rules.append(self.node_rule[old])
        edges = sorted((remap[s], remap[d], k, v) for s, d, k, v in self.edges)
        finals = [{remap[f] for f in fs if alive[f]} for fs in self.finals]
        return OraclePda(rules, edges, self.names, [remap[s] for s in self.start], finals, self.root)


# -- Thompson construction: REF pda.py:246-329 -------------------------------------

def build_raw_pda(g: ParsedGrammar) -> OraclePda:
    w = _Work()
    w.names = list(g.names)
    rid = {n: i for i, n in enumerate(g.names)}
    w.root = rid[g.root]
    w.start = [0] * len(g.names)
    w.finals = [set() for _ in g.names]

    def edge(s, d, k, v=None):
        w.edges.append([s, d, k, v])

    def emit(e, src, r):
        if isinstance(e, Eps):
            return src
        if isinstance(e, Lit):
            for byte in e.data:
                n = w.node(r)
                edge(src, n, CHAR, ((byte, byte),))
                src = n
            return src
        if isinstance(e, Bytes):
            n = w.node(r)
            edge(src, n, CHAR, mask_to_ranges(e.mask))
            return n
        if isinstance(e, Seq):
            for x in e.items:
                src = emit(x, src, r)
            return src
        if isinstance(e, Alt):
            join = w.node(r)
            for x in e.items:
                head = w.node(r)
                edge(src, head, EPS)
                edge(emit(x, head, r), join, EPS)
            return join
        if isinstance(e, Rep):
            cur = src
            for _ in range(e.lo):
                cur = emit(e.item, cur, r)
            if e.hi is None:
                loop = w.node(r)
                edge(cur, loop, EPS)
                it = e.item
                if isinstance(it, Bytes):
                    edge(loop, loop, CHAR, mask_to_ranges(it.mask))
                elif isinstance(it, Lit) and len(it.data) == 1:
                    edge(loop, loop, CHAR, ((it.data[0], it.data[0]),))
                else:
                    edge(emit(it, loop, r), loop, EPS)
                return loop
            for _ in range(e.hi - e.lo):
                nxt = emit(e.item, cur, r)
                if any(x[0] == nxt for x in w.edges):
                    fresh = w.node(r)
                    edge(nxt, fresh, EPS)
                    nxt = fresh
                edge(cur, nxt, EPS)
                cur = nxt
            return cur
        if isinstance(e, Ref):
            ret = w.node(r)
            edge(src, ret, RULE, rid[e.name])
            return ret
        raise TypeError(e)

    for r, name in enumerate(g.names):
        entry = w.node(r)
        w.start[r] = entry
        w.finals[r] = {emit(normalize(g.bodies[name]), entry, r)}
    return w.freeze()


# -- rule inlining: REF pda.py:336-396 ---------------------------------------------

def inline_rules(p: OraclePda, max_rule_size: int = 16, max_result_size: int = 512) -> OraclePda:
    w = _Work.of(p)
    nr = len(w.names)
    while True:
        sizes = [0] * nr
        for r in w.node_rule:
            sizes[r] += 1
        refs = [False] * nr
        for s, _, k, _ in w.edges:
            if k == RULE:
                refs[w.node_rule[s]] = True
        ok = {r for r in range(nr) if not refs[r] and sizes[r] <= max_rule_size}
        changed = False
        for host in range(nr):
            sites = [i for i, (s, _, k, v) in enumerate(w.edges) if k == RULE and v in ok and w.node_rule[s] == host]
            if not sites or sizes[host] + sum(sizes[w.edges[i][3]] for i in sites) > max_result_size:
                continue
            for i in sites:
                src, ret, _, callee = w.edges[i]
                copy = {}
                for old in sorted(j for j, rr in enumerate(w.node_rule) if rr == callee):
                    copy[old] = w.node(host)
                for s, d, k, v in list(w.edges):
                    if w.node_rule[s] == callee and s in copy:
                        w.edges.append([copy[s], copy[d], k, v])
                w.edges.append([src, copy[w.start[callee]], EPS, None])
                for f in w.finals[callee]:
                    w.edges.append([copy[f], ret, EPS, None])
                w.edges[i] = [src, src, EPS, None]
            changed = True
            sizes = [0] * nr
            for r in w.node_rule:
                sizes[r] += 1
        if not changed:
            break
    w.edges = [e for e in w.edges if not (e[2] == EPS and e[0] == e[1])]
    return w.freeze([True] * len(w.node_rule))


# -- node merging: REF pda.py:403-535 ------------------------------------------------

def merge_nodes(p: OraclePda) -> OraclePda:
    w = _Work.of(p)
    n = len(w.node_rule)
    alive = [True] * n
    final = [False] * n
    for fs in w.finals:
        for f in fs:
            final[f] = True
    is_start = [False] * n
    for s in w.start:
        is_start[s] = True
    outs = [set() for _ in range(n)]
    ins = [set() for _ in range(n)]
    live = [True] * len(w.edges)
    for i, (s, d, _, _) in enumerate(w.edges):
        outs[s].add(i)
        ins[d].add(i)

    def drop_edge(i):
        live[i] = False
        s, d, _, _ = w.edges[i]
        outs[s].discard(i)
        ins[d].discard(i)

    def absorb(keep, gone):
        for i in list(ins[gone]):
            ins[gone].discard(i)
            w.edges[i][1] = keep
            ins[keep].add(i)
        for i in list(outs[gone]):
            outs[gone].discard(i)
            w.edges[i][0] = keep
            outs[keep].add(i)
        if final[gone]:
            final[keep] = True
        if is_start[gone]:
            is_start[keep] = True
            w.start = [keep if s == gone else s for s in w.start]
        alive[gone] = False

    def dedupe():
        hit, seen = False, {}
        for i, e in enumerate(w.edges):
            if not live[i]:
                continue
            s, d, k, v = e
            key = (s, d, k, v)
            if (k == EPS and s == d) or key in seen:
                drop_edge(i)
                hit = True
            else:
                seen[key] = i
        return hit

    def siblings():
        hit = False
        for u in range(n):
            if not alive[u]:
                continue
            by_label: Dict[tuple, list] = {}
            for i in sorted(outs[u]):
                _, d, k, v = w.edges[i]
                by_label.setdefault((k, v), []).append(d)
            for ds in by_label.values():
                cand = [d for d in dict.fromkeys(ds) if d != u and not is_start[d] and len(ins[d]) == 1]
                if len(cand) >= 2:
                    for d in cand[1:]:
                        absorb(cand[0], d)
                    hit = True
        return hit

    def contract():
        hit = False
        for i in range(len(w.edges)):
            if not live[i]:
                continue
            s, t, k, _ = w.edges[i]
            if k != EPS:
                continue
            if s == t:
                drop_edge(i)
                hit = True
            elif len(ins[t]) == 1 and not is_start[t]:
                drop_edge(i)
                absorb(s, t)
                hit = True
            elif len(outs[s]) == 1 and (not final[s] or final[t]):
                drop_edge(i)
                absorb(t, s)
                hit = True
        return hit

    while True:
        c = dedupe()
        c |= siblings()
        c |= dedupe()
        c |= contract()
        if not c:
            break
    w.edges = [e for i, e in enumerate(w.edges) if live[i]]
    w.finals = [{f for f in range(n) if alive[f] and final[f] and w.node_rule[f] == r} for r in range(len(w.names))]
    return w.freeze(alive)


def build_oracle_pda(g: ParsedGrammar, merge: bool = True, inline: bool = True) -> OraclePda:
    """REF bundle.py:75-88 pipeline: build, merge, (inline, merge) x <= 8."""
    p = build_raw_pda(g)
    if merge:
        p = merge_nodes(p)
    if inline:
        for _ in range(8):
            shape = (p.node_count, len(p.edges))
            p = inline_rules(p)
            if merge:
                p = merge_nodes(p)
            if (p.node_count, len(p.edges)) == shape:
                break
    return p


def reachable_tops(p: OraclePda) -> List[int]:
    """REF pda.py:601-632: the cache key set."""
    start = p.start_node()
    seen = {start}
    work = [start]
    while work:
        u = work.pop()
        nxt = [d for _, d in p.char_out[u]] + list(p.eps_out[u])
        for r, ret in p.rule_out[u]:
            nxt += [p.rule_start[r], ret]
        for v in nxt:
            if v not in seen:
                seen.add(v)
                work.append(v)
    cand = {start}
    for u in seen:
        cand.update(d for _, d in p.char_out[u])
        cand.update(ret for _, ret in p.rule_out[u])
    return sorted(v for v in cand if v in seen and not (p.dead_end[v] and p.node_rule[v] != p.root))


# -- naive set-of-stacks interpreter: REF pda.py:547-594 -----------------------------

def _close_stacks(p: OraclePda, states: set, cap: int) -> set:
    seen = set(states)
    work = list(states)
    while work:
        st = work.pop()
        top = st[-1]
        nxt = [st[:-1] + (d,) for d in p.eps_out[top]]
        nxt += [st[:-1] + (ret, p.rule_start[r]) for r, ret in p.rule_out[top]]
        if p.is_final[top] and len(st) > 1:
            nxt.append(st[:-1])
        for ns in nxt:
            if ns not in seen:
                seen.add(ns)
                work.append(ns)
                if len(seen) > cap:
                    raise OracleStateLimit(f"state set exceeded cap of {cap}")
    return seen


def step_stacks(p: OraclePda, states, data: bytes, cap: int = STATE_CAP) -> frozenset:
    cur = _close_stacks(p, set(states), cap)
    for b in data:
        nxt = {st[:-1] + (d,) for st in cur for d in p.byte_targets[st[-1]][b]}
        if not nxt:
            return frozenset()
        cur = _close_stacks(p, nxt, cap)
    return frozenset(cur)


def stacks_accept(p: OraclePda, states) -> bool:
    return any(len(s) == 1 and p.is_final[s[0]] and p.node_rule[s[0]] == p.root for s in states)

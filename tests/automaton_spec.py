"""Executable specification of the native front end (csrc/front_end.cpp),
test infrastructure only: the same pipeline in Python — per-rule NFA over
byte classes, subset construction + Moore minimisation, inlining,
silent-move pre-closure, follow automaton — whose tables the native build
must equal array for array (tests/test_frontend.py).  The product uses
paper_2411_15100_b200.automaton.build_tables_native.  Not covered here: the
C++ front end's epsilon-free NFA fallback for rules whose subset
construction exceeds max_dfa_states (front_end.cpp eps_free); this spec
raises GrammarError there instead.
"""

from __future__ import annotations

from typing import Dict, List, Optional, Tuple

import numpy as np

from paper_2411_15100_b200.automaton import (DEFAULT_STATE_CAP, NODE_DEAD_END, NODE_POP, AutomatonOptions,  # noqa: F401
                                             CompiledTables, StateLimitError, _FOLLOW_ANY, _FOLLOW_DEAD)
from paper_2411_15100_b200.grammar import Alt, Bytes, Eps, GrammarError, Lit, ParsedGrammar, Ref, Rep, Seq  # noqa: F401
from dataclasses import dataclass  # noqa: E402

# ---------------------------------------------------------------------------
# byte classes


def byte_partition(masks) -> Tuple[List[int], int]:
    """Coarsest partition of 0..255 refining every mask: class id per byte."""
    cls = [0] * 256
    n = 1
    for m in masks:
        remap: Dict[Tuple[int, bool], int] = {}
        nxt = [0] * 256
        for b in range(256):
            key = (cls[b], bool((m >> b) & 1))
            if key not in remap:
                remap[key] = len(remap)
            nxt[b] = remap[key]
        cls, n = nxt, len(remap)
    # canonical numbering: by first byte of each class
    order: Dict[int, int] = {}
    for b in range(256):
        order.setdefault(cls[b], len(order))
    return [order[c] for c in cls], n


def _class_set(mask: int, cls: List[int]) -> int:
    out = 0
    b = mask
    while b:
        low = b & -b
        out |= 1 << cls[low.bit_length() - 1]
        b ^= low
    return out


# ---------------------------------------------------------------------------
# per-rule automata


class _Nfa:
    """Epsilon NFA of one rule: byte edges labelled with class sets."""

    def __init__(self):
        self.byte: List[List[Tuple[int, int]]] = []  # (class_set, dst)
        self.call: List[List[Tuple[int, int]]] = []  # (rid, dst)
        self.eps: List[List[int]] = []
        self.start = 0
        self.finals: set = set()

    def new(self) -> int:
        self.byte.append([])
        self.call.append([])
        self.eps.append([])
        return len(self.byte) - 1


@dataclass
class _Dfa:
    """Deterministic rule automaton: trans[s][class] = t, calls[s][rid] = t."""

    trans: List[Dict[int, int]]
    calls: List[Dict[int, int]]
    finals: List[bool]
    start: int = 0

    @property
    def size(self) -> int:
        return len(self.trans)


def _build_nfa(expr, rid_of: Dict[str, int], cls: List[int]) -> _Nfa:
    a = _Nfa()
    memo_sets: Dict[int, int] = {}

    def cset(mask: int) -> int:
        got = memo_sets.get(mask)
        if got is None:
            got = memo_sets[mask] = _class_set(mask, cls)
        return got

    def emit(e, s: int) -> int:
        if isinstance(e, Eps):
            return s
        if isinstance(e, Bytes):
            t = a.new()
            a.byte[s].append((cset(e.mask), t))
            return t
        if isinstance(e, Lit):
            for byte in e.data:
                t = a.new()
                a.byte[s].append((cset(1 << byte), t))
                s = t
            return s
        if isinstance(e, Seq):
            for item in e.items:
                s = emit(item, s)
            return s
        if isinstance(e, Alt):
            join = a.new()
            for item in e.items:
                head = a.new()
                a.eps[s].append(head)
                a.eps[emit(item, head)].append(join)
            return join
        if isinstance(e, Rep):
            for _ in range(e.lo):
                head = a.new()
                a.eps[s].append(head)
                s = emit(e.item, head)
            if e.hi is None:
                loop = a.new()
                a.eps[s].append(loop)
                body = a.new()
                a.eps[loop].append(body)
                a.eps[emit(e.item, body)].append(loop)
                return loop
            exit_ = a.new()
            a.eps[s].append(exit_)
            for _ in range(e.hi - e.lo):
                head = a.new()
                a.eps[s].append(head)
                s = emit(e.item, head)
                a.eps[s].append(exit_)
            return exit_
        if isinstance(e, Ref):
            t = a.new()
            a.call[s].append((rid_of[e.name], t))
            return t
        raise TypeError(e)

    a.start = a.new()
    a.finals = {emit(expr, a.start)}
    return a


def _dfa_as_nfa(d: _Dfa) -> _Nfa:
    a = _Nfa()
    for _ in range(d.size):
        a.new()
    for s in range(d.size):
        for c, t in d.trans[s].items():
            a.byte[s].append((1 << c, t))
        for r, t in d.calls[s].items():
            a.call[s].append((r, t))
    a.start = d.start
    a.finals = {s for s in range(d.size) if d.finals[s]}
    return a


def _determinize(a: _Nfa, max_states: int) -> _Dfa:
    def close(states) -> frozenset:
        seen = set(states)
        work = list(states)
        while work:
            u = work.pop()
            for v in a.eps[u]:
                if v not in seen:
                    seen.add(v)
                    work.append(v)
        return frozenset(seen)

    start = close([a.start])
    ids = {start: 0}
    order = [start]
    trans: List[Dict[int, int]] = []
    calls: List[Dict[int, int]] = []
    finals: List[bool] = []
    i = 0
    while i < len(order):
        S = order[i]
        i += 1
        by_class: Dict[int, set] = {}
        by_rule: Dict[int, set] = {}
        for u in S:
            for cs, v in a.byte[u]:
                while cs:
                    low = cs & -cs
                    by_class.setdefault(low.bit_length() - 1, set()).add(v)
                    cs ^= low
            for r, v in a.call[u]:
                by_rule.setdefault(r, set()).add(v)
        def target(vs) -> int:
            T = close(vs)
            if T not in ids:
                ids[T] = len(order)
                order.append(T)
                if len(order) > max_states:
                    raise GrammarError(f"rule automaton exceeds {max_states} states after determinisation")
            return ids[T]

        row = {c: target(vs) for c, vs in by_class.items()}
        crow = {r: target(vs) for r, vs in by_rule.items()}
        trans.append(row)
        calls.append(crow)
        finals.append(any(u in a.finals for u in S))
    return _Dfa(trans, calls, finals, 0)


def _minimize(d: _Dfa) -> _Dfa:
    """Moore partition refinement; unreachable states never exist here."""
    n = d.size
    block = [0] * n
    keys = {}
    for s in range(n):
        k = (d.finals[s], tuple(sorted(d.trans[s])), tuple(sorted(d.calls[s])))
        block[s] = keys.setdefault(k, len(keys))
    nb = len(keys)
    while True:
        keys = {}
        nxt = [0] * n
        for s in range(n):
            k = (
                block[s],
                tuple((c, block[t]) for c, t in sorted(d.trans[s].items())),
                tuple((r, block[t]) for r, t in sorted(d.calls[s].items())),
            )
            nxt[s] = keys.setdefault(k, len(keys))
        if len(keys) == nb:
            break
        block, nb = nxt, len(keys)
    # renumber blocks in BFS order from the start for determinism
    rep = {}
    for s in range(n):
        rep.setdefault(block[s], s)
    order = [block[d.start]]
    seen = {block[d.start]: 0}
    i = 0
    while i < len(order):
        s = rep[order[i]]
        i += 1
        for _, t in sorted(d.trans[s].items()):
            if block[t] not in seen:
                seen[block[t]] = len(order)
                order.append(block[t])
        for _, t in sorted(d.calls[s].items()):
            if block[t] not in seen:
                seen[block[t]] = len(order)
                order.append(block[t])
    trans, calls, finals = [], [], []
    for b in order:
        s = rep[b]
        trans.append({c: seen[block[t]] for c, t in d.trans[s].items()})
        calls.append({r: seen[block[t]] for r, t in d.calls[s].items()})
        finals.append(d.finals[s])
    return _Dfa(trans, calls, finals, 0)


def _inline_into(host: _Dfa, callees: Dict[int, _Dfa]) -> _Nfa:
    a = _dfa_as_nfa(host)
    base_size = host.size
    copies: Dict[Tuple[int, int], int] = {}
    for s in range(base_size):
        keep = []
        for r, t in a.call[s]:
            if r not in callees:
                keep.append((r, t))
                continue
            sub = callees[r]
            off = a.new()
            for _ in range(sub.size - 1):
                a.new()
            for q in range(sub.size):
                for c, v in sub.trans[q].items():
                    a.byte[off + q].append((1 << c, off + v))
                for r2, v in sub.calls[q].items():
                    a.call[off + q].append((r2, off + v))
                if sub.finals[q]:
                    a.eps[off + q].append(t)
            a.eps[s].append(off + sub.start)
        a.call[s] = keep
    return a


# ---------------------------------------------------------------------------
# tables



def build_tables(g: ParsedGrammar, opts: Optional[AutomatonOptions] = None) -> CompiledTables:
    opts = opts or AutomatonOptions()
    names = list(g.names)
    rid_of = {nm: i for i, nm in enumerate(names)}

    masks = set()
    for body in g.bodies.values():
        stack = [body]
        while stack:
            e = stack.pop()
            if isinstance(e, Bytes):
                masks.add(e.mask)
            elif isinstance(e, Lit):
                masks.update(1 << b for b in e.data)
            elif isinstance(e, (Seq, Alt)):
                stack.extend(e.items)
            elif isinstance(e, Rep):
                stack.append(e.item)
    cls, n_classes = byte_partition(sorted(masks))

    nfas = {rid_of[nm]: _build_nfa(g.bodies[nm], rid_of, cls) for nm in names}
    if not opts.determinize:
        raise NotImplementedError("determinize=False is not supported by the device tables")
    dfas = {r: _minimize(_determinize(a, opts.max_dfa_states)) for r, a in nfas.items()}
    root = rid_of[g.root]

    if opts.inline:
        for _ in range(64):
            inlinable = {
                r: d
                for r, d in dfas.items()
                if not any(d.calls[s] for s in range(d.size)) and d.size <= opts.inline_max_rule_states
            }
            if opts.inline_calls:
                # live callers per rule (the root counts as called from outside)
                callers: Dict[int, set] = {r: set() for r in dfas}
                seen, work = {root}, [root]
                while work:
                    h = work.pop()
                    for s_ in range(dfas[h].size):
                        for r in dfas[h].calls[s_]:
                            callers[r].add(h)
                            if r not in seen:
                                seen.add(r)
                                work.append(r)
                for r in sorted(seen):
                    d = dfas[r]
                    if r in inlinable or r == root or len(callers[r]) != 1 or r in callers[r]:
                        continue
                    if d.size <= opts.inline_max_result_states:
                        inlinable[r] = d
            changed = False
            for host in list(dfas):
                hd = dfas[host]
                targets = {r for s in range(hd.size) for r in hd.calls[s] if r in inlinable and r != host}
                if not targets:
                    continue
                new = _minimize(_determinize(_inline_into(hd, {r: inlinable[r] for r in targets}), opts.max_dfa_states))
                if new.size > opts.inline_max_result_states:
                    continue
                dfas[host] = new
                changed = True
            if not changed:
                break

    # keep rules reachable from the root
    live = {root}
    work = [root]
    while work:
        r = work.pop()
        d = dfas[r]
        for s in range(d.size):
            for q in d.calls[s]:
                if q not in live:
                    live.add(q)
                    work.append(q)
    kept = sorted(live)
    new_rid = {r: i for i, r in enumerate(kept)}
    offset = {}
    n_nodes = 0
    for r in kept:
        offset[r] = n_nodes
        n_nodes += dfas[r].size
    node_rule = np.zeros(n_nodes, dtype=np.int32)
    trans_n: List[Dict[int, int]] = []
    calls_n: List[List[Tuple[int, int]]] = []  # (new rid, return node)
    final_n: List[bool] = []
    rule_start = {}
    for r in kept:
        d, o = dfas[r], offset[r]
        rule_start[new_rid[r]] = o + d.start
        for s in range(d.size):
            node_rule[o + s] = new_rid[r]
            trans_n.append({c: o + t for c, t in d.trans[s].items()})
            calls_n.append(sorted((new_rid[q], o + t) for q, t in d.calls[s].items()))
            final_n.append(d.finals[s])
    n_rules = len(kept)
    root_n = new_rid[root]
    start_node = rule_start[root_n]
    dead_end = [final_n[u] and not trans_n[u] and not calls_n[u] for u in range(n_nodes)]

    # silent-move pre-closure per node (relative stacks, REF cache.py:110-143)
    pop_flag = [False] * n_nodes
    push_ids: Dict[tuple, int] = {(): 0}
    push_pool: List[int] = []
    push_off: Dict[tuple, int] = {(): 0}
    rows: List[List[List[Tuple[int, int]]]] = []  # per node: per class list of (target, push)
    cap = opts.state_cap
    for u in range(n_nodes):
        seen = {((), u)}
        work = [((), u)]
        while work:
            P, m = work.pop()
            nxt = [(P + (ret,), rule_start[q]) for q, ret in calls_n[m]]
            if final_n[m]:
                if P:
                    nxt.append((P[:-1], P[-1]))
                else:
                    pop_flag[u] = True
            for st in nxt:
                if st not in seen:
                    seen.add(st)
                    work.append(st)
                    if len(seen) > cap:
                        raise StateLimitError(f"branch set exceeded cap of {cap}")
        per_class: Dict[int, list] = {}
        for P, m in sorted(seen):
            for c, d in trans_n[m].items():
                PP = P
                while dead_end[d] and PP:
                    d, PP = PP[-1], PP[:-1]
                lst = per_class.setdefault(c, [])
                if (PP, d) not in lst:
                    lst.append((PP, d))
        rows.append(per_class)

    trans_off = np.zeros(n_nodes * n_classes + 1, dtype=np.int64)
    trans_flat: List[int] = []
    keys = {start_node}
    for u in range(n_nodes):
        pc = rows[u]
        for c in range(n_classes):
            trans_off[u * n_classes + c] = len(trans_flat) // 2
            for P, d in sorted(pc.get(c, ()), key=lambda x: (x[1], x[0])):
                if len(P) > 255:
                    raise StateLimitError("push run longer than 255 frames")
                if P not in push_off:
                    push_off[P] = len(push_pool)
                    push_pool.extend(P)
                    if len(push_pool) >= (1 << 24):
                        raise StateLimitError("push pool exceeds 16M entries")
                trans_flat += [d, push_off[P] | (len(P) << 24)]
                keys.add(d)
                keys.update(P)
    trans_off[n_nodes * n_classes] = len(trans_flat) // 2
    cache_keys = sorted(k for k in keys if not (dead_end[k] and node_rule[k] != root_n))

    flags = np.zeros(n_nodes, dtype=np.uint8)
    for u in range(n_nodes):
        flags[u] = (NODE_POP if pop_flag[u] else 0) | (NODE_DEAD_END if dead_end[u] else 0)

    f_start, f_next, n_f = _follow_dfa(
        n_nodes, n_rules, n_classes, root_n, trans_n, calls_n, final_n, node_rule, opts
    )

    t = CompiledTables(
        n_nodes=n_nodes,
        n_rules=n_rules,
        n_classes=n_classes,
        start_node=start_node,
        root_rule=root_n,
        rule_names=[names[r] for r in kept],
        byte_class=np.asarray(cls, dtype=np.uint8),
        trans_off=trans_off.astype(np.int32),
        trans=np.asarray(trans_flat, dtype=np.int64).astype(np.int32),
        push_pool=np.asarray(push_pool if push_pool else [0], dtype=np.int32),
        node_flags=flags,
        node_rule=node_rule,
        cache_keys=np.asarray(cache_keys, dtype=np.int32),
        follow_start=f_start,
        follow_next=f_next,
        n_fstates=n_f,
    )
    raw_off, raw = [0], []
    for u in range(n_nodes):
        raw += [(c, d) for c, d in sorted(trans_n[u].items())]
        raw += [(-(q + 1), ret) for q, ret in calls_n[u]]
        raw_off.append(len(raw))
    t.raw_off = np.asarray(raw_off, dtype=np.int32)
    t.raw = np.asarray(raw, dtype=np.int32).reshape(-1, 2) if raw else np.zeros((0, 2), dtype=np.int32)
    t.finals = np.asarray(final_n, dtype=np.uint8)
    t.rule_start = np.asarray([rule_start[r] for r in range(n_rules)], dtype=np.int32)
    t.stats = {
        "nodes": n_nodes,
        "rules": n_rules,
        "classes": n_classes,
        "transitions": len(trans_flat) // 2,
        "keys": len(cache_keys),
        "follow_states": n_f,
    }
    return t


def _follow_dfa(n_nodes, n_rules, n_classes, root, trans_n, calls_n, final_n, node_rule, opts):
    """Follow automaton of every rule (REF cache.py:241-333), determinised.

    State sets hold automaton nodes plus END; a node with rule calls is a
    wildcard stop; a final node cascades into the follow set of its rule (END
    for the root).  Returns (start[n_rules], next[n_states*n_classes], n)."""
    if not opts.ctx_expansion:
        return np.full(n_rules, _FOLLOW_ANY, dtype=np.int32), np.zeros(n_classes, dtype=np.int32), 0
    END = -1
    seeds: Dict[int, set] = {r: set() for r in range(n_rules)}
    for u in range(n_nodes):
        for q, ret in calls_n[u]:
            seeds[q].add(ret)
    wildnode = [bool(calls_n[u]) for u in range(n_nodes)]

    def expand(S):
        seen = set(S)
        work = [s for s in S if s != END]
        wild = False
        while work:
            s = work.pop()
            if wildnode[s]:
                wild = True
                continue
            if final_n[s]:
                r = node_rule[s]
                for t in seeds[r]:
                    if t not in seen:
                        seen.add(t)
                        work.append(t)
                if r == root:
                    seen.add(END)
        return frozenset(seen), wild

    ids: Dict[frozenset, int] = {}
    order: List[frozenset] = []
    rows: List[List[int]] = []

    def intern(S, wild) -> int:
        if wild:
            return _FOLLOW_ANY
        if not S:
            return _FOLLOW_DEAD
        got = ids.get(S)
        if got is None:
            if len(order) >= opts.max_follow_states:
                return _FOLLOW_ANY  # sound over-approximation
            got = ids[S] = len(order)
            order.append(S)
        return got

    start = np.zeros(n_rules, dtype=np.int32)
    for r in range(n_rules):
        seed = set(seeds[r])
        if r == root:
            seed.add(END)
        if not seed:
            start[r] = _FOLLOW_ANY  # no information: anything may follow
            continue
        S, wild = expand(seed)
        start[r] = intern(S, wild)
    i = 0
    while i < len(order):
        S = order[i]
        i += 1
        row = [_FOLLOW_DEAD] * n_classes
        by_class: Dict[int, set] = {}
        for s in S:
            if s == END:
                continue
            for c, d in trans_n[s].items():
                by_class.setdefault(c, set()).add(d)
        for c in sorted(by_class):  # canonical numbering (front_end.cpp does the same)
            T, wild = expand(by_class[c])
            row[c] = intern(T, wild)
        rows.append(row)
    nxt = np.asarray(rows if rows else [[_FOLLOW_DEAD] * n_classes], dtype=np.int32).reshape(-1)
    return start, nxt, len(order)


# ---------------------------------------------------------------------------
# native front end (csrc/front_end.cpp): same tables, built in C++



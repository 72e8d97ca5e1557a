"""Oracle adaptive token-mask cache: restatement of REF cache.py (sorted
sweep with LCP rollback, classification, FollowFsa context expansion,
adaptive storage, build_mask_cache).  TEST INFRASTRUCTURE ONLY."""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from .pda import OraclePda, OracleStateLimit, reachable_tops

EMPTY = -1
BRANCH_CAP = 4096  # REF cache.py:58
ACCEPT_HEAVY, REJECT_HEAVY, BITSET_FORM = 0, 1, 2  # REF cache.py:344


class InternArena:
    """REF pstack.py interning mode (41-52): equal (parent, node) => equal handle."""

    def __init__(self):
        self.parent: List[int] = []
        self.node: List[int] = []
        self.ids: Dict[tuple, int] = {}

    def push(self, parent: int, node: int) -> int:
        h = self.ids.get((parent, node))
        if h is None:
            h = self.ids[(parent, node)] = len(self.parent)
            self.parent.append(parent)
            self.node.append(node)
        return h


@dataclass
class SweepOut:
    accepted: list
    rejected: list
    dependents: list  # (key, [remainders])
    bytes_examined: int


def sweep(p: OraclePda, items, lcps, starts, *, synthetic: bool, cap: int = BRANCH_CAP) -> SweepOut:
    """REF cache.py:88-193.  items: [(key, bytes)] sorted; lcps aligned;
    starts: [(chain tuple, node)]."""
    A = InternArena()
    par, nod = A.parent, A.node
    bt, eps, rout, fin, quiet, dead = p.byte_targets, p.eps_out, p.rule_out, p.is_final, p.quiet, p.dead_end
    rstart = p.rule_start

    def closure(branches):
        popped = False
        seen = set(branches)
        work = [x for x in branches if not quiet[x[1]]]
        while work:
            h, n = work.pop()
            cand = [(h, d) for d in eps[n]] + [(A.push(h, ret), rstart[r]) for r, ret in rout[n]]
            if fin[n]:
                if h == EMPTY:
                    popped = True
                else:
                    cand.append((par[h], nod[h]))
            for t in cand:
                if t not in seen:
                    seen.add(t)
                    if not quiet[t[1]]:
                        work.append(t)
            if len(seen) > cap:
                raise OracleStateLimit(f"branch set exceeded cap of {cap}")
        if any(dead[n] and h != EMPTY for h, n in seen):
            seen = {(h, n) for h, n in seen if not (dead[n] and h != EMPTY)}
        return seen, popped

    init = []
    for chain, n in starts:
        h = EMPTY
        for r in chain:
            h = A.push(h, r)
        init.append((h, n))
    st0, pop0 = closure(init)
    ckpt, pops = [st0], [pop0]
    acc, rej, deps = [], [], []
    examined = 0
    for (key, tok), lcp in zip(items, lcps):
        del ckpt[lcp + 1:]
        del pops[lcp + 1:]
        states = ckpt[-1]
        for i in range(lcp, len(tok)):
            b = tok[i]
            examined += 1
            popped = False
            if states:
                stepped = set()
                noisy = False
                for h, n in states:
                    for d in bt[n][b]:
                        stepped.add((h, d))
                        noisy |= not quiet[d]
                if not stepped:
                    states = frozenset()
                elif noisy:
                    states, popped = closure(stepped)
                else:
                    states = stepped
            ckpt.append(states)
            pops.append(popped)
        if states:
            acc.append(key)
        elif synthetic and any(pops):
            deps.append((key, [tok[d:] for d, f in enumerate(pops) if f]))
        else:
            rej.append(key)
    return SweepOut(acc, rej, deps, examined)


class FollowFsa:
    """REF cache.py:241-333: byte strings that may follow a rule."""

    END = -2

    def __init__(self, p: OraclePda):
        self.p = p
        starts = {r: set() for r in range(len(p.rule_names))}
        for s, d, k, v in p.edges:
            if k == 2:  # RULE
                starts[v].add(d)
        self.starts = {r: tuple(sorted(x)) for r, x in starts.items()}
        self.wild = [bool(p.rule_out[i]) for i in range(p.node_count)]
        self.base: Dict[int, object] = {}
        self.memo: Dict[tuple, bool] = {}

    def expand(self, states):
        p = self.p
        seen = set(states)
        work = list(states)
        wild = False
        while work:
            s = work.pop()
            if s == self.END:
                continue
            if self.wild[s]:
                wild = True
                continue
            for d in p.eps_out[s]:
                if d not in seen:
                    seen.add(d)
                    work.append(d)
            if p.is_final[s]:
                r = p.node_rule[s]
                for t in self.starts[r]:
                    if t not in seen:
                        seen.add(t)
                        work.append(t)
                if r == p.root:
                    seen.add(self.END)
        return frozenset(seen), wild

    def start_states(self, rid):
        if rid not in self.base:
            seed = set(self.starts[rid])
            if rid == self.p.root:
                seed.add(self.END)
            self.base[rid] = self.expand(seed) if seed else None
        return self.base[rid]

    def allows(self, rid: int, rem: bytes) -> bool:
        key = (rid, rem)
        if key in self.memo:
            return self.memo[key]
        base = self.start_states(rid)
        ok = True
        if base is not None:
            states, wild = base
            if not wild:
                for b in rem:
                    nxt = {d for s in states if s != self.END and not self.wild[s] for d in self.p.byte_targets[s][b]}
                    if not nxt:
                        ok = False
                        break
                    states, wild = self.expand(nxt)
                    if wild:
                        break
        self.memo[key] = ok
        return ok


def pack_bits(ids, vocab_size: int) -> np.ndarray:
    """REF cache.py:349-355."""
    words = np.zeros((vocab_size + 31) // 32, dtype=np.uint32)
    if len(ids):
        a = np.asarray(ids, dtype=np.uint32)
        np.bitwise_or.at(words, a >> 5, np.uint32(1) << (a & np.uint32(31)))
    return words


@dataclass
class Entry:
    variant: int
    ids: np.ndarray
    bits: Optional[np.ndarray]
    dependent: np.ndarray


def choose_storage(acc, rej, dep, vocab_size: int) -> Entry:
    """REF cache.py:389-413: byte-minimal variant, ties AH > RH > BITSET."""
    acc = np.asarray(sorted(acc), dtype=np.uint32)
    rej = np.asarray(sorted(rej), dtype=np.uint32)
    dep = np.asarray(sorted(dep), dtype=np.uint32)
    sizes = [4 * (len(rej) + len(dep)), 4 * (len(acc) + len(dep)), (vocab_size + 7) // 8 + 4 * len(dep)]
    v = sizes.index(min(sizes))
    if v == ACCEPT_HEAVY:
        return Entry(v, rej, None, dep)
    if v == REJECT_HEAVY:
        return Entry(v, acc, None, dep)
    return Entry(v, np.zeros(0, np.uint32), pack_bits(acc, vocab_size), dep)


@dataclass
class OracleCache:
    vocab_size: int
    entries: Dict[int, Entry]
    stats: dict = field(default_factory=dict)


def sorted_items(vocab):
    """REF vocab.py:227-234 + cache.py:534-543: non-special tokens by bytes
    (ties by id) with LCPs; empty tokens are forced rejects."""
    ids = sorted((t for t in range(vocab.size) if t not in vocab.special_tokens), key=lambda t: (vocab.tokens[t], t))
    items, lcps, forced = [], [], []
    prev = None
    for t in ids:
        tok = vocab.tokens[t]
        if not tok:
            forced.append(t)
            continue
        lcp = 0
        if prev is not None:
            m = min(len(prev), len(tok))
            while lcp < m and prev[lcp] == tok[lcp]:
                lcp += 1
        items.append((t, tok))
        lcps.append(lcp)
        prev = tok
    return items, lcps, forced


def build_oracle_cache(p: OraclePda, vocab, ctx: bool = True, keys=None) -> OracleCache:
    """REF cache.py:516-574."""
    follow = FollowFsa(p) if ctx else None
    items, lcps, forced = sorted_items(vocab)
    entries = {}
    stats = {"accepted_total": 0, "rejected_total": 0, "dependent_before": 0, "dependent_total": 0}
    for node in (keys if keys is not None else reachable_tops(p)):
        res = sweep(p, items, lcps, [((), node)], synthetic=True)
        rej = res.rejected + forced
        dep = []
        for tid, rems in res.dependents:
            if follow is None or any(follow.allows(p.node_rule[node], r) for r in rems):
                dep.append(tid)
            else:
                rej.append(tid)
        entries[node] = choose_storage(res.accepted, rej, dep, vocab.size)
        stats["accepted_total"] += len(res.accepted)
        stats["rejected_total"] += len(rej)
        stats["dependent_before"] += len(res.dependents)
        stats["dependent_total"] += len(dep)
    stats["entries"] = len(entries)
    return OracleCache(vocab.size, entries, stats)

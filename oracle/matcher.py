"""Oracle runtime matcher: restatement of REF matcher.py (closure, spent-final
rewriting, accept, Algorithm-1 cached fill with dependent resolution, EOS,
rollback window, branch, jump-forward) and the language-level brute-force
mask of REF tests/conftest.py:149-159.  TEST INFRASTRUCTURE ONLY.

Stacks live in an interning arena (REF pstack.py interning mode): equal
content => equal handle, so dedupe-by-content (REF matcher.py:202-206) is
dedupe by (handle, node).  Handles are never reclaimed (an oracle does not
need the reference's refcounting, which only bounds memory)."""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass
from typing import Optional

import numpy as np

from paper_2411_15100_b200.grammar import parse_grammar

from .cache import (ACCEPT_HEAVY, BRANCH_CAP, EMPTY, REJECT_HEAVY, InternArena, OracleCache, build_oracle_cache,
                    pack_bits, sorted_items, sweep)
from .pda import OraclePda, OracleStateLimit, build_oracle_pda, stacks_accept, step_stacks


class OracleMatcherError(RuntimeError):
    pass


@dataclass
class OracleBundle:
    pda: OraclePda
    cache: Optional[OracleCache]
    vocab: object


def compile_oracle_bundle(text: str, vocab, *, merge=True, inline=True, cache=True, ctx=True) -> OracleBundle:
    """REF bundle.py:65-93."""
    p = build_oracle_pda(parse_grammar(text), merge=merge, inline=inline)
    c = build_oracle_cache(p, vocab, ctx=ctx and cache) if cache else None
    return OracleBundle(p, c, vocab)


class OracleMatcher:
    def __init__(self, bundle: OracleBundle, history_window: int = 32, dep_threshold: int = 64):
        self.b = bundle
        self.p = bundle.pda
        self.v = bundle.vocab
        self.window = history_window
        self.dep_threshold = dep_threshold
        self.arena = InternArena()
        self.history = deque()
        self.terminated = False
        p = self.p
        self.root_finals = {n for n in range(p.node_count) if p.is_final[n] and p.node_rule[n] == p.root}
        self.universe = pack_bits([t for t in range(self.v.size)
                                   if t not in self.v.special_tokens and self.v.tokens[t]], self.v.size)
        self.tops = [(EMPTY, p.start_node())]
        self._dep_items = {}

    # -- REF matcher.py:162-217 ---------------------------------------------------
    def _close(self, branches):
        p, A = self.p, self.arena
        seen = set(branches)
        work = list(branches)
        while work:
            h, n = work.pop()
            cand = [(h, d) for d in p.eps_out[n]] + [(A.push(h, ret), p.rule_start[r]) for r, ret in p.rule_out[n]]
            if p.is_final[n] and h != EMPTY:
                cand.append((A.parent[h], A.node[h]))
            for t in cand:
                if t not in seen:
                    seen.add(t)
                    work.append(t)
            if len(seen) > BRANCH_CAP:
                raise OracleMatcherError(f"stack set exceeded cap of {BRANCH_CAP}")
        return seen

    def _rewrite(self, stepped):
        A, dead = self.arena, self.p.dead_end
        out = set()
        for h, n in stepped:
            while dead[n] and h != EMPTY:
                h, n = A.parent[h], A.node[h]
            out.add((h, n))
        return sorted(out)

    def _sim(self, branches, data: bytes):
        bt = self.p.byte_targets
        states = branches
        for b in data:
            stepped = {(h, d) for h, n in self._close(states) for d in bt[n][b]}
            if not stepped:
                return None
            states = self._rewrite(stepped)
        return states

    def closed_facts(self):
        """REF matcher.py:219-237: (terminable, union of first bytes)."""
        closed = self._close(self.tops)
        term = any(h == EMPTY and n in self.root_finals for h, n in closed)
        fb = 0
        for _, n in closed:
            fb |= self.p.first_bytes[n]
        return term, fb

    def _push_history(self):
        self.history.append((self.tops, self.terminated))
        while len(self.history) > self.window:
            self.history.popleft()

    # -- REF matcher.py:248-326 ------------------------------------------------------
    def accept_bytes(self, data: bytes) -> bool:
        if self.terminated:
            raise OracleMatcherError("matcher is terminated")
        if not data:
            self._push_history()
            self.tops = list(self.tops)
            return True
        out = self._sim(self.tops, data)
        if out is None:
            return False
        self._push_history()
        self.tops = out
        return True

    def accept_token(self, tid: int) -> bool:
        if self.terminated:
            raise OracleMatcherError("matcher is terminated")
        if not 0 <= tid < self.v.size:
            raise OracleMatcherError(f"token id {tid} out of range")
        if tid == self.v.eos_id:
            if not self.closed_facts()[0]:
                return False
            self._push_history()
            self.tops = list(self.tops)
            self.terminated = True
            return True
        if tid in self.v.special_tokens or not self.v.tokens[tid]:
            return False
        return self.accept_bytes(self.v.tokens[tid])

    def rollback(self, steps: int):
        if steps < 0 or steps > len(self.history):
            raise OracleMatcherError(f"cannot roll back {steps} steps (history {len(self.history)})")
        for _ in range(steps):
            self.tops, self.terminated = self.history.pop()

    def branch(self) -> "OracleMatcher":
        m = object.__new__(OracleMatcher)
        m.__dict__.update(self.__dict__)
        m.history = deque(self.history)
        m.tops = list(self.tops)
        return m

    def can_terminate(self) -> bool:
        return self.closed_facts()[0]

    # -- REF matcher.py:377-444 (Algorithm 1) ----------------------------------------------
    def fill(self) -> np.ndarray:
        if self.terminated:
            raise OracleMatcherError("matcher is terminated")
        if self.b.cache is None:
            words = self._fill_brute()
        else:
            words = self._fill_cached()
        if self.closed_facts()[0]:
            e = self.v.eos_id
            words[e >> 5] |= np.uint32(1 << (e & 31))
        tail = self.v.size & 31
        if tail:
            words[-1] &= np.uint32((1 << tail) - 1)
        return words

    def _fill_cached(self) -> np.ndarray:
        W = (self.v.size + 31) // 32
        prej = np.full(W, 0xFFFFFFFF, dtype=np.uint32)
        pacc = np.zeros(W, dtype=np.uint32)
        for h, n in self.tops:
            e = self.b.cache.entries[n]
            dacc, drej = self._resolve((h, n), e.dependent)
            if e.variant == REJECT_HEAVY:
                pacc |= pack_bits(np.concatenate([e.ids, np.asarray(dacc, np.uint32)]), self.v.size)
            elif e.variant == ACCEPT_HEAVY:
                prej &= pack_bits(np.concatenate([e.ids, np.asarray(drej, np.uint32)]), self.v.size)
            else:
                prej &= ~(e.bits | pack_bits(dacc, self.v.size))
        return ~(prej & ~pacc) & self.universe

    def _materialize(self, h):
        out = []
        while h != EMPTY:
            out.append(self.arena.node[h])
            h = self.arena.parent[h]
        return tuple(reversed(out))

    def _resolve(self, top, dep_ids):
        if not len(dep_ids):
            return [], []
        h, n = top
        content = [(self._materialize(h), n)]
        toks = self.v.tokens
        if len(dep_ids) > self.dep_threshold:
            if n not in self._dep_items:
                pairs = sorted((toks[t], int(t)) for t in dep_ids)
                items = [(t, b) for b, t in pairs]
                lcps = [0]
                for k in range(1, len(items)):
                    a, b = items[k - 1][1], items[k][1]
                    i = 0
                    while i < min(len(a), len(b)) and a[i] == b[i]:
                        i += 1
                    lcps.append(i)
                self._dep_items[n] = (items, lcps)
            items, lcps = self._dep_items[n]
            res = sweep(self.p, items, lcps, content, synthetic=False)
            return res.accepted, res.rejected
        acc, rej = [], []
        for t in dep_ids:
            res = sweep(self.p, [(int(t), toks[int(t)])], [0], content, synthetic=False)
            (acc if res.accepted else rej).append(int(t))
        return acc, rej

    def _fill_brute(self) -> np.ndarray:
        items, lcps, _ = sorted_items(self.v)
        contents = [(self._materialize(h), n) for h, n in self.tops]
        res = sweep(self.p, items, lcps, contents, synthetic=False)
        return pack_bits(np.asarray(res.accepted, dtype=np.uint32), self.v.size) & self.universe

    def jump_forward(self, max_len: int = 4096) -> bytes:
        """REF matcher.py:464-486."""
        m = self.branch()
        out = bytearray()
        while len(out) < max_len:
            term, fb = m.closed_facts()
            if term or bin(fb).count("1") != 1:
                break
            b = fb.bit_length() - 1
            if not m.accept_bytes(bytes([b])):
                break
            out.append(b)
        return bytes(out)


def brute_force_mask(p: OraclePda, vocab, consumed: bytes) -> list:
    """REF tests/conftest.py:149-159 over REF pda.py:583-585: the
    language-level ground truth (small vocabularies only)."""
    stacks = step_stacks(p, [(p.start_node(),)], consumed)
    out = [t for t in range(vocab.size)
           if t not in vocab.special_tokens and vocab.tokens[t] and step_stacks(p, stacks, vocab.tokens[t])]
    if stacks_accept(p, stacks):
        out.append(vocab.eos_id)
    return out


__all__ = ["OracleMatcher", "OracleBundle", "OracleMatcherError", "compile_oracle_bundle", "brute_force_mask",
           "OracleStateLimit"]

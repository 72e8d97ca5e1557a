"""Pure-Python interpreter of the device automaton tables (test helper).

Mirrors the semantics of the CUDA walker in
paper_2411_15100_b200/csrc/device.cuh (Walker::step, terminable) over a
CompiledTables, so CPU tests can check the host front end (language
equality against the oracle) without a GPU.  Never used by the product.
Stacks are tuples of return nodes plus the resting node."""

from __future__ import annotations


class TableSim:
    def __init__(self, t):
        self.t = t
        self.C = t.n_classes
        self.off = t.trans_off.tolist()
        self.tr = t.trans.tolist()
        self.pool = t.push_pool.tolist()
        self.flags = t.node_flags.tolist()
        self.cls = t.byte_class.tolist()

    def start(self):
        return frozenset([((), self.t.start_node)])

    def _trans(self, m, c):
        i = m * self.C + c
        for k in range(self.off[i], self.off[i + 1]):
            d, pk = self.tr[2 * k], self.tr[2 * k + 1] & 0xFFFFFFFF
            off, ln = pk & 0xFFFFFF, pk >> 24
            yield tuple(self.pool[off : off + ln]), d

    def step(self, states, b):
        """One byte from a set of (chain, node); returns (new set, popped_bottom)."""
        out = set()
        popped = False
        c = self.cls[b]
        for chain, m in states:
            while True:
                for P, d in self._trans(m, c):
                    ch = chain + P
                    if not P:
                        while (self.flags[d] & 2) and ch:
                            d, ch = ch[-1], ch[:-1]
                    out.add((ch, d))
                if not (self.flags[m] & 1):
                    break
                if not chain:
                    popped = True
                    break
                m, chain = chain[-1], chain[:-1]
        return frozenset(out), popped

    def walk(self, states, data):
        for b in data:
            states, _ = self.step(states, b)
            if not states:
                break
        return states

    def terminable(self, states):
        for chain, m in states:
            if (self.flags[m] & 1) and all(self.flags[r] & 1 for r in chain):
                return True
        return False

    def accepts(self, data):
        return self.terminable(self.walk(self.start(), data))

    def mask_ids(self, states, vocab_tokens, specials, eos):
        out = []
        for tid, tok in enumerate(vocab_tokens):
            if tid in specials or not tok:
                continue
            if self.walk(states, tok):
                out.append(tid)
        if self.terminable(states):
            out.append(eos)
        return sorted(out)

"""grammask-compatible adapter: the reference's own API over the B200 engine.

Names and behaviour of REF bundle.py:31-93 (CompileOptions, Bundle,
compile_bundle) and REF matcher.py:39-495 (TokenMask, Matcher), so the
reference's tests and decode loops can drive this engine by changing an
import.  Everything computes on the GPU; TokenMask is the host-side wire
format (u32 little-endian words, bit i%32 of word i//32 = token i, bits >= V
zero; REF matcher.py:39-100, docs/formats.md:7-12) that fill copies into.

Intentional differences (structure, never mask bits):
* ``merge=False`` still determinises rule automata (language-preserving);
  automaton statistics and stack counts therefore differ from the reference.
* ``cache=False`` marks every token context-dependent, so the fill kernel
  walks the whole vocabulary per step (the reference's brute-force path,
  REF matcher.py:446-460, on the GPU).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from .automaton import AutomatonOptions, StateLimitError
from .engine import DeviceVocab, MatcherError, compile_on_device
from .grammar import GrammarError
from .matcher import SlotMatcher
from .vocab import Vocabulary

__all__ = ["CompileOptions", "Bundle", "compile_bundle", "load_bundle", "save_bundle", "TokenMask", "Matcher",
           "MatcherError", "GrammarError", "StateLimitError"]


@dataclass
class CompileOptions:
    """REF bundle.py:31-52; cache off => ctx expansion off."""

    inline: bool = True
    merge: bool = True
    cache: bool = True
    ctx_expansion: bool = True
    inline_max_rule_size: int = 16
    inline_max_result_size: int = 512

    def __post_init__(self):
        if not self.cache:
            self.ctx_expansion = False


_DEVICE_VOCABS: dict = {}


def device_vocab(vocab: Vocabulary) -> DeviceVocab:
    key = (torch.cuda.current_device(), vocab.content_hash())
    dv = _DEVICE_VOCABS.get(key)
    if dv is None:
        dv = _DEVICE_VOCABS[key] = DeviceVocab(vocab)
    return dv


class _CompiledHandle:
    """Duck-typed CompiledGrammar for SlotMatcher."""

    def __init__(self, dev):
        self._dev = dev


@dataclass
class Bundle:
    grammar_text: str
    vocab_hash: bytes
    vocab_size: int
    options: CompileOptions
    compiled: object  # engine.CompiledDeviceGrammar; None until a Matcher binds a vocabulary (load_bundle)
    image: object = None  # bundle_io.BundleImage of a loaded GMB1 file (save_bundle writes it back verbatim)

    def ensure_compiled(self, vocab: Vocabulary):
        """Device-compile a loaded bundle's grammar for ``vocab`` (once)."""
        if self.compiled is None:
            aopts = AutomatonOptions(inline=self.options.inline, ctx_expansion=self.options.ctx_expansion)
            self.compiled = compile_on_device(self.grammar_text, device_vocab(vocab), aopts,
                                              uncached=not self.options.cache)
        return self.compiled

    @property
    def stats(self) -> dict:
        return self.compiled.stats

    @property
    def compile_ms(self) -> dict:
        return self.compiled.timings_ms


def compile_bundle(grammar_text: str, vocab: Vocabulary, options: Optional[CompileOptions] = None, *,
                   group=None) -> Bundle:
    """Parse, build the device automaton, run the K1/K1b cache build
    (REF bundle.py:65-93)."""
    opts = options or CompileOptions()
    aopts = AutomatonOptions(inline=opts.inline, ctx_expansion=opts.ctx_expansion)
    dv = device_vocab(vocab)
    dev = compile_on_device(grammar_text, dv, aopts, group=group, uncached=not opts.cache)
    return Bundle(grammar_text, vocab.content_hash(), vocab.size, opts, dev)


def _options_from_flags(flags: int) -> CompileOptions:
    from .bundle_io import FLAG_CACHE, FLAG_CTX, FLAG_INLINE, FLAG_MERGE

    return CompileOptions(inline=bool(flags & FLAG_INLINE), merge=bool(flags & FLAG_MERGE),
                          cache=bool(flags & FLAG_CACHE), ctx_expansion=bool(flags & FLAG_CTX))


def load_bundle(data: bytes) -> Bundle:
    """Read a GMB1 bundle (REF bundle.py:186-206).  The engine needs its
    normalized grammar text and option flags; the grammar is compiled on the
    device when a Matcher binds a vocabulary (the vocabulary hash is checked
    first, as the reference does).  The file's automaton and GMC1 sections
    are kept, so save_bundle returns the same bytes."""
    from .bundle_io import read_bundle

    img = read_bundle(data)
    return Bundle(img.grammar_text, img.vocab_hash, img.vocab_size, _options_from_flags(img.flags), None, img)


def save_bundle(bundle: Bundle) -> bytes:
    """GMB1 bytes of a bundle (REF bundle.py:167-183).  A loaded bundle is
    written back verbatim; one compiled here is exported with this engine's
    automaton as the PDA section (per-rule DFAs: byte-range and rule-call
    edges, rule starts and finals) and its device cache as the GMC1 section
    (per cache-key node: accepted / rejected / dependent ids in the adaptive
    byte-minimal encoding).  Deterministic for identical inputs."""
    from . import bundle_io as bio

    if bundle.image is not None:
        return bio.write_bundle(bundle.image)
    dev = bundle.compiled
    t = dev.tables
    o = bundle.options
    flags = ((bio.FLAG_INLINE if o.inline else 0) | (bio.FLAG_MERGE if o.merge else 0) |
             (bio.FLAG_CACHE if o.cache else 0) | (bio.FLAG_CTX if o.ctx_expansion else 0))
    class_bytes = [0] * t.n_classes
    for b in range(256):
        class_bytes[int(t.byte_class[b])] |= 1 << b
    edges = []
    for u in range(t.n_nodes):
        rows = t.raw[int(t.raw_off[u]):int(t.raw_off[u + 1])]
        by_dst: dict = {}
        for sym, dst in rows:
            if sym >= 0:
                by_dst[int(dst)] = by_dst.get(int(dst), 0) | class_bytes[int(sym)]
        for dst in sorted(by_dst):
            edges.append((u, dst, bio.EDGE_CHAR, bio.byte_ranges(by_dst[dst])))
        for sym, dst in rows:
            if sym < 0:
                edges.append((u, int(dst), bio.EDGE_RULE, int(-sym - 1)))
    rules = []
    for r in range(t.n_rules):
        finals = [u for u in range(t.n_nodes) if t.node_rule[u] == r and t.finals[u]]
        rules.append((t.rule_names[r], int(t.rule_start[r]), finals))
    pda = bio.PdaImage([int(x) for x in t.node_rule], edges, rules, int(t.root_rule))
    cache = None
    if o.cache:
        v = dev.dvocab.vocab
        acc_rows, dep_off, dep_ids = dev.cache.export()
        acc_bits = np.unpackbits(acc_rows.cpu().numpy().view(np.uint8), axis=1, bitorder="little")[:, : v.size]
        universe = np.asarray([i for i in range(v.size) if i not in v.special_tokens], dtype=np.uint32)
        entries = {}
        for k, node in enumerate(t.cache_keys):
            acc = np.nonzero(acc_bits[k])[0].astype(np.uint32)
            dep = np.asarray(dep_ids[dep_off[k]:dep_off[k + 1]], dtype=np.uint32)
            rej = np.setdiff1d(universe, np.concatenate([acc, dep]))
            entries[int(node)] = bio.choose_storage(acc, rej, dep, v.size)
        cache = bio.CacheImage(v.size, entries)
    return bio.write_bundle(bio.BundleImage(flags, bundle.vocab_size, bundle.vocab_hash, bundle.grammar_text, pda,
                                            cache))


class TokenMask:
    """Host bitset over the vocabulary (REF matcher.py:39-100)."""

    __slots__ = ("vocab_size", "words")

    def __init__(self, vocab_size: int, words: Optional[np.ndarray] = None):
        self.vocab_size = vocab_size
        n = (vocab_size + 31) // 32
        if words is None:
            words = np.zeros(n, dtype=np.uint32)
        elif len(words) != n:
            raise ValueError(f"expected {n} words, got {len(words)}")
        self.words = words

    def _trim(self):
        tail = self.vocab_size & 31
        if tail and len(self.words):
            self.words[-1] &= np.uint32((1 << tail) - 1)

    def is_allowed(self, tid: int) -> bool:
        return bool((int(self.words[tid >> 5]) >> (tid & 31)) & 1)

    def set_bit(self, tid: int):
        self.words[tid >> 5] |= np.uint32(1 << (tid & 31))

    def clear(self):
        self.words[:] = 0

    def count(self) -> int:
        return int(np.unpackbits(self.words.view(np.uint8)).sum())

    def allowed_ids(self) -> np.ndarray:
        bits = np.unpackbits(self.words.view(np.uint8), bitorder="little")[: self.vocab_size]
        return np.nonzero(bits)[0]

    def to_bytes(self) -> bytes:
        return self.words.astype("<u4").tobytes()

    @classmethod
    def from_bytes(cls, vocab_size: int, data: bytes) -> "TokenMask":
        return cls(vocab_size, np.frombuffer(data, dtype="<u4").astype(np.uint32))

    def to_hex(self) -> str:
        return self.to_bytes().hex()

    def copy(self) -> "TokenMask":
        return TokenMask(self.vocab_size, self.words.copy())

    def __eq__(self, other) -> bool:
        return (isinstance(other, TokenMask) and self.vocab_size == other.vocab_size
                and bool(np.array_equal(self.words, other.words)))

    __hash__ = None


class Matcher:
    """REF matcher.py:103-495 over a device slot."""

    def __init__(self, bundle: Bundle, vocab: Vocabulary, history_window: int = 32, *,
                 branch_cap: int = 4096, dependent_sweep_threshold: int = 64, _core: Optional[SlotMatcher] = None):
        if bundle.vocab_hash != vocab.content_hash():
            raise MatcherError(
                f"vocabulary does not match bundle (hash {vocab.content_hash().hex()[:12]}... "
                f"vs bundle {bundle.vocab_hash.hex()[:12]}...)"
            )
        del branch_cap, dependent_sweep_threshold  # device walker limits are fixed
        self._bundle = bundle
        self._v = vocab
        if _core is None:
            bundle.ensure_compiled(vocab)
        self._core = _core if _core is not None else SlotMatcher(_CompiledHandle(bundle.compiled), history_window)
        self._closed = False
        self._row = torch.empty((1, (vocab.size + 31) // 32), dtype=torch.int32, device=self._core.pool.device)

    def _check_open(self):
        if self._closed:
            raise MatcherError("matcher is closed")

    # -- accepting ---------------------------------------------------------------
    def accept_bytes(self, data: bytes) -> bool:
        self._check_open()
        return self._core.accept_bytes(bytes(data))

    def accept_token(self, tid: int) -> bool:
        self._check_open()
        if not 0 <= tid < self._v.size:
            raise MatcherError(f"token id {tid} out of range")
        return self._core.accept_token(tid)

    # -- rollback / branching -------------------------------------------------------
    @property
    def history_depth(self) -> int:
        return self._core.info()["history_len"]

    @property
    def terminated(self) -> bool:
        return self._core.info()["terminated"]

    def can_terminate(self) -> bool:
        self._check_open()
        return self._core.info()["terminable"]

    def rollback(self, steps: int):
        self._check_open()
        if steps < 0 or steps > self.history_depth:
            raise MatcherError(f"cannot roll back {steps} steps (history {self.history_depth})")
        if steps:
            self._core.rollback(steps)

    def branch(self) -> "Matcher":
        self._check_open()
        m = Matcher.__new__(Matcher)
        m._bundle, m._v, m._closed = self._bundle, self._v, False
        m._core = self._core.fork()
        m._row = torch.empty_like(self._row)
        return m

    def close(self):
        if not self._closed:
            self._closed = True
            self._core.release()

    # -- masks -------------------------------------------------------------------------
    def next_token_mask(self) -> TokenMask:
        out = TokenMask(self._v.size)
        self.fill_next_token_mask(out)
        return out

    def fill_next_token_mask(self, out: TokenMask):
        self._check_open()
        if out.vocab_size != self._v.size:
            raise MatcherError("mask size does not match the vocabulary")
        if self._core.info()["terminated"]:
            raise MatcherError("matcher is terminated")
        self._core.fill_row(self._row, 0, need_apply=False)
        out.words[:] = self._row[0].cpu().numpy().view(np.uint32)
        self._core.check()  # this request's device error (e.g. over the 4096-stack cap), REF matcher.py:188-189

    def fill_device_row(self, bitmask: torch.Tensor, index: int = 0):
        """Fill bitmask[index] in HBM without the host copy."""
        self._check_open()
        self._core.fill_row(bitmask, index, need_apply=False)

    # -- jump-forward / introspection --------------------------------------------------
    def find_jump_forward_bytes(self, max_len: int = 4096) -> bytes:
        self._check_open()
        if self._core.info()["terminated"]:
            raise MatcherError("matcher is terminated")
        return self._core.jump_forward(max_len)

    def stack_count(self) -> int:
        return self._core.info()["n_stacks"]

    def stack_contents(self) -> list:
        return sorted(self._core.materialize(h) + (n,) for h, n in self._core.info()["stacks"])

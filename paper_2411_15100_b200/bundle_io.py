"""GMB1 bundle / GMC1 mask-cache files.

Reader and writer for the reference's on-disk formats (REF docs/formats.md:
14-57; REF bundle.py:101-206, cache.py:418-486): little-endian, deterministic,
re-serialising a parsed file reproduces its bytes.  ``compat.load_bundle``
turns a reference bundle into a device-compiled one (the normalized grammar
text and the option flags are all the engine needs; the reference's PDA and
cache sections are kept verbatim so ``compat.save_bundle`` writes the same
bytes back), and ``export_bundle`` writes a bundle for a grammar compiled
here, with this engine's automaton as the PDA section and its device cache as
the GMC1 section (per-node accepted / rejected / dependent ids in the
reference's byte-minimal adaptive encoding, REF cache.py:384-402).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

__all__ = ["PdaImage", "CacheEntry", "CacheImage", "BundleImage", "read_bundle", "write_bundle", "read_cache",
           "write_cache", "choose_storage", "FLAG_INLINE", "FLAG_MERGE", "FLAG_CACHE", "FLAG_CTX"]

BUNDLE_MAGIC, BUNDLE_VERSION = b"GMB1", 1
CACHE_MAGIC, CACHE_VERSION = b"GMC1", 1
FLAG_INLINE, FLAG_MERGE, FLAG_CACHE, FLAG_CTX = 1, 2, 4, 8
EDGE_EPS, EDGE_CHAR, EDGE_RULE = 0, 1, 2
ACCEPT_HEAVY, REJECT_HEAVY, BITSET_FORM = 0, 1, 2


@dataclass
class PdaImage:
    """The automaton section: nodes, edges (src, dst, kind, data), rules
    (name, start, sorted finals), root rule id."""

    node_rule: List[int]
    edges: List[Tuple[int, int, int, object]]  # data: byte ranges (CHAR), rule id (RULE), None (EPS)
    rules: List[Tuple[str, int, List[int]]]
    root: int

    @property
    def node_count(self) -> int:
        return len(self.node_rule)


@dataclass
class CacheEntry:
    variant: int
    ids: np.ndarray            # rejected ids (accept-heavy) / accepted ids (reject-heavy)
    bits: Optional[np.ndarray]  # accepted bitset words (bitset form)
    dependent: np.ndarray


@dataclass
class CacheImage:
    vocab_size: int
    entries: Dict[int, CacheEntry] = field(default_factory=dict)


@dataclass
class BundleImage:
    flags: int
    vocab_size: int
    vocab_hash: bytes
    grammar_text: str
    pda: PdaImage
    cache: Optional[CacheImage]


class _Reader:
    def __init__(self, data: bytes, pos: int = 0):
        self.data = data
        self.pos = pos

    def take(self, fmt: str):
        try:
            vals = struct.unpack_from(fmt, self.data, self.pos)
        except struct.error as e:
            raise ValueError(f"truncated file: {e}") from None
        self.pos += struct.calcsize(fmt)
        return vals

    def take_bytes(self, n: int) -> bytes:
        if self.pos + n > len(self.data):
            raise ValueError("truncated file")
        raw = self.data[self.pos:self.pos + n]
        self.pos += n
        return raw

    def take_str(self) -> str:
        (n,) = self.take("<I")
        return self.take_bytes(n).decode("utf-8")

    def take_u32s(self, n: int) -> np.ndarray:
        return np.frombuffer(self.take_bytes(4 * n), dtype="<u4").astype(np.uint32)


def _pack_str(s: str) -> bytes:
    raw = s.encode("utf-8")
    return struct.pack("<I", len(raw)) + raw


# ---------------------------------------------------------------- GMC1

def read_cache(data: bytes) -> CacheImage:
    if data[:4] != CACHE_MAGIC:
        raise ValueError("not a mask cache blob")
    r = _Reader(data, 4)
    version, vocab_size, n_entries = r.take("<III")
    if version != CACHE_VERSION:
        raise ValueError(f"unsupported cache version {version}")
    entries = {}
    for _ in range(n_entries):
        node, variant = r.take("<IB")
        (n,) = r.take("<I")
        vals = r.take_u32s(n)
        (nd,) = r.take("<I")
        dep = r.take_u32s(nd)
        if variant == BITSET_FORM:
            entries[node] = CacheEntry(variant, np.zeros(0, dtype=np.uint32), vals, dep)
        elif variant in (ACCEPT_HEAVY, REJECT_HEAVY):
            entries[node] = CacheEntry(variant, vals, None, dep)
        else:
            raise ValueError(f"unknown cache entry variant {variant}")
    return CacheImage(vocab_size, entries)


def write_cache(c: CacheImage) -> bytes:
    out = [CACHE_MAGIC, struct.pack("<III", CACHE_VERSION, c.vocab_size, len(c.entries))]
    for node in sorted(c.entries):
        e = c.entries[node]
        out.append(struct.pack("<IB", node, e.variant))
        vals = e.bits if e.variant == BITSET_FORM else e.ids
        vals = np.asarray(vals, dtype="<u4")
        out.append(struct.pack("<I", len(vals)))
        out.append(vals.tobytes())
        dep = np.asarray(e.dependent, dtype="<u4")
        out.append(struct.pack("<I", len(dep)))
        out.append(dep.tobytes())
    return b"".join(out)


def _variant_size(variant: int, n_ids: int, n_dep: int, vocab_size: int) -> int:
    if variant == BITSET_FORM:
        return (vocab_size + 7) // 8 + 4 * n_dep
    return 4 * (n_ids + n_dep)


def choose_storage(accepted, rejected, dependent, vocab_size: int) -> CacheEntry:
    """Byte-minimal encoding, ties accept-heavy, reject-heavy, bitset
    (REF cache.py:384-402, docs/formats.md:30-33)."""
    acc = np.unique(np.asarray(accepted, dtype=np.uint32))
    rej = np.unique(np.asarray(rejected, dtype=np.uint32))
    dep = np.unique(np.asarray(dependent, dtype=np.uint32))
    sizes = (_variant_size(ACCEPT_HEAVY, len(rej), len(dep), vocab_size),
             _variant_size(REJECT_HEAVY, len(acc), len(dep), vocab_size),
             _variant_size(BITSET_FORM, 0, len(dep), vocab_size))
    v = min(range(3), key=lambda i: sizes[i])
    if v == ACCEPT_HEAVY:
        return CacheEntry(ACCEPT_HEAVY, rej, None, dep)
    if v == REJECT_HEAVY:
        return CacheEntry(REJECT_HEAVY, acc, None, dep)
    words = np.zeros((vocab_size + 31) // 32, dtype=np.uint32)
    if len(acc):
        np.bitwise_or.at(words, acc >> 5, np.uint32(1) << (acc & np.uint32(31)))
    return CacheEntry(BITSET_FORM, np.zeros(0, dtype=np.uint32), words, dep)


# ---------------------------------------------------------------- GMB1

def _read_pda(r: _Reader) -> PdaImage:
    n_nodes, n_edges, n_rules = r.take("<III")
    (root,) = r.take("<I")
    node_rule = [int(x) for x in r.take_u32s(n_nodes)]
    edges = []
    for _ in range(n_edges):
        src, dst, kind = r.take("<IIB")
        if kind == EDGE_CHAR:
            (n,) = r.take("<H")
            data = tuple(r.take("<BB") for _ in range(n))
        elif kind == EDGE_RULE:
            data = r.take("<I")[0]
        elif kind == EDGE_EPS:
            data = None
        else:
            raise ValueError(f"unknown edge kind {kind}")
        edges.append((src, dst, kind, data))
    rules = []
    for _ in range(n_rules):
        name = r.take_str()
        start, nf = r.take("<II")
        rules.append((name, start, [int(x) for x in r.take_u32s(nf)]))
    return PdaImage(node_rule, edges, rules, root)


def _write_pda(p: PdaImage) -> bytes:
    out = [struct.pack("<III", p.node_count, len(p.edges), len(p.rules)), struct.pack("<I", p.root)]
    out.append(np.asarray(p.node_rule, dtype="<u4").tobytes())
    for src, dst, kind, data in p.edges:
        out.append(struct.pack("<IIB", src, dst, kind))
        if kind == EDGE_CHAR:
            out.append(struct.pack("<H", len(data)))
            out.append(b"".join(struct.pack("<BB", lo, hi) for lo, hi in data))
        elif kind == EDGE_RULE:
            out.append(struct.pack("<I", data))
    for name, start, finals in p.rules:
        out.append(_pack_str(name))
        out.append(struct.pack("<II", start, len(finals)))
        out.append(np.asarray(sorted(finals), dtype="<u4").tobytes())
    return b"".join(out)


def read_bundle(data: bytes) -> BundleImage:
    if data[:4] != BUNDLE_MAGIC:
        raise ValueError("not a grammask bundle")
    r = _Reader(data, 4)
    version, flags = r.take("<II")
    if version != BUNDLE_VERSION:
        raise ValueError(f"unsupported bundle version {version}")
    (vocab_size,) = r.take("<I")
    vocab_hash = r.take_bytes(32)
    text = r.take_str()
    (pda_len,) = r.take("<I")
    pr = _Reader(r.take_bytes(pda_len))
    pda = _read_pda(pr)
    if pr.pos != pda_len:
        raise ValueError("trailing bytes in the automaton section")
    (cache_len,) = r.take("<I")
    cache = read_cache(r.take_bytes(cache_len)) if cache_len else None
    return BundleImage(flags, vocab_size, vocab_hash, text, pda, cache)


def write_bundle(b: BundleImage) -> bytes:
    out = [BUNDLE_MAGIC, struct.pack("<II", BUNDLE_VERSION, b.flags), struct.pack("<I", b.vocab_size), b.vocab_hash,
           _pack_str(b.grammar_text)]
    pda = _write_pda(b.pda)
    out += [struct.pack("<I", len(pda)), pda]
    if b.cache is not None:
        blob = write_cache(b.cache)
        out += [struct.pack("<I", len(blob)), blob]
    else:
        out.append(struct.pack("<I", 0))
    return b"".join(out)


def byte_ranges(mask: int) -> Tuple[Tuple[int, int], ...]:
    """Sorted disjoint (lo, hi) byte ranges of a 256-bit mask."""
    out, b = [], 0
    while b < 256:
        if (mask >> b) & 1:
            lo = b
            while b + 1 < 256 and (mask >> (b + 1)) & 1:
                b += 1
            out.append((lo, b))
        b += 1
    return tuple(out)

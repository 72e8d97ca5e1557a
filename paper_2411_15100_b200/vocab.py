"""Vocabulary model, JSON loader and the synthetic workload vocabulary.

* ``Vocabulary`` carries token bytes, special ids (always including EOS) and
  the sha256 content hash used to refuse mismatched bundles
  (REF vocab.py:111-145, matcher.py:118-122).
* ``loads_vocab`` reads the reference's vocabulary JSON format
  (REF vocab.py:148-175, docs/formats.md:59-72): ``\\xHH`` and ``\\\\`` are
  resolved after JSON decoding; ``byte_level`` uses the GPT-2 printable-byte
  table.
* ``synth_vocab`` regenerates the reference's deterministic byte-level-BPE
  shaped vocabulary (REF synthvocab.py:63-154) — the bench and parity
  workloads are defined on it, so it must be identical token for token; the
  content hash is pinned in tests/golden.
"""

from __future__ import annotations

import hashlib
import json
import random
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

__all__ = ["VocabError", "Vocabulary", "vocab_from_tokens", "loads_vocab", "load_vocab", "synth_vocab",
           "BYTE_LEVEL_DECODE"]


class VocabError(ValueError):
    """Malformed vocabulary."""


def _gpt2_byte_table():
    printable = [*range(0x21, 0x7F), *range(0xA1, 0xAD), *range(0xAE, 0x100)]
    enc = {b: chr(b) for b in printable}
    extra = 0
    for b in range(256):
        if b not in enc:
            enc[b] = chr(0x100 + extra)
            extra += 1
    return enc, {c: b for b, c in enc.items()}


BYTE_LEVEL_ENCODE, BYTE_LEVEL_DECODE = _gpt2_byte_table()


@dataclass(frozen=True)
class Vocabulary:
    tokens: tuple
    special_tokens: frozenset
    eos_id: int

    @property
    def size(self) -> int:
        return len(self.tokens)

    def is_special(self, tid: int) -> bool:
        return tid in self.special_tokens

    def content_hash(self) -> bytes:
        """sha256 over b"VOC1", eos, sorted specials, "|", len-prefixed tokens
        (REF vocab.py:124-134)."""
        h = hashlib.sha256(b"VOC1")
        h.update(int(self.eos_id).to_bytes(4, "little"))
        h.update(b"".join(int(t).to_bytes(4, "little") for t in sorted(self.special_tokens)))
        h.update(b"|")
        h.update(b"".join(len(t).to_bytes(4, "little") + t for t in self.tokens))
        return h.digest()

    def packed(self):
        """(bytes uint8[], offsets int64[V+1]) for the C ABI."""
        lens = np.fromiter((len(t) for t in self.tokens), dtype=np.int64, count=self.size)
        off = np.zeros(self.size + 1, dtype=np.int64)
        np.cumsum(lens, out=off[1:])
        data = np.frombuffer(b"".join(self.tokens), dtype=np.uint8) if off[-1] else np.zeros(1, np.uint8)
        return data, off


def vocab_from_tokens(tokens: Iterable, eos_id: int, special: Sequence[int] = ()) -> Vocabulary:
    toks = tuple(bytes(t) for t in tokens)
    if not 0 <= eos_id < len(toks):
        raise VocabError(f"eos_id {eos_id} outside vocabulary of size {len(toks)}")
    spec = frozenset(special) | {eos_id}
    if any(not 0 <= s < len(toks) for s in spec):
        raise VocabError("special token id outside vocabulary")
    return Vocabulary(toks, spec, eos_id)


def _unescape(s: str) -> bytes:
    out = bytearray()
    i, n = 0, len(s)
    while i < n:
        if s[i] == "\\" and i + 1 < n:
            if s[i + 1] == "x":
                hx = s[i + 2 : i + 4]
                if len(hx) == 2 and all(c in "0123456789abcdefABCDEF" for c in hx):
                    out.append(int(hx, 16))
                    i += 4
                    continue
            elif s[i + 1] == "\\":
                out.append(0x5C)
                i += 2
                continue
        out += s[i].encode("utf-8")
        i += 1
    return bytes(out)


def loads_vocab(text: str) -> Vocabulary:
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as exc:
        raise VocabError(f"vocabulary is not valid JSON: {exc}") from exc
    if not isinstance(doc, dict) or "tokens" not in doc:
        raise VocabError("vocabulary must be an object with a 'tokens' array")
    raw = doc["tokens"]
    if not isinstance(raw, list) or not all(isinstance(t, str) for t in raw):
        raise VocabError("'tokens' must be an array of strings")
    if "eos_id" not in doc:
        raise VocabError("vocabulary is missing 'eos_id'")
    if doc.get("byte_level", False):
        toks = []
        for i, s in enumerate(raw):
            try:
                toks.append(bytes(BYTE_LEVEL_DECODE[c] for c in s))
            except KeyError as exc:
                raise VocabError(f"token {i}: character {exc.args[0]!r} is not in the byte-level table") from None
    else:
        toks = [_unescape(s) for s in raw]
    special = doc.get("special", [])
    if not isinstance(special, list) or not all(isinstance(x, int) for x in special):
        raise VocabError("'special' must be an array of token ids")
    if len(set(special)) != len(special):
        raise VocabError("duplicate ids in 'special'")
    return vocab_from_tokens(toks, doc["eos_id"], special)


def load_vocab(path) -> Vocabulary:
    with open(path, encoding="utf-8") as fh:
        return loads_vocab(fh.read())


# ---------------------------------------------------------------------------
# synthetic vocabulary (workload generator; REF synthvocab.py:63-154)

_C = "bcdfghjklmnpqrstvwz"
_V = "aeiouy"
_SUFFIX = ["", "s", "ing", "ed", "er", "ly", "tion", "ment"]
_WS = [b" " * k for k in range(2, 9)] + [b"\n", b"\n\n", b"\t", b"\r\n", b" \n", b"\n ", b"\t\t"]
_PUNCT = [
    b". ", b", ", b"! ", b"? ", b"; ", b": ", b"'s", b"' ", b" (", b") ", b"--", b"...", b".\n", b",\n",
    b" - ", b"n't", b"'re", b"'ve",
    b'":', b'",', b'"}', b'"]', b'" ', b'":"', b'": ', b'{"', b', "', b'},', b'],', b'"",', b'ively"',
    b'="', b'()', b'");', b'%,', b'\\"',
]
_QWORDS = ["the", "and", "for", "with", "that", "name", "value", "data", "true", "this", "type", "id", "key",
           "a", "b", "c", "x", "n", "to", "of", "in", "is", "it", "on"]
_UTF8 = ["é", "ü", "ñ", "ç", "ß", "→", "…", "–", "°", "€", "中", "文", "日", "語", " é", " ü", "ä", "ö", "è", "à"]
_FRAGS = [b"\xc3", b"\xe2\x80", b"\xf0\x9f", b"\xe2", b"\xc2"]
_DIGITS = [b"0,", b"1,", b"0.", b"1.", b"2:", b"1]", b"2}", b"3a", b" 1", b" 2"]
_BRACKETS = [b"[1", b"[0", b"[[", b"]]", b"[ ", b" [", b"{ ", b" {", b"}\n", b"]\n", b"()", b"(s", b")(",
             b"[i", b"{}", b"[]"]


def _syllables(rng: random.Random, with_suffix: bool) -> str:
    parts = []
    for _ in range(rng.choice((1, 1, 2, 2, 2, 3, 3, 4))):
        parts += [rng.choice(_C), rng.choice(_V)]
        if rng.random() < 0.3:
            parts.append(rng.choice(_C))
    w = "".join(parts)
    return w + rng.choice(_SUFFIX) if with_suffix else w


def synth_vocab(size: int = 32000, seed: int = 23917, profile: str = "text") -> Vocabulary:
    """Deterministic synthetic byte-level vocabulary of exactly ``size``
    tokens; ids 0..255 are the single bytes, the last three ids are the
    specials <unk>, <pad>, <eos> (EOS last)."""
    if size < 512:
        raise ValueError("synthetic vocabularies start at 512 tokens")
    counts = {"text": (12, 24, 12, 48, 6)}
    if profile == "mixed":
        counts["mixed"] = (int(size * 0.02), int(size * 0.012), int(size * 0.008), int(size * 0.03), 14)
    if profile not in counts:
        raise ValueError(f"unknown profile {profile!r}")
    n_digit, n_quote, n_bracket, n_punct, n_ws = counts[profile]
    rng = random.Random(seed)
    toks = [bytes([b]) for b in range(256)]
    have = set(toks)

    def put(t: bytes):
        if t and t not in have:
            have.add(t)
            toks.append(t)

    for t in _WS[:n_ws]:
        put(t)
    for i in range(n_digit):
        put(_DIGITS[i] if i < len(_DIGITS)
            else "".join(rng.choice("0123456789") for _ in range(rng.choice((2, 2, 3, 4)))).encode())
    quotes = ['"' + w for w in _QWORDS] + [w + '"' for w in _QWORDS[:8]]
    for i in range(n_quote):
        put(quotes[i].encode() if i < len(quotes) else ('"' + _syllables(rng, True)).encode())
    for i in range(n_bracket):
        put(_BRACKETS[i] if i < len(_BRACKETS) else (rng.choice("[{(") + _syllables(rng, True)[:3]).encode())
    for i in range(n_punct):
        put(_PUNCT[i] if i < len(_PUNCT) else (_syllables(rng, True)[:4] + rng.choice(".,;:!?")).encode())
    for s in _UTF8:
        put(s.encode())
    for t in _FRAGS:
        put(t)
    limit = size - 3
    while len(toks) < limit:
        stem = _syllables(rng, False)
        forms = [stem] + [stem + e for e in rng.sample(_SUFFIX[1:], k=rng.randrange(1, 4))]
        chosen = []
        for w in forms:
            r = rng.random()
            if r < 0.45:
                chosen.append(" " + w)
            elif r < 0.55:
                chosen += [w.capitalize(), " " + w]
            else:
                chosen.append(w)
        for w in chosen:
            if len(toks) < limit:
                put(w.encode())
    toks = toks[:limit] + [b"<unk>", b"<pad>", b"<eos>"]
    return vocab_from_tokens(toks, eos_id=size - 1, special=[size - 3, size - 2, size - 1])

"""Test workloads: the reference's fixture vocabularies and grammars.

toy200 / gen vocabularies restate REF tests/conftest.py:24-68 (their content
hashes are pinned in golden/vocab_hashes.json); grammar texts come from
golden/languages.json (written by tools/make_golden.py from the reference).
"""

from __future__ import annotations

import gzip
import json
import random
from functools import lru_cache
from pathlib import Path

from paper_2411_15100_b200.vocab import synth_vocab, vocab_from_tokens

GOLDEN = Path(__file__).resolve().parent / "golden"


def build_toy200():
    toks = [bytes([b]) for b in range(0x20, 0x7F)] + [b"\n", b"\t", b"\r"]
    words = ("true false null tr ue als ll ab abc cat dog read ready reader").split()
    words += ['":', '",', '"}', '"]', '{"', '["', '"a"', '"b', "], ", "}, ", ", ", ": ", '": ', "[]", "{}",
              "[[", "]]", "12", "34", "3.5", "-1", "0.", "e+", "1e9", "00", "+(", ")*", ")+", "((", "))", "*(",
              "<a>", "</a>", "<b>", "</b>", "<a", "a>", "</", "get_weather", "get_time", "name", "unit", "count",
              "tags", '\\"', "\\n", "\\u00", "u00", "  ", "   ", " \n"]
    toks += [w.encode() for w in words]
    out, seen = [], set()
    for t in toks:
        if t not in seen:
            seen.add(t)
            out.append(t)
    rng = random.Random(99)
    syll = ["ta", "mi", "ro", "zen", "ki", "la", "vo", "nu", "pe", "sh"]
    while len(out) < 199:
        w = "".join(rng.choice(syll) for _ in range(rng.randrange(1, 4))).encode()
        if w not in seen:
            seen.add(w)
            out.append(w)
    return vocab_from_tokens(out[:199] + [b"<eos>"], eos_id=199, special=[199])


def build_gen_vocab():
    singles = 'acefghilmnorstuw_012[]{},:.+-*/()<>"\\ \n'
    toks = [c.encode() for c in singles] + [w.encode() for w in ["true", "false", "null", "get_weather", "get_time"]]
    toks += [c.encode() for c in ['":', '",', '"}', '"]', "},", "],", "</", "</a>", "</b>", "a>", "b>", ")*", ")+", "))"]]
    return vocab_from_tokens(toks + [b"<eos>"], eos_id=len(toks), special=[len(toks)])


@lru_cache(maxsize=None)
def vocab_by_name(name: str):
    if name == "toy200":
        return build_toy200()
    if name == "gen":
        return build_gen_vocab()
    size, prof = name.split(":")
    return synth_vocab(int(size), profile=prof)


@lru_cache(maxsize=None)
def languages() -> dict:
    return json.loads((GOLDEN / "languages.json").read_text())


def grammar_text(name: str) -> str:
    lang = languages()
    if name in lang["grammars"]:
        return lang["grammars"][name]
    return lang["extra_grammars"][name]


def mask_fixtures():
    return sorted(p.name for p in GOLDEN.glob("masks_*.json.gz"))


@lru_cache(maxsize=None)
def load_fixture(fname: str) -> dict:
    with gzip.open(GOLDEN / fname, "rt", encoding="utf-8") as fh:
        return json.load(fh)

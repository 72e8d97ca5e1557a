"""Generate tests/golden/* from the REAL reference (grammask), imported from
/root/reference/pkg/src.  Run here (the reference does not exist on the GPU
box):

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden.py

Fixtures written (all deterministic, seeded):
  vocab_hashes.json    content hashes of synth_vocab sizes/profiles
  masks_<name>.json.gz per (grammar, vocabulary): token trajectories and the
                       reference's mask after every prefix, as full hex words
                       (small vocabularies) or sha256 + popcount (large)
  languages.json       oracle_accepts verdicts for probe strings, and
                       grammar/schema error cases with the reference's
                       exception class and message
"""

from __future__ import annotations

import gzip
import hashlib
import itertools
import json
import random
import sys
import time
import zlib
from pathlib import Path

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

from conftest import build_gen_vocab, build_toy200, FIVE_GRAMMARS, PROBE_ALPHABETS  # noqa: E402
from grammask.bundle import compile_bundle  # noqa: E402
from grammask.grammar import GrammarError, parse_grammar  # noqa: E402
from grammask.grammars import ARITHMETIC, JSON_ECMA404, SAMPLE_SCHEMA, XML_TOY  # noqa: E402
from grammask.matcher import Matcher, TokenMask  # noqa: E402
from grammask.pda import StateLimitError, build_pda, oracle_accepts  # noqa: E402
from grammask.schema import SchemaError, schema_to_grammar_text  # noqa: E402
from grammask.synthvocab import synth_vocab  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def mask_record(mask: TokenMask, full: bool) -> dict:
    raw = mask.to_bytes()
    rec = {"sha256": hashlib.sha256(raw).hexdigest(), "count": mask.count()}
    if full:
        rec["hex"] = raw.hex()
    return rec


def structured_pick(ids, vocab, rng, bias):
    """Structure-biased sampler (SURVEY §7 hard part 7): prefer short tokens
    made of structural bytes with probability ``bias``."""
    structural = set(b'{}[]",:<>/()+-*0123456789 ')
    if rng.random() < bias:
        short = [t for t in ids if t != vocab.eos_id and 0 < len(vocab.tokens[t]) <= 3
                 and all(c in structural for c in vocab.tokens[t])]
        if short:
            return int(short[rng.randrange(len(short))])
    return int(ids[rng.randrange(len(ids))])


def trajectories(bundle, vocab, n_traj, max_steps, seed, bias, full):
    rng = random.Random(seed)
    out = []
    for _ in range(n_traj):
        m = Matcher(bundle, vocab, history_window=1)
        toks, masks = [], []
        for _ in range(max_steps):
            mask = m.next_token_mask()
            masks.append(mask_record(mask, full))
            ids = mask.allowed_ids()
            if len(ids) == 0:
                break
            pick = structured_pick(ids, vocab, rng, bias)
            toks.append(pick)
            if pick == vocab.eos_id:
                break
            assert m.accept_token(pick)
        out.append({"tokens": toks, "masks": masks, "terminable_end": None})
    return out


def write_gz(name, doc):
    with gzip.open(OUT / name, "wt", encoding="utf-8") as fh:
        json.dump(doc, fh, separators=(",", ":"))


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    t0 = time.time()
    # 1. vocab hashes
    vh = {}
    for size, prof in [(512, "text"), (4000, "mixed"), (32000, "text"), (32000, "mixed"), (128256, "text")]:
        vh[f"{size}:{prof}"] = synth_vocab(size, profile=prof).content_hash().hex()
    toy, gen = build_toy200(), build_gen_vocab()
    vh["toy200"] = toy.content_hash().hex()
    vh["gen"] = gen.content_hash().hex()
    (OUT / "vocab_hashes.json").write_text(json.dumps(vh, indent=1) + "\n")

    grammars = dict(FIVE_GRAMMARS)
    # 2. small vocabularies: full masks
    for vname, vocab in [("toy200", toy), ("gen", gen)]:
        for gname, text in grammars.items():
            b = compile_bundle(text, vocab)
            trajs = []
            for bias in (0.0, 0.7):
                trajs += trajectories(b, vocab, 12, 24, seed=zlib.crc32(f"{gname}:{bias}".encode()) % 1000 + 7, bias=bias, full=True)
            write_gz(f"masks_{gname}_{vname}.json.gz", {"grammar": gname, "vocab": vname, "trajectories": trajs})
            print(vname, gname, f"{time.time() - t0:.1f}s", flush=True)

    # 3. synthetic vocabularies: digests
    plan = [
        ("json", JSON_ECMA404, 32000, "text", 4, 120),
        ("schema", schema_to_grammar_text(SAMPLE_SCHEMA), 32000, "text", 4, 80),
        ("arithmetic", ARITHMETIC, 32000, "text", 3, 80),
        ("xml", XML_TOY, 32000, "text", 3, 60),
        ("json", JSON_ECMA404, 4000, "mixed", 6, 100),
        ("json", JSON_ECMA404, 128256, "text", 2, 60),
        ("schema", schema_to_grammar_text(SAMPLE_SCHEMA), 128256, "text", 2, 40),
    ]
    for gname, text, size, prof, n_traj, steps in plan:
        vocab = synth_vocab(size, profile=prof)
        b = compile_bundle(text, vocab)
        trajs = []
        for i, bias in enumerate((0.0, 0.7)):
            trajs += trajectories(b, vocab, n_traj // 2 or 1, steps, seed=1000 + i, bias=bias, full=False)
        write_gz(f"masks_{gname}_{size}_{prof}.json.gz",
                 {"grammar": gname, "vocab": f"{size}:{prof}", "trajectories": trajs,
                  "ref_stats": {"entries": b.cache.stats.entry_count,
                                "dependent_total": b.cache.stats.dependent_total}})
        print(gname, size, prof, f"{time.time() - t0:.1f}s", flush=True)

    # 4. languages + error KATs
    lang = {"accepts": [], "errors": []}
    for gname, text in grammars.items():
        p = build_pda(parse_grammar(text))
        alpha = PROBE_ALPHABETS[gname]
        rng = random.Random(5)
        probes = set()
        for n in range(0, 5):
            for tup in itertools.product(alpha, repeat=n):
                probes.add(bytes(tup))
        for _ in range(300):
            probes.add(bytes(rng.choice(alpha) for _ in range(rng.randrange(5, 12))))
        for s in sorted(probes):
            lang["accepts"].append([gname, s.hex(), oracle_accepts(p, s)])
    extra = {
        "utf8class": 'root ::= [a-zé-ü中\\u00ff-\\u0101]+',
        "negated": 'root ::= "\\"" [^"\\\\]* "\\""',
        "bytes": 'root ::= "\\xC3" [\\x80-\\xBF] | "ab"{2,3} "c"?',
        "escapes": 'root ::= "\\n\\t\\r\\\'\\u00e9" [\\]\\-\\^\\[]+ [-a] [a-] []x]',
        "empty": 'root ::= "" | "a" b\nb ::= ""',
        "repeat": 'root ::= ("ab" | "c"){1,3} "d"{0,2} ("e"+)?',
    }
    for ename, text in extra.items():
        p = build_pda(parse_grammar(text))
        alpha = sorted(set(b"abcde\"\\\n\t\r'\xc3\xa9\x80\xbf]-^[x") | set("é中ÿĀā".encode()))
        rng = random.Random(9)
        probes = {b""}
        for _ in range(400):
            probes.add(bytes(rng.choice(alpha) for _ in range(rng.randrange(1, 7))))
        grammars_extra_ok = [s for s in probes]
        # also sample strings that are accepted: random walk through oracle
        for s in sorted(grammars_extra_ok):
            lang["accepts"].append([ename, s.hex(), oracle_accepts(p, s)])
    lang["extra_grammars"] = extra
    lang["grammars"] = grammars
    err_cases = [
        "", "root ::= a", "root ::= \"a\"\nroot ::= \"b\"", "root ::= root", "root ::= \"a",
        "root ::= [a", "root ::= [z-a]", "root ::= \"\\q\"", "root ::= \"a\"{3,2}", "root ::= \"a\"{,2}",
        "root ::= [^é]", "root ::= \"\\x4\"", "root ::= )", "root ::= [^\\x00-\\xFF]",
        "root ::= \"a\" | [^\\x00-\\xFF]", "root = \"a\"", "::= \"a\"", "root ::= \"a\" $",
        "a ::= b\nb ::= a", "root ::= \"x\" ( \"a\"", "root ::= [\\uD800-\\uDFFF]",
    ]
    for text in err_cases:
        try:
            build_pda(parse_grammar(text))
            lang["errors"].append([text, None, None])
        except GrammarError as exc:
            lang["errors"].append([text, "GrammarError", str(exc)])
    left = 'root ::= root "a" | "b"'
    try:
        from grammask.synthvocab import synth_vocab as sv  # noqa: F401
        compile_bundle(left, toy)
        lang["left_recursion"] = None
    except StateLimitError as exc:
        lang["left_recursion"] = ["StateLimitError", str(exc)]
    schema_cases = {
        "sample": SAMPLE_SCHEMA,
        "bool": '{"type": "boolean"}',
        "enum": '{"enum": ["a", 1, true, null, 2.5]}',
        "opt": '{"type":"object","properties":{"a":{"type":"integer"},"b":{"type":"string"}},"additionalProperties":false}',
        "arr": '{"type":"array","items":{"type":"number"},"minItems":2,"maxItems":4}',
        "arr0": '{"type":"array","items":{"type":"null"},"maxItems":0}',
        "nested": '{"type":"object","properties":{"x":{"type":"array","items":{"type":"object","properties":{"k":{"const":"v"}},"required":["k"],"additionalProperties":false}}},"required":["x"],"additionalProperties":false}',
    }
    schema_bad = ['{"type": "object"}', '{"type": ["a"]}', '{"pattern": "x"}', '{"enum": []}', '{"type":"array"}',
                  'not json', '{"type":"array","items":{"type":"null"},"minItems":3,"maxItems":2}']
    lang["schemas"] = {}
    for sname, sch in schema_cases.items():
        for ws in (True, False):
            text = schema_to_grammar_text(sch, whitespace=ws)
            p = build_pda(parse_grammar(text))
            docs = []
            rngs = random.Random(3)
            base = [b'{"name": "get_weather", "count": 3}', b'{"name":"get_time","count":-10,"tags":["x"]}',
                    b'true', b'false', b' null', b'"a"', b'1', b'2.5', b'{}', b'{"a":1}', b'{"b":"q"}',
                    b'{"a":1,"b":"q"}', b'[1,2]', b'[1,2,3,4]', b'[1,2,3,4,5]', b'[]', b'[ ]', b'[null]',
                    b'{"x":[]}', b'{"x":[{"k":"v"}]}', b'{"x": [ {"k": "v"} , {"k":"v"} ] }', b'[1]']
            for d in base:
                docs.append([d.hex(), oracle_accepts(p, d)])
            for _ in range(40):
                d = bytearray(rngs.choice(base))
                if d:
                    i = rngs.randrange(len(d))
                    d[i:i + 1] = bytes([rngs.choice(b' ,{}[]":0123aeflnrstux')])
                docs.append([bytes(d).hex(), oracle_accepts(p, bytes(d))])
            lang["schemas"][f"{sname}:{int(ws)}"] = {"schema": sch, "docs": docs}
    lang["schema_errors"] = []
    for sch in schema_bad:
        try:
            schema_to_grammar_text(sch)
            lang["schema_errors"].append([sch, None])
        except SchemaError as exc:
            lang["schema_errors"].append([sch, str(exc)])
    (OUT / "languages.json").write_text(json.dumps(lang, indent=0) + "\n")
    print("done", f"{time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()

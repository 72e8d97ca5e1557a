"""Host front end vs the reference (CPU): language, errors, vocabularies,
schema lowering.  Golden verdicts come from the reference itself
(tools/make_golden.py); the device tables are interpreted by tests/tablesim.py."""

import json

import pytest

from automaton_spec import build_tables
from paper_2411_15100_b200.automaton import StateLimitError
from paper_2411_15100_b200.grammar import GrammarError, parse_grammar
from paper_2411_15100_b200.schema import SchemaError, schema_to_grammar_text
from tablesim import TableSim
from workloads import GOLDEN, build_gen_vocab, build_toy200, grammar_text, languages, vocab_by_name


def test_vocab_hashes_match_reference():
    want = json.loads((GOLDEN / "vocab_hashes.json").read_text())
    assert build_toy200().content_hash().hex() == want["toy200"]
    assert build_gen_vocab().content_hash().hex() == want["gen"]
    for key in ("512:text", "4000:mixed", "32000:text"):
        assert vocab_by_name(key).content_hash().hex() == want[key], key


@pytest.mark.slow
def test_synth_vocab_128k_matches_reference():
    want = json.loads((GOLDEN / "vocab_hashes.json").read_text())
    assert vocab_by_name("128256:text").content_hash().hex() == want["128256:text"]


def _sims():
    lang = languages()
    names = sorted({g for g, _, _ in lang["accepts"]})
    return {n: TableSim(build_tables(parse_grammar(grammar_text(n)))) for n in names}


def test_language_equals_reference_oracle():
    sims = _sims()
    bad = []
    for g, hx, want in languages()["accepts"]:
        if sims[g].accepts(bytes.fromhex(hx)) != want:
            bad.append((g, hx, want))
    assert not bad, bad[:10]


@pytest.mark.parametrize("inline", [False, True])
def test_language_independent_of_inlining(inline):
    from paper_2411_15100_b200.automaton import AutomatonOptions

    for g in languages()["grammars"]:
        sim = TableSim(build_tables(parse_grammar(grammar_text(g)), AutomatonOptions(inline=inline)))
        for gg, hx, want in languages()["accepts"]:
            if gg == g:
                assert sim.accepts(bytes.fromhex(hx)) == want, (g, hx)


def test_grammar_errors_match_reference():
    for text, cls, msg in languages()["errors"]:
        if cls is None:
            build_tables(parse_grammar(text))
            continue
        with pytest.raises(GrammarError) as ei:
            build_tables(parse_grammar(text))
        assert str(ei.value) == msg, (text, str(ei.value), msg)


def test_left_recursion_raises_state_limit():
    kind, msg = languages()["left_recursion"]
    assert kind == "StateLimitError"
    with pytest.raises(StateLimitError, match="exceeded cap"):
        build_tables(parse_grammar('root ::= root "a" | "b"'))


def test_schema_language_matches_reference():
    for key, case in languages()["schemas"].items():
        ws = bool(int(key.split(":")[1]))
        sim = TableSim(build_tables(parse_grammar(schema_to_grammar_text(case["schema"], whitespace=ws))))
        for hx, want in case["docs"]:
            assert sim.accepts(bytes.fromhex(hx)) == want, (key, bytes.fromhex(hx))


def test_schema_errors_match_reference():
    for sch, msg in languages()["schema_errors"]:
        if msg is None:
            schema_to_grammar_text(sch)
            continue
        with pytest.raises(SchemaError) as ei:
            schema_to_grammar_text(sch)
        assert str(ei.value).split(":")[0] == msg.split(":")[0], (sch, str(ei.value), msg)


def test_masks_on_small_vocab_match_golden():
    """Full-mask KAT on the toy200/gen fixtures via the table interpreter."""
    from workloads import load_fixture, mask_fixtures

    for fname in mask_fixtures():
        fx = load_fixture(fname)
        if fx["vocab"] not in ("toy200", "gen"):
            continue
        vocab = vocab_by_name(fx["vocab"])
        sim = TableSim(build_tables(parse_grammar(grammar_text(fx["grammar"]))))
        for traj in fx["trajectories"][:6]:
            st = sim.start()
            for step, rec in enumerate(traj["masks"]):
                ids = sim.mask_ids(st, vocab.tokens, vocab.special_tokens, vocab.eos_id)
                words = bytearray(4 * ((vocab.size + 31) // 32))
                for t in ids:
                    words[t >> 3] |= 1 << (t & 7)
                assert words.hex() == rec["hex"], (fname, step)
                if step >= len(traj["tokens"]) or traj["tokens"][step] == vocab.eos_id:
                    break
                st = sim.walk(st, vocab.tokens[traj["tokens"][step]])


def _schema_variants(n):
    import random

    words = ["name", "unit", "count", "tags", "city", "time", "zone", "level", "mode", "query", "id", "score"]
    lits = ["get_weather", "get_time", "search", "celsius", "on", "off", "red", "blue"]
    out = []
    for k in range(n):
        rng = random.Random(500 + k)
        names = rng.sample(words, rng.randint(2, 5))
        props = {}
        for nm in names:
            kind = rng.choice(["enum", "string", "integer", "array", "number", "boolean"])
            if kind == "enum":
                props[nm] = {"enum": rng.sample(lits, rng.randint(2, 3))}
            elif kind == "array":
                lo = rng.randint(0, 2)
                props[nm] = {"type": "array", "items": {"type": "string"}, "minItems": lo, "maxItems": lo + 2}
            else:
                props[nm] = {"type": kind}
        out.append({"type": "object", "properties": props, "required": names[:1], "additionalProperties": False})
    return out


def test_native_front_end_tables_identical():
    """The C++ front end (gm_front_end_build, §8f rank 2) builds exactly the
    tables of the Python specification (tests/automaton_spec.py build_tables), array for
    array, for every reference grammar and 24 schema grammars; host only."""
    import numpy as np

    from paper_2411_15100_b200.automaton import AutomatonOptions, build_tables_native
    from paper_2411_15100_b200.compiler import BUILTIN_JSON_GRAMMAR

    lang = languages()
    texts = {"builtin_json": BUILTIN_JSON_GRAMMAR, **lang["grammars"], **lang["extra_grammars"]}
    for k, sc in enumerate(_schema_variants(24)):
        texts[f"schema{k}"] = schema_to_grammar_text(json.dumps(sc))
    fields = ["n_nodes", "n_rules", "n_classes", "start_node", "root_rule", "rule_names", "byte_class", "trans_off",
              "trans", "push_pool", "node_flags", "node_rule", "cache_keys", "follow_start", "follow_next",
              "n_fstates", "raw_off", "raw", "finals", "rule_start"]
    for opts in (AutomatonOptions(), AutomatonOptions(inline=False), AutomatonOptions(ctx_expansion=False)):
        for name, text in texts.items():
            g = parse_grammar(text)
            a, b = build_tables(g, opts), build_tables_native(g, opts)
            for f in fields:
                x, y = getattr(a, f), getattr(b, f)
                if isinstance(x, np.ndarray):
                    assert np.array_equal(x, y), (name, f)
                else:
                    assert x == y, (name, f)


def test_native_front_end_errors():
    from paper_2411_15100_b200.automaton import build_tables_native

    with pytest.raises(StateLimitError):
        build_tables_native(parse_grammar('root ::= root "a" | "b"'))


def test_dfa_limit_falls_back_to_nfa():
    """A rule whose subset construction would exceed max_dfa_states (2^18
    subsets here) keeps an epsilon-free NFA (front_end.cpp eps_free): same
    language, several targets per (node, class)."""
    import random
    import re

    import numpy as np

    from paper_2411_15100_b200.automaton import AutomatonOptions, build_tables_native
    from paper_2411_15100_b200.grammar import parse_grammar

    t = build_tables_native(parse_grammar('root ::= [ab]* "a" [ab]{17} "."'), AutomatonOptions())
    assert np.diff(t.trans_off).max() >= 2 and t.n_nodes < 100
    sim = TableSim(t)
    rx = re.compile(rb"[ab]*a[ab]{17}\.")
    rng = random.Random(3)
    for _ in range(300):
        s = bytes(rng.choice(b"ab") for _ in range(rng.randrange(15, 26))) + (b"." if rng.random() < 0.8 else b"")
        assert sim.accepts(s) == bool(rx.fullmatch(s)), s


def _parse_both(text, root=None):
    """(python result, native result): ('ok', names, root, ir) or
    ('err', message, line, col) for each parser."""
    import numpy as np

    from paper_2411_15100_b200.automaton import encode_ir, parse_grammar_native
    from paper_2411_15100_b200.grammar import GrammarError

    out = []
    for native in (False, True):
        try:
            if native:
                g = parse_grammar_native(text, root)
                out.append(("ok", g.names, g.root, np.asarray(g.ir).tolist()))
            else:
                g = parse_grammar(text, root)
                ir, _ = encode_ir(g)
                out.append(("ok", g.names, g.root, np.asarray(ir).tolist()))
        except GrammarError as e:
            out.append(("err", str(e), e.line, e.col))
    return out


def test_native_parser_equals_python_parser():
    """The C++ parser (csrc/grammar_parse.cpp) gives the Python
    specification's IR, rule names and root for every reference grammar,
    schema lowering and the golden error cases — and the same GrammarError
    message and position on every error, including fuzzed mutations."""
    import json
    import random
    import sys

    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))
    from bench_config5 import mutate_schema

    lang = languages()
    texts = list(lang["grammars"].values()) + list(lang["extra_grammars"].values())
    texts += [schema_to_grammar_text(json.dumps(mutate_schema(i)), whitespace=bool(i % 2)) for i in range(24)]
    texts += [t for t, _, _ in lang["errors"]]
    texts += ['root ::= "\\u00e9" [\\u0100-\\uFFFF] "x"{2,} "y"{,3}', 'a ::= "x"\nroot ::= a a', "root ::= [^\\xff]",
              "root ::= [z-a]", 'root ::= "a" {3}', "r ::= [\\u0041-\\u00ff]", 'root ::= "\\ud800"', "x ::= ( )",
              'root ::= "a" | | "b"', "root ::= [a-]", "root ::= []a]", "root ::= [^]x]", '# c\nroot ::= "a" # t']
    rng = random.Random(11)
    base = list(texts)
    for _ in range(400):  # random single-character mutations of valid grammars
        t = rng.choice(base)
        if not t:
            continue
        i = rng.randrange(len(t))
        t = t[:i] + rng.choice('"[]()|*+?{},:=\\-^#\n xaé') + t[i + 1:]
        texts.append(t)
    for t in texts:
        for root in (None, "root"):
            py, nat = _parse_both(t, root)
            assert py == nat, (t, root, py[:2], nat[:2])

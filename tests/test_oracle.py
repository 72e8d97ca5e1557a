"""Pin the CPU oracle (oracle/) against the real reference's golden vectors,
and against its own language-level brute force (REF tests/conftest.py:149-159)."""

import hashlib
import random

import pytest

from oracle import brute_force_mask, compile_oracle_bundle
from oracle.matcher import OracleMatcher
from oracle.pda import build_raw_pda, stacks_accept, step_stacks
from paper_2411_15100_b200.grammar import parse_grammar
from workloads import grammar_text, languages, load_fixture, mask_fixtures, vocab_by_name


def test_oracle_language_equals_reference():
    lang = languages()
    pdas = {}
    for g, hx, want in lang["accepts"]:
        if g not in pdas:
            pdas[g] = build_raw_pda(parse_grammar(grammar_text(g)))
        p = pdas[g]
        got = stacks_accept(p, step_stacks(p, [(p.start_node(),)], bytes.fromhex(hx)))
        assert got == want, (g, hx)


def _replay(fname, limit_traj=None):
    fx = load_fixture(fname)
    vocab = vocab_by_name(fx["vocab"])
    b = compile_oracle_bundle(grammar_text(fx["grammar"]), vocab)
    n = 0
    for traj in fx["trajectories"][:limit_traj]:
        m = OracleMatcher(b, history_window=1)
        for step, rec in enumerate(traj["masks"]):
            raw = m.fill().astype("<u4").tobytes()
            if "hex" in rec:
                assert raw.hex() == rec["hex"], (fname, step)
            assert hashlib.sha256(raw).hexdigest() == rec["sha256"], (fname, step)
            n += 1
            if step >= len(traj["tokens"]):
                break
            assert m.accept_token(traj["tokens"][step])
            if traj["tokens"][step] == vocab.eos_id:
                break
    return n


@pytest.mark.parametrize("fname", [f for f in mask_fixtures() if "toy200" in f or "gen" in f or "4000" in f])
def test_oracle_matches_golden_small(fname):
    assert _replay(fname) > 0


@pytest.mark.slow
@pytest.mark.parametrize("fname", [f for f in mask_fixtures() if "32000" in f])
def test_oracle_matches_golden_32k(fname):
    assert _replay(fname, limit_traj=2) > 0


def test_oracle_cached_equals_brute_force():
    vocab = vocab_by_name("toy200")
    rng = random.Random(7)
    for g in ("array_string", "json", "arithmetic", "xml", "schema"):
        b = compile_oracle_bundle(grammar_text(g), vocab)
        for _ in range(4):
            m = OracleMatcher(b)
            consumed = b""
            for _ in range(rng.randrange(1, 8)):
                words = m.fill()
                ids = [t for t in range(vocab.size) if (int(words[t >> 5]) >> (t & 31)) & 1]
                assert ids == sorted(brute_force_mask(b.pda, vocab, consumed)), (g, consumed)
                pick = ids[rng.randrange(len(ids))]
                if pick == vocab.eos_id:
                    break
                assert m.accept_token(pick)
                consumed += vocab.tokens[pick]

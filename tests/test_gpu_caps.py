"""Wide stack sets and per-request errors, pinned to the REAL reference
(tests/golden/caps.json.gz, written by tools/make_golden_caps.py from
grammask).

* ``ambig40`` / ``ambig300`` keep 40 / 300 stacks alive (more than every
  local walker holds): the overflow walker (global-memory lanes, up to the
  reference's 4096 cap, REF matcher.py:116, 188-189), wide ring entries and
  the batched wide fill must reproduce the reference's masks bit for bit,
  through the grammask API (K2 + K4), the batched XGrammar API and the fused
  K5 step.
* ``dfa_blowup`` (``[ab]* "a" [ab]{17} "."``): over the front end's 200k
  DFA-state limit, so the rule stays an epsilon-free NFA (front_end.cpp
  eps_free) with up to 18 live stacks — same masks as the reference.
* ``ambig_over_cap`` (4200 alternatives): the reference's compile raises
  StateLimitError (REF cache.py:58, 137-138); so does ours.
* errors are attributed to the request that caused them (per-slot error
  words, K4/K5 flag bit 1), never to a neighbour.
"""

import gzip
import json
from functools import lru_cache

import numpy as np
import pytest

from workloads import GOLDEN

pytestmark = pytest.mark.gpu


@lru_cache(maxsize=None)
def caps():
    with gzip.open(GOLDEN / "caps.json.gz", "rt", encoding="utf-8") as fh:
        return json.load(fh)


@lru_cache(maxsize=None)
def caps_vocab():
    from paper_2411_15100_b200.vocab import vocab_from_tokens

    toks = [bytes.fromhex(h) for h in caps()["vocab_tokens"]]
    return vocab_from_tokens(toks, eos_id=len(toks) - 1, special=[len(toks) - 1])


CASES = ["ambig40", "ambig300", "deep_ambig", "dfa_blowup"]


@pytest.mark.parametrize("case", CASES)
def test_wide_sets_grammask_api(case):
    """K2 fill + K4 accept, one request at a time (REF matcher.py:273, 377)."""
    from paper_2411_15100_b200.compat import Matcher, compile_bundle

    doc = caps()["cases"][case]
    vocab = caps_vocab()
    bundle = compile_bundle(doc["grammar"], vocab)
    checked = 0
    for traj in doc["trajectories"]:
        m = Matcher(bundle, vocab, history_window=4)
        toks = traj["tokens"]
        for step, rec in enumerate(traj["masks"]):
            assert m.next_token_mask().to_bytes().hex() == rec["hex"], (case, step)
            checked += 1
            if step >= len(toks) or toks[step] == vocab.eos_id:
                break
            assert m.accept_token(toks[step]), (case, step)
        m.close()
    assert checked > 10


@pytest.mark.parametrize("case", CASES)
def test_wide_sets_batched_and_fused(case):
    """The same trajectories in one batch: batched K2 + K4, then the fused K5
    step (accept + fill + apply) — masks equal the reference's, logits exact."""
    import torch

    import paper_2411_15100_b200 as gm

    doc = caps()["cases"][case]
    vocab = caps_vocab()
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    compiled = gm.GrammarCompiler(info, cache_enabled=False).compile_grammar(doc["grammar"])
    trajs = doc["trajectories"]
    B = len(trajs)
    steps = min(len(t["masks"]) for t in trajs)
    W = (vocab.size + 31) // 32

    def want(s):
        return np.stack([np.frombuffer(bytes.fromhex(t["masks"][s]["hex"]), dtype=np.int32) for t in trajs])

    batch = gm.BatchGrammarMatcher()
    ms = [gm.GrammarMatcher(compiled) for _ in range(B)]
    bm = gm.allocate_token_bitmask(B, vocab.size)
    for s in range(steps):
        batch.batch_fill_next_token_bitmask(ms, bm)
        assert np.array_equal(bm.cpu().numpy(), want(s)), (case, "batched", s)
        if any(s >= len(t["tokens"]) for t in trajs):
            break
        assert all(batch.batch_accept_token(ms, [t["tokens"][s] for t in trajs]))

    ms = [gm.GrammarMatcher(compiled) for _ in range(B)]
    vp = (vocab.size + 7) // 8 * 8  # 16-byte aligned rows for the fused apply
    logits = torch.randn(B, vp, device="cuda").to(torch.bfloat16)[:, : vocab.size]
    for s in range(steps):
        keep = logits.clone()
        if s == 0:
            batch.batch_step(ms, None, bitmask=bm, logits=logits)
        else:
            flags = batch.batch_step(ms, [t["tokens"][s - 1] for t in trajs], bitmask=bm, logits=logits)
            assert (flags.cpu().numpy() == 1).all(), (case, "fused accept", s)
        w = want(s)
        assert np.array_equal(bm.cpu().numpy(), w), (case, "fused", s)
        allowed = torch.from_numpy(np.unpackbits(w.view(np.uint8), axis=1, bitorder="little")[:, : vocab.size]
                                   .astype(bool)).cuda()
        expect = torch.where(allowed, keep, torch.full_like(keep, float("-inf")))
        assert torch.equal(logits.view(torch.int16), expect.view(torch.int16)), (case, "apply", s)
        if any(s >= len(t["tokens"]) for t in trajs):
            break
    assert W > 0


def test_over_cap_raises_like_reference():
    """4200 live alternatives: more than the 4096 cap -> StateLimitError at
    compile, as the reference (its message: 'branch set exceeded cap of 4096')."""
    from paper_2411_15100_b200.automaton import StateLimitError
    from paper_2411_15100_b200.compat import compile_bundle

    doc = caps()["cases"]["ambig_over_cap"]
    assert doc["compile_error"][0] == "StateLimitError"
    n = doc["grammar_alternatives"]
    alts = " | ".join(f"a{i}" for i in range(1, n + 1))
    rules = "\n".join(f'a{i} ::= "x" a{i} "y" | "z{i}"' for i in range(1, n + 1))
    with pytest.raises(StateLimitError, match="cap of 4096"):
        compile_bundle(f"root ::= {alts}\n{rules}\n", caps_vocab())


def test_errors_are_per_request():
    """A terminated request's error lands on that request only: batched fill
    raises its MatcherError (request index attached), K5 flags it with bit 1,
    DecodeLoop.flags raises for it, and a healthy neighbour's own calls stay
    clean (REF matcher.py:379-381)."""
    import torch

    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200.engine import MatcherError
    from paper_2411_15100_b200.graph import DecodeLoop

    vocab = caps_vocab()
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    compiled = gm.GrammarCompiler(info, cache_enabled=False).compile_grammar('root ::= "x" | "xy"')
    tid = {bytes.fromhex(h): i for i, h in enumerate(caps()["vocab_tokens"])}
    ms = [gm.GrammarMatcher(compiled) for _ in range(3)]
    assert ms[1].accept_token(tid[b"x"]) and ms[1].accept_token(vocab.eos_id)  # request 1 terminated
    batch = gm.BatchGrammarMatcher()
    bm = gm.allocate_token_bitmask(3, vocab.size)
    with pytest.raises(MatcherError, match="terminated") as ei:
        batch.batch_fill_next_token_bitmask(ms, bm)
    assert getattr(ei.value, "request_index", None) == 1
    # the neighbours are clean: their own checks raise nothing
    need = ms[0].fill_next_token_bitmask(bm, 0)
    assert need
    # K5: accepting on the terminated request flags it (bit 1), not the others
    flags = batch.batch_step(ms, [tid[b"x"], tid[b"x"], tid[b"x"]], bitmask=bm).cpu().numpy()
    assert flags[0] == 1 and flags[2] == 1 and flags[1] & 2, flags
    with pytest.raises(MatcherError) as ei:
        batch.check_errors(ms, flags)
    assert getattr(ei.value, "request_index", None) == 1
    # native decode loop: the flags of the failed request raise, for it alone
    ms2 = [gm.GrammarMatcher(compiled) for _ in range(2)]
    assert ms2[0].accept_token(tid[b"x"]) and ms2[0].accept_token(vocab.eos_id)
    logits = [torch.zeros(2, (vocab.size + 7) // 8 * 8, device="cuda", dtype=torch.bfloat16)]
    loop = DecodeLoop(ms2, [gm.allocate_token_bitmask(2, vocab.size)], logits, recycle=False)
    loop.step(np.asarray([tid[b"x"], tid[b"x"]], np.int32), 0)
    with pytest.raises(MatcherError) as ei:
        loop.flags(0)
    assert getattr(ei.value, "request_index", None) == 0
    assert loop.flags(0, raise_errors=False)[1] == 1
    loop.close()

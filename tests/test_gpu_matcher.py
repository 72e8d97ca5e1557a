"""Matcher behaviour KATs on the GPU through the grammask-compatible API.

Each test restates a reference test (REF tests/test_matcher.py, cited per
test) and checks the device engine against the reference's expected values,
the CPU oracle, or the oracle's language-level brute force."""

import random

import numpy as np
import pytest

from oracle import brute_force_mask, compile_oracle_bundle
from oracle.matcher import OracleMatcher
from paper_2411_15100_b200.vocab import vocab_from_tokens
from workloads import grammar_text, vocab_by_name

pytestmark = pytest.mark.gpu

ARRAY_STRING = None


def make_vocab(tokens, specials=("<eos>",)):
    toks = [bytes(t) if not isinstance(t, str) else t.encode() for t in tokens]
    toks += [s.encode() for s in specials]
    n = len(toks)
    return vocab_from_tokens(toks, eos_id=n - 1, special=list(range(n - len(specials), n)))


@pytest.fixture(scope="module")
def fig2():
    from paper_2411_15100_b200.compat import compile_bundle

    vocab = make_vocab([bytes([b]) for b in b'[]",abx\\'] + [b"ab", b'"]', b'",', b'a"', b'""', b"]]", b"],", b'["'])
    text = grammar_text("array_string")
    return compile_bundle(text, vocab), vocab, text


def test_mask_wire_format():  # REF test_matcher.py:31-44
    from paper_2411_15100_b200.compat import TokenMask

    m = TokenMask(70)
    for t in (0, 33, 69):
        m.set_bit(t)
    raw = m.to_bytes()
    assert len(raw) == 12 and raw[0] == 0x01 and raw[4] == 0x02
    assert TokenMask.from_bytes(70, raw) == m
    assert list(m.allowed_ids()) == [0, 33, 69] and m.count() == 3


def test_vocab_hash_mismatch(fig2):  # REF test_matcher.py:58-62
    from paper_2411_15100_b200.compat import Matcher, MatcherError

    bundle, _, _ = fig2
    with pytest.raises(MatcherError, match="does not match"):
        Matcher(bundle, make_vocab([b"a", b"b"]))


def test_mask_equals_brute_force_and_accept_consistency(fig2):  # REF test_matcher.py:65-88
    from paper_2411_15100_b200.compat import Matcher

    bundle, vocab, text = fig2
    ob = compile_oracle_bundle(text, vocab)
    rng = random.Random(11)
    for _ in range(12):
        m = Matcher(bundle, vocab, history_window=64)
        consumed = b""
        for _ in range(rng.randrange(0, 8)):
            mask = m.next_token_mask()
            assert list(mask.allowed_ids()) == sorted(brute_force_mask(ob.pda, vocab, consumed))
            for tid in range(vocab.size):
                probe = m.branch()
                try:
                    assert probe.accept_token(tid) == mask.is_allowed(tid), (consumed, tid)
                finally:
                    probe.close()
            ids = mask.allowed_ids()
            pick = int(ids[rng.randrange(len(ids))])
            if pick == vocab.eos_id:
                break
            assert m.accept_token(pick)
            consumed += vocab.tokens[pick]
        m.close()


def test_rejection_keeps_state(fig2):  # REF test_matcher.py:103-110
    from paper_2411_15100_b200.compat import Matcher

    bundle, vocab, _ = fig2
    m = Matcher(bundle, vocab, history_window=16)
    before = m.next_token_mask()
    assert not m.accept_bytes(b"[x")
    assert m.next_token_mask() == before
    assert m.accept_bytes(b"")
    assert m.history_depth == 1
    assert m.next_token_mask() == before


def test_empty_and_special_tokens_rejected():  # REF test_matcher.py:113-123
    from paper_2411_15100_b200.compat import Matcher, compile_bundle

    vocab = vocab_from_tokens([b"a", b"", b"<pad>", b"<eos>"], eos_id=3, special=[2, 3])
    m = Matcher(compile_bundle('root ::= "a" | ""', vocab), vocab)
    mask = m.next_token_mask()
    assert mask.is_allowed(0) and not mask.is_allowed(1) and not mask.is_allowed(2) and mask.is_allowed(3)
    assert not m.accept_token(1)
    assert not m.accept_token(2)


def test_eos_semantics(fig2):  # REF test_matcher.py:126-139
    from paper_2411_15100_b200.compat import Matcher, MatcherError

    bundle, vocab, _ = fig2
    m = Matcher(bundle, vocab)
    assert not m.can_terminate()
    assert not m.accept_token(vocab.eos_id)
    assert m.accept_bytes(b"[]")
    assert m.can_terminate()
    assert m.accept_token(vocab.eos_id)
    assert m.terminated
    with pytest.raises(MatcherError, match="terminated"):
        m.next_token_mask()
    m.rollback(1)
    assert not m.terminated
    assert m.can_terminate()


def test_forced_grammar_eos_only():  # REF test_matcher.py:142-148
    from paper_2411_15100_b200.compat import Matcher, compile_bundle

    vocab = make_vocab([b"a", b"b"])
    m = Matcher(compile_bundle('root ::= "a"', vocab), vocab)
    assert m.accept_token(0)
    assert list(m.next_token_mask().allowed_ids()) == [vocab.eos_id]


def test_rollback_round_trip_and_bounds(fig2):  # REF test_matcher.py:154-181
    from paper_2411_15100_b200.compat import Matcher, MatcherError

    bundle, vocab, _ = fig2
    m = Matcher(bundle, vocab, history_window=8)
    fresh = m.next_token_mask()
    assert m.accept_bytes(b"[")
    assert m.accept_bytes(b'"a')
    m.rollback(2)
    assert m.next_token_mask() == fresh
    assert m.accept_bytes(b"[") and m.accept_bytes(b'"a')
    snap = m.next_token_mask()
    m.rollback(1)
    assert m.accept_bytes(b'"a')
    assert m.next_token_mask() == snap
    w = Matcher(bundle, vocab, history_window=4)
    for _ in range(6):
        assert w.accept_bytes(b"[")
    assert w.history_depth == 4
    with pytest.raises(MatcherError, match="roll back"):
        w.rollback(5)
    w.rollback(4)


def test_rollback_determinism_random(fig2):  # REF test_matcher.py:184-205
    from paper_2411_15100_b200.compat import Matcher

    bundle, vocab, _ = fig2
    rng = random.Random(3)
    for _ in range(10):
        m = Matcher(bundle, vocab, history_window=32)
        accepted = []
        for _ in range(rng.randrange(1, 10)):
            ids = m.next_token_mask().allowed_ids()
            pick = int(ids[rng.randrange(len(ids))])
            if pick == vocab.eos_id:
                break
            m.accept_token(pick)
            accepted.append(pick)
        if not accepted:
            continue
        k = rng.randrange(1, len(accepted) + 1)
        before = m.next_token_mask()
        m.rollback(k)
        for tid in accepted[-k:]:
            assert m.accept_token(tid)
        assert m.next_token_mask() == before


def test_branch_divergence(fig2):  # REF test_matcher.py:211-226
    from paper_2411_15100_b200.compat import Matcher

    bundle, vocab, _ = fig2
    a = Matcher(bundle, vocab)
    a.accept_bytes(b"[")
    b = a.branch()
    assert a.next_token_mask() == b.next_token_mask()
    a.accept_bytes(b'"x"')
    b.accept_bytes(b"]")
    ra = Matcher(bundle, vocab)
    ra.accept_bytes(b'["x"')
    rb = Matcher(bundle, vocab)
    rb.accept_bytes(b"[]")
    assert a.next_token_mask() == ra.next_token_mask()
    assert b.can_terminate() == rb.can_terminate()


def test_closed_matcher_raises(fig2):  # REF test_matcher.py:240-246
    from paper_2411_15100_b200.compat import Matcher, MatcherError

    bundle, vocab, _ = fig2
    m = Matcher(bundle, vocab)
    m.close()
    with pytest.raises(MatcherError, match="closed"):
        m.next_token_mask()
    with pytest.raises(MatcherError, match="closed"):
        m.branch()


@pytest.mark.parametrize("grammar,toks,prefix,want,cap", [
    ('root ::= "true"', [b"t", b"r", b"u", b"e"], b"", b"true", 4096),          # REF :306-313
    ('root ::= "\\"k\\":" [0-9]', [b"k", b'"', b":", b"1"], b'"k', b'":', 4096),  # REF :321-326
    ('root ::= "ab" | "a"', [b"a", b"b"], b"", b"a", 4096),                       # REF :329-333
    ('root ::= "aaaaaaaaaa"', [b"a"], b"", b"aaaa", 4),                           # REF :336-339
])
def test_jump_forward(grammar, toks, prefix, want, cap):
    from paper_2411_15100_b200.compat import Matcher, compile_bundle

    vocab = make_vocab(toks)
    m = Matcher(compile_bundle(grammar, vocab), vocab)
    if prefix:
        assert m.accept_bytes(prefix)
    assert m.find_jump_forward_bytes(max_len=cap) == want
    assert m.find_jump_forward_bytes(max_len=cap) == want  # state unchanged


def test_jump_forward_stops_at_choice(fig2):  # REF test_matcher.py:316-318
    from paper_2411_15100_b200.compat import Matcher

    bundle, vocab, _ = fig2
    assert Matcher(bundle, vocab).find_jump_forward_bytes() == b""


def test_uncached_fill_matches_cached(fig2):  # REF test_matcher.py:345-363
    from paper_2411_15100_b200.compat import CompileOptions, Matcher, compile_bundle

    bundle, vocab, text = fig2
    plain = compile_bundle(text, vocab, CompileOptions(inline=False, merge=False, cache=False))
    rng = random.Random(23)
    a, b = Matcher(bundle, vocab), Matcher(plain, vocab)
    for _ in range(12):
        ma, mb = a.next_token_mask(), b.next_token_mask()
        assert ma == mb
        ids = ma.allowed_ids()
        pick = int(ids[rng.randrange(len(ids))])
        if pick == vocab.eos_id:
            break
        assert a.accept_token(pick) and b.accept_token(pick)


@pytest.mark.parametrize("name", ["array_string", "json", "arithmetic", "xml", "schema"])
def test_lockstep_vs_oracle_random_walks(name):
    """Device masks == oracle masks along random walks (toy200, REF
    tests/test_acceptance.py:54-88 style), including EOS and state resets."""
    from paper_2411_15100_b200.compat import Matcher, compile_bundle

    vocab = vocab_by_name("toy200")
    text = grammar_text(name)
    bundle = compile_bundle(text, vocab)
    ob = compile_oracle_bundle(text, vocab)
    rng = random.Random(2024)
    for _ in range(20):
        m, r = Matcher(bundle, vocab, history_window=1), OracleMatcher(ob, history_window=1)
        for _ in range(rng.randrange(1, 16)):
            got = m.next_token_mask().words
            assert np.array_equal(got, r.fill()), name
            ids = [t for t in range(vocab.size) if (int(got[t >> 5]) >> (t & 31)) & 1]
            pick = ids[rng.randrange(len(ids))]
            assert m.accept_token(pick) and r.accept_token(pick)
            if pick == vocab.eos_id:
                break
        m.close()


def test_guided_generation_is_in_language():  # REF test_matcher.py:376-386
    from oracle.pda import stacks_accept, step_stacks
    from paper_2411_15100_b200.compat import Matcher, compile_bundle

    vocab = vocab_by_name("gen")
    rng = random.Random(4)
    for name in ("array_string", "json", "arithmetic", "xml", "schema"):
        text = grammar_text(name)
        bundle = compile_bundle(text, vocab)
        ob = compile_oracle_bundle(text, vocab)
        for _ in range(3):
            m = Matcher(bundle, vocab)
            out = b""
            for _ in range(4096):
                ids = m.next_token_mask().allowed_ids()
                pick = int(ids[rng.randrange(len(ids))])
                assert m.accept_token(pick)
                if pick == vocab.eos_id:
                    break
                out += vocab.tokens[pick]
            assert stacks_accept(ob.pda, step_stacks(ob.pda, [(ob.pda.start_node(),)], out)), (name, out)
            m.close()


@pytest.mark.parametrize("grammar,dtype,B", [("json", "float32", 6), ("json", "bfloat16", 6), ("json", "bfloat16", 100),
                                             ("sql", "bfloat16", 6), ("sql", "float32", 6)])
def test_fused_fill_apply_equals_separate(grammar, dtype, B):
    """K3 (one kernel) == K2 fill then K0 apply == torch.where(bit, x, -inf),
    bit for bit, along a trajectory (B = 6: several CTAs per request, each
    with its word range; B = 100: one CTA per request; the SQL grammar's
    identifier-class masks take K0's load-blend-store path for dense mixed
    chunks, and the fused apply blends the rows of the keys its per-key
    policy flagged at build)."""
    import torch

    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200.engine import get_pool
    from paper_2411_15100_b200.matcher import batch_fill, batch_fill_apply

    vocab = vocab_by_name("4000:mixed")
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    gc = gm.GrammarCompiler(info)
    compiled = gc.compile_builtin_json_grammar() if grammar == "json" else gc.compile_grammar(grammar_text(grammar))
    ms = [gm.GrammarMatcher(compiled) for _ in range(B)]
    pool = get_pool()
    slots = torch.tensor([m.slot for m in ms], dtype=torch.int32, device="cuda")
    dt = getattr(torch, dtype)
    bits = torch.arange(32, device="cuda", dtype=torch.int32)
    g = torch.Generator(device="cuda").manual_seed(3)
    W = (vocab.size + 31) // 32
    for step in range(12):
        logits = torch.randn(B, vocab.size, device="cuda", generator=g).to(dt)
        a, b = logits.clone(), logits.clone()
        bm1 = torch.empty((B, W), dtype=torch.int32, device="cuda")
        bm2 = torch.empty((B, W), dtype=torch.int32, device="cuda")
        batch_fill(pool, slots, bm1)
        gm.apply_token_bitmask_inplace(a, bm1)
        batch_fill_apply(pool, slots, b, bm2)
        assert torch.equal(bm1, bm2)
        allowed = ((bm1.unsqueeze(-1) >> bits) & 1).reshape(B, -1)[:, :vocab.size].bool()
        want = torch.where(allowed, logits, torch.full_like(logits, float("-inf")))
        iv = torch.int16 if dt != torch.float32 else torch.int32
        assert torch.equal(a.view(iv), want.view(iv))
        assert torch.equal(a.view(torch.int16 if dt != torch.float32 else torch.int32),
                           b.view(torch.int16 if dt != torch.float32 else torch.int32))
        c = logits.clone()
        batch_fill_apply(pool, slots, c)  # no bitmask output
        assert torch.equal(a.view(torch.int8), c.view(torch.int8))
        b[:, vocab.eos_id] = float("-inf")
        if not bool(torch.isfinite(b.float()).any(-1).all()):  # a request can only end (EOS): trajectory done
            break
        toks = b.float().argmax(-1).tolist()
        assert all(gm.BatchGrammarMatcher.batch_accept_token(ms, toks))


@pytest.mark.parametrize("name", ["json", "xml", "arithmetic", "sql"])
@pytest.mark.parametrize("with_logits", [False, True])
def test_step_kernel_equals_accept_then_fill(name, with_logits):
    """K5 (accept + recycle + fill [+ apply] in one launch) == K4 accept,
    recycle, then K2 fill (+ K0 apply), bit for bit, including rejected
    tokens (state unchanged) and requests that finish and restart."""
    import torch

    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200.engine import get_pool
    from paper_2411_15100_b200.matcher import batch_accept, batch_fill, batch_recycle, batch_step

    vocab = vocab_by_name("4000:mixed")
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    text = gm.BUILTIN_JSON_GRAMMAR if name == "json" else grammar_text(name)
    compiled = gm.GrammarCompiler(info).compile_grammar(text)
    B, W = 8, (vocab.size + 31) // 32
    pool = get_pool()
    ref = [gm.GrammarMatcher(compiled) for _ in range(B)]
    new = [gm.GrammarMatcher(compiled) for _ in range(B)]
    s_ref = torch.tensor([m.slot for m in ref], dtype=torch.int32, device="cuda")
    s_new = torch.tensor([m.slot for m in new], dtype=torch.int32, device="cuda")
    bm_ref = torch.empty((B, W), dtype=torch.int32, device="cuda")
    bm_new = torch.empty((B, W), dtype=torch.int32, device="cuda")
    acc_ref = torch.empty(B, dtype=torch.uint8, device="cuda")
    acc_new = torch.empty(B, dtype=torch.uint8, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(5)
    rng = random.Random(11)
    toks = None
    for step in range(40):
        logits = torch.randn(B, vocab.size, device="cuda", generator=g).to(torch.bfloat16)
        la, lb = logits.clone(), logits.clone()
        if toks is not None:
            batch_accept(pool, s_ref, toks, acc_ref)
            batch_recycle(pool, s_ref)
        batch_fill(pool, s_ref, bm_ref)
        gm.apply_token_bitmask_inplace(la, bm_ref)
        if with_logits:
            batch_step(pool, s_new, toks, acc_new if toks is not None else None, bm_new, lb, recycle=True)
        else:
            batch_step(pool, s_new, toks, acc_new if toks is not None else None, bm_new, recycle=True)
        assert torch.equal(bm_ref, bm_new), step
        if toks is not None:
            assert torch.equal(acc_ref, acc_new), step
        if with_logits:
            assert torch.equal(la.view(torch.int16), lb.view(torch.int16)), step
        # next tokens: mostly allowed ones (EOS preferred when allowed, so
        # requests finish and restart), sometimes an arbitrary (likely rejected) id
        allowed = ((bm_ref.unsqueeze(-1) >> torch.arange(32, device="cuda", dtype=torch.int32)) & 1).reshape(B, -1)
        pick = []
        for r in range(B):
            ids = allowed[r, :vocab.size].nonzero().flatten().tolist()
            if rng.random() < 0.1 or not ids:
                pick.append(rng.randrange(vocab.size - 1))
            elif vocab.eos_id in ids and rng.random() < 0.5:
                pick.append(vocab.eos_id)
            else:
                pick.append(rng.choice(ids))
        toks = torch.tensor(pick, dtype=torch.int32, device="cuda")
    pool.check()


@pytest.mark.parametrize("zero_copy", [True, False])
def test_decode_step_graph_equals_eager(zero_copy):
    """DecodeStepGraph (host ids -> K5 -> host flags, captured; zero-copy or
    with copy-engine H2D/D2H) == eager batch_step."""
    import torch

    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200.engine import get_pool
    from paper_2411_15100_b200.graph import DecodeStepGraph
    from paper_2411_15100_b200.matcher import batch_step

    vocab = vocab_by_name("4000:mixed")
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    compiled = gm.GrammarCompiler(info).compile_builtin_json_grammar()
    B, W = 6, (vocab.size + 31) // 32
    pool = get_pool()
    ref = [gm.GrammarMatcher(compiled) for _ in range(B)]
    new = [gm.GrammarMatcher(compiled) for _ in range(B)]
    s_ref = torch.tensor([m.slot for m in ref], dtype=torch.int32, device="cuda")
    bm_ref = torch.empty((B, W), dtype=torch.int32, device="cuda")
    bm_new = torch.empty((B, W), dtype=torch.int32, device="cuda")
    acc_ref = torch.empty(B, dtype=torch.uint8, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(9)
    bufs = [torch.empty(B, vocab.size, device="cuda", dtype=torch.bfloat16) for _ in range(2)]
    step = DecodeStepGraph(new, bm_new, bufs, recycle=True, zero_copy=zero_copy)
    rng = random.Random(4)
    toks = None
    for it in range(30):
        base = torch.randn(B, vocab.size, device="cuda", generator=g).to(torch.bfloat16)
        la = base.clone()
        i = it % 2
        bufs[i].copy_(base)
        torch.cuda.synchronize()
        if toks is None:
            batch_step(pool, s_ref, None, None, bm_ref, la, recycle=True)
            step.first(i)
        else:
            batch_step(pool, s_ref, torch.tensor(toks, dtype=torch.int32, device="cuda"), acc_ref, bm_ref, la,
                       recycle=True)
            acc = step.run(toks, i)
            assert acc.tolist() == acc_ref.tolist(), (it, toks, acc.tolist(), acc_ref.tolist(), step.tokens[i].tolist())
        torch.cuda.synchronize()
        step.stream.synchronize()
        assert torch.equal(bm_ref, bm_new), it
        assert torch.equal(la.view(torch.int16), bufs[i].view(torch.int16)), it
        allowed = ((bm_ref.unsqueeze(-1) >> torch.arange(32, device="cuda", dtype=torch.int32)) & 1).reshape(B, -1)
        toks = []
        for r in range(B):
            ids = allowed[r, :vocab.size].nonzero().flatten().tolist()
            toks.append(vocab.eos_id if (vocab.eos_id in ids and rng.random() < 0.5) else rng.choice(ids))
    pool.check()


def test_decode_step_graph_queued_back_to_back():
    """Steps queued without host syncs (wait=False, 3 buffers reused over 14
    steps) give the same accepted flags and masks as eager batch_step."""
    import torch

    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200.engine import get_pool
    from paper_2411_15100_b200.graph import DecodeStepGraph
    from paper_2411_15100_b200.matcher import batch_step

    vocab = vocab_by_name("4000:mixed")
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    compiled = gm.GrammarCompiler(info).compile_builtin_json_grammar()
    B, W, n_buf, S = 5, (vocab.size + 31) // 32, 3, 14
    pool = get_pool()
    ref = [gm.GrammarMatcher(compiled) for _ in range(B)]
    s_ref = torch.tensor([m.slot for m in ref], dtype=torch.int32, device="cuda")
    bm = torch.empty((B, W), dtype=torch.int32, device="cuda")
    acc = torch.empty(B, dtype=torch.uint8, device="cuda")
    lg = torch.zeros(B, vocab.size, device="cuda", dtype=torch.bfloat16)
    rng = random.Random(11)
    toks, masks, accs = [None], [], []
    for s in range(S):
        batch_step(pool, s_ref, None if s == 0 else torch.tensor(toks[s], dtype=torch.int32, device="cuda"),
                   None if s == 0 else acc, bm, lg, recycle=True)
        masks.append(bm.clone())
        accs.append(acc.tolist() if s else None)
        allowed = ((bm.unsqueeze(-1) >> torch.arange(32, device="cuda", dtype=torch.int32)) & 1).reshape(B, -1)
        nxt = []
        for r in range(B):
            ids = allowed[r, :vocab.size].nonzero().flatten().tolist()
            nxt.append(rng.choice(ids))
        toks.append(nxt)
    new = [gm.GrammarMatcher(compiled) for _ in range(B)]
    bms = [torch.empty((B, W), dtype=torch.int32, device="cuda") for _ in range(n_buf)]
    bufs = [torch.zeros(B, vocab.size, device="cuda", dtype=torch.bfloat16) for _ in range(n_buf)]
    step = DecodeStepGraph(new, bms, bufs, recycle=True)

    def check(s):
        i = s % n_buf
        step.done[i].synchronize()
        assert torch.equal(bms[i], masks[s]), s
        if s:
            assert step.accepted_host[i].tolist() == accs[s], s

    for s in range(S):
        if s >= n_buf:
            check(s - n_buf)
        if s == 0:
            step.first(0)
            step.done[0].record(step.stream)
        else:
            step.run(toks[s], s % n_buf, wait=False)
    step.stream.synchronize()
    for s in range(S - n_buf, S):
        check(s)
    pool.check()


@pytest.mark.parametrize("copy_path", [False, True])
def test_decode_loop_native_equals_eager(copy_path, monkeypatch):
    """DecodeLoop (native gm_decoder_*: host ids -> K5 (ids in the launch
    parameters, or pinned staging + H2D copy with GMASK_DECODER_COPY=1) ->
    accepted flags D2H, steps queued back to back over 3 reused buffers) ==
    eager batch_step: same accepted flags and masks at every step."""
    import numpy as np
    import torch

    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200.engine import get_pool
    from paper_2411_15100_b200.graph import DecodeLoop
    from paper_2411_15100_b200.matcher import batch_step

    vocab = vocab_by_name("4000:mixed")
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    compiled = gm.GrammarCompiler(info).compile_builtin_json_grammar()
    B, W, n_buf, S = 7, (vocab.size + 31) // 32, 3, 16
    pool = get_pool()
    ref = [gm.GrammarMatcher(compiled) for _ in range(B)]
    s_ref = torch.tensor([m.slot for m in ref], dtype=torch.int32, device="cuda")
    bm = torch.empty((B, W), dtype=torch.int32, device="cuda")
    acc = torch.empty(B, dtype=torch.uint8, device="cuda")
    lg = torch.zeros(B, vocab.size, device="cuda", dtype=torch.bfloat16)
    rng = random.Random(5)
    toks, masks, accs = [None], [], []
    for s in range(S):
        batch_step(pool, s_ref, None if s == 0 else torch.tensor(toks[s], dtype=torch.int32, device="cuda"),
                   None if s == 0 else acc, bm, lg, recycle=True)
        masks.append(bm.clone())
        accs.append(acc.tolist() if s else [0] * B)
        allowed = ((bm.unsqueeze(-1) >> torch.arange(32, device="cuda", dtype=torch.int32)) & 1).reshape(B, -1)
        nxt = []
        for r in range(B):
            ids = allowed[r, :vocab.size].nonzero().flatten().tolist()
            nxt.append(rng.choice(ids) if rng.random() < 0.9 else vocab.size - 2)  # some rejected specials
        toks.append(nxt)
    new = [gm.GrammarMatcher(compiled) for _ in range(B)]
    bms = [torch.empty((B, W), dtype=torch.int32, device="cuda") for _ in range(n_buf)]
    bufs = [torch.zeros(B, vocab.size, device="cuda", dtype=torch.bfloat16) for _ in range(n_buf)]
    monkeypatch.setenv("GMASK_DECODER_COPY", "1" if copy_path else "0")
    loop = DecodeLoop(new, bms, bufs, recycle=True)
    out = np.zeros(B, dtype=np.uint8)

    def check(s):
        i = s % n_buf
        loop.flags(i, out=out, wait=True)
        assert out.tolist() == accs[s], s
        assert torch.equal(bms[i], masks[s]), s

    for s in range(S):
        if s >= n_buf:
            check(s - n_buf)
        loop.step(None if s == 0 else np.asarray(toks[s], dtype=np.int32), s % n_buf)
    torch.cuda.synchronize()
    for s in range(S - n_buf, S):
        check(s)
    loop.close()
    pool.check()


@pytest.mark.parametrize("grammar", ["json", "arithmetic"])
def test_k5_small_arena_collisions(grammar):
    """K5 with a 1,024-slot arena (hash-slot collisions frequent: exercises the
    deferred interning's end-of-kernel repair) stays bit-exact with the oracle
    over 60 steps of 16 requests."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, GMASK_ARENA_LOG2="10")
    res = subprocess.run([sys.executable, os.path.join(here, "_small_arena_k5.py"), grammar], env=env,
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    assert "ok" in res.stdout

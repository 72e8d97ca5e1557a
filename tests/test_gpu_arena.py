"""Arena reclamation (REF pstack.py:85-111: frames no live stack references
are reclaimed).  Two pools run the same requests in lockstep: pool A with a
tiny arena (1,024 frames) that is collected as the requests run, pool B with
a large one that never is.  Randomly nested arrays / objects over thousands
of steps —
far more distinct stacks than A could ever hold — must give identical masks
and accept flags in both, including rollbacks across a collection, with no
arena-full error in A; the released requests' frames are reclaimed."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(steps, collect_every, arena_log2=10, B=32):
    import torch

    import bench
    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200.engine import MatcherPool
    from paper_2411_15100_b200.matcher import SlotMatcher, batch_step

    vocab = gm.synth_vocab(32000)
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    # nested arrays / objects of arrays / objects: every nesting order is a
    # distinct stack, so the requests keep creating frames
    compiled = gm.GrammarCompiler(info).compile_grammar(
        'root ::= v\nv ::= "[" (v ("," v)*)? "]" | "{" (v ("," v)*)? "}" | "1"')
    pa = MatcherPool(capacity=B + 8, max_window=8, arena_log2=arena_log2)
    pb = MatcherPool(capacity=B + 8, max_window=8, arena_log2=22)
    ma = [SlotMatcher(compiled, 8, pa) for _ in range(B)]
    mb = [SlotMatcher(compiled, 8, pb) for _ in range(B)]
    sa = torch.tensor([m.slot for m in ma], dtype=torch.int32, device="cuda")
    sb = torch.tensor([m.slot for m in mb], dtype=torch.int32, device="cuda")
    W = (vocab.size + 31) // 32
    bma = torch.empty((B, W), dtype=torch.int32, device="cuda")
    bmb = torch.empty_like(bma)
    acc_a = torch.empty(B, dtype=torch.uint8, device="cuda")
    acc_b = torch.empty_like(acc_a)
    structural = torch.from_numpy(bench.structural_flags(vocab, frozenset(b'{}[]",:0123456789 '))).cuda()
    # random nesting: openers / closers preferred at random, so the requests
    # walk many distinct stacks (array and object frames in every order)
    def only(chars, need):
        return torch.tensor([t != vocab.eos_id and 0 < len(tok) <= 3 and all(c in chars for c in tok)
                             and any(c in need for c in tok) for t, tok in enumerate(vocab.tokens)], device="cuda")
    openers = only(set(b"[{,"), set(b"[{"))
    closers = only(set(b"]},1"), set(b"]}"))
    gen = torch.Generator(device="cuda").manual_seed(5)
    rows = torch.arange(B, device="cuda")
    toks = None
    peak = 0
    collections = 0
    for s in range(steps):
        batch_step(pa, sa, toks, acc_a if toks is not None else None, bma, recycle=True)
        batch_step(pb, sb, toks, acc_b if toks is not None else None, bmb, recycle=True)
        assert torch.equal(bma, bmb), f"mask diverged at step {s}"
        if toks is not None:
            assert torch.equal(acc_a, acc_b), f"accept diverged at step {s}"
        allowed = bench.unpack_allowed(bma, vocab.size)
        allowed[:, vocab.eos_id] &= (torch.rand(B, device="cuda", generator=gen) < 0.02)  # keep documents open
        u = torch.rand(B, 1, device="cuda", generator=gen)
        # 30 steps nesting deeper, 30 unwinding: every descent builds fresh
        # frames (random array / object order), the live set stays bounded
        deeper = (s // 30) % 2 == 0
        for pref, lo, hi in ((openers, 0.0, 0.7 if deeper else 0.1), (closers, 0.7 if deeper else 0.1, 0.8)):
            pick = (u >= lo) & (u < hi)
            sub = allowed & pref.view(1, -1)
            use = pick & sub.any(dim=1, keepdim=True)
            allowed = torch.where(use, sub, allowed)
        toks = bench.sample_tokens(allowed, structural, s, rows).to(torch.int32)
        if s % 97 == 50:  # roll back two requests by one token in both pools (history kept alive by the collector)
            for m in (ma[3], mb[3], ma[7], mb[7]):
                if m.info()["history_len"] >= 1:
                    m.rollback(1)
            batch_step(pa, sa, None, None, bma, recycle=False)
            batch_step(pb, sb, None, None, bmb, recycle=False)
            assert torch.equal(bma, bmb), f"mask diverged after rollback at step {s}"
            allowed = bench.unpack_allowed(bma, vocab.size)
            allowed[:, vocab.eos_id] = False
            toks = bench.sample_tokens(allowed, structural, s, rows).to(torch.int32)
        if collect_every and s % collect_every == collect_every - 1:
            st = pa.arena_stats()
            peak = max(peak, st["live"] + st["tombstones"])
            pa.collect()
            collections += 1
    pa.check()
    pb.check()
    return pa, pb, peak, collections, ma


def test_collection_keeps_long_runs_within_a_small_arena():
    pa, pb, peak, collections, ma = _run(steps=2500, collect_every=20)
    st_b = pb.arena_stats()
    st_a = pa.arena_stats()
    print("arena A", st_a, "peak", peak, "collections", collections, "| arena B (never collected)", st_b)
    # pool B (never collected) holds many more frames than pool A can
    assert st_b["live"] > 2 * st_a["capacity"], st_b
    assert collections >= 100 and peak <= st_a["capacity"]
    # releasing the requests frees their frames at the next collection
    for m in ma:
        m.release()
    pa.collect()
    assert pa.arena_stats()["live"] == 0

"""Subprocess body of test_k5_small_arena_collisions (GMASK_ARENA_LOG2=10):
K5 decode steps over a tiny arena, where the deferred interning's hash-slot
handles collide often, against the oracle's masks."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import paper_2411_15100_b200 as gm  # noqa: E402
from oracle import compile_oracle_bundle  # noqa: E402
from oracle.matcher import OracleMatcher  # noqa: E402
from paper_2411_15100_b200.engine import get_pool  # noqa: E402
from paper_2411_15100_b200.matcher import batch_step  # noqa: E402
from workloads import grammar_text, vocab_by_name  # noqa: E402


def main():
    vocab = vocab_by_name("4000:mixed")
    text = grammar_text(sys.argv[1])
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    compiled = gm.GrammarCompiler(info, cache_enabled=False).compile_grammar(text)
    ob = compile_oracle_bundle(text, vocab)
    B, W, S = 16, (vocab.size + 31) // 32, 60
    pool = get_pool()
    ms = [gm.GrammarMatcher(compiled) for _ in range(B)]
    refs = [OracleMatcher(ob) for _ in range(B)]
    slots = torch.tensor([m.slot for m in ms], dtype=torch.int32, device="cuda")
    bm = torch.empty((B, W), dtype=torch.int32, device="cuda")
    acc = torch.empty(B, dtype=torch.uint8, device="cuda")
    lg = torch.zeros(B, vocab.size, device="cuda", dtype=torch.bfloat16)
    rng = np.random.default_rng(3)
    toks = None
    for s in range(S):
        batch_step(pool, slots, None if toks is None else torch.tensor(toks, dtype=torch.int32, device="cuda"),
                   None if toks is None else acc, bm, lg, recycle=False)
        if toks is not None:
            assert acc.cpu().numpy().all(), s
        want = np.stack([r.fill() for r in refs]).view(np.int32)
        assert np.array_equal(bm.cpu().numpy(), want), f"mask mismatch at step {s}"
        allowed = np.unpackbits(want.view(np.uint8), axis=1, bitorder="little")[:, : vocab.size].astype(bool)
        allowed[:, vocab.eos_id] = False
        toks = []
        for r in range(B):
            ids = np.flatnonzero(allowed[r])
            toks.append(int(rng.choice(ids)))
        for r, t in zip(refs, toks):
            assert r.accept_token(t)
    pool.check()
    print("ok", get_pool().capacity)


if __name__ == "__main__":
    main()

"""Host-side cost of the per-step public calls (no device sync inside):
how long Python + ctypes take to enqueue one decode step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2411_15100_b200 as gm  # noqa: E402


def main():
    torch.cuda.set_device(0)
    vocab = gm.synth_vocab(128256)
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    compiled = gm.GrammarCompiler(info).compile_builtin_json_grammar()
    B = 128
    ms = [gm.GrammarMatcher(compiled) for _ in range(B)]
    batch = gm.BatchGrammarMatcher()
    bitmask = torch.empty((B, (vocab.size + 31) // 32), dtype=torch.int32, device="cuda")
    logits = torch.randn(B, vocab.size, device="cuda").to(torch.bfloat16)
    toks = torch.full((B,), 2**30, dtype=torch.int32, device="cuda")  # invalid ids: rejected, state unchanged
    acc = torch.empty(B, dtype=torch.uint8, device="cuda")
    pinned = torch.zeros(B, dtype=torch.int32).pin_memory()
    for name, fn in [
        ("batch_step (fill+apply only)", lambda: batch.batch_step(ms, None, bitmask=bitmask, logits=logits)),
        ("H2D copy 512 B", lambda: toks.copy_(pinned, non_blocking=True)),
        ("batch_fill_and_apply", lambda: batch.batch_fill_and_apply(ms, logits, bitmask)),
        ("apply_token_bitmask_inplace", lambda: gm.apply_token_bitmask_inplace(logits, bitmask)),
    ]:
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        n = 200
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        print(f"{name:34s} host enqueue {1e6 * (t1 - t0) / n:8.1f} us/call")


if __name__ == "__main__":
    main()

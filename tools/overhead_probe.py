"""Diagnostic: fixed per-launch cost after an L2 flush vs the work itself.

Times (CUDA events, mean of N) a 1-element torch kernel, a 32.8 MB torch
fill, K0 apply over real JSON masks, and K3 fill+apply, each with and without
the bench's 256 MiB L2 flush in front.  Run on the GPU box:
    python tools/overhead_probe.py
"""

import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200.engine import get_pool
    from paper_2411_15100_b200.matcher import batch_fill, batch_fill_apply

    dev = torch.device("cuda", 0)
    V, B = 128256, 128
    W = (V + 31) // 32
    vocab = gm.synth_vocab(V)
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    compiled = gm.GrammarCompiler(info, cache_enabled=False).compile_builtin_json_grammar()
    pool = get_pool()
    matchers = [gm.GrammarMatcher(compiled) for _ in range(B)]
    slots = torch.tensor([m.slot for m in matchers], dtype=torch.int32, device=dev)
    bitmask = torch.empty((B, W), dtype=torch.int32, device=dev)
    logits = torch.randn(B, V, device=dev).to(torch.bfloat16)
    tiny = torch.zeros(1, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
    batch_fill(pool, slots, bitmask)
    # a mixed mask: half the rows from the start state (structural: mostly masked), half all-allowed but 1 word
    real_mask = bitmask.clone()
    real_mask[B // 2:] = -1
    real_mask[B // 2:, ::7] = 0
    stream = torch.cuda.current_stream()
    a = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
    for _ in range(200):
        a @ a
    torch.cuda.synchronize()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]

    def t(fn, do_flush, n=100, spin=False):
        ms = []
        for i in range(n + 5):
            if do_flush:
                flush.zero_()
            if spin:  # keep the GPU busy so the host is ahead: measures GPU-side time only
                torch.cuda._sleep(100_000)
            e0, e1 = evs[i]
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            if i >= 5:
                ms.append(e0.elapsed_time(e1) * 1e3)
        return statistics.fmean(ms), statistics.median(ms)

    cases = {
        "empty (no kernel)": lambda: None,
        "tiny torch kernel": lambda: tiny.add_(1),
        "torch fill 32.8MB bf16": lambda: logits.fill_(float("-inf")),
        "K0 apply (start-state masks)": lambda: gm.apply_token_bitmask_inplace(logits, bitmask),
        "K0 apply (mixed masks)": lambda: gm.apply_token_bitmask_inplace(logits, real_mask),
        "K0 apply (all allowed)": lambda: gm.apply_token_bitmask_inplace(logits, torch.full_like(bitmask, -1)),
        "K2 fill": lambda: batch_fill(pool, slots, bitmask),
        "K3 fill+apply": lambda: batch_fill_apply(pool, slots, logits, bitmask),
    }
    allow_all = torch.full_like(bitmask, -1)
    cases["K0 apply (all allowed)"] = lambda: gm.apply_token_bitmask_inplace(logits, allow_all)
    masked = (~torch.from_numpy(__import__("numpy").unpackbits(bitmask.cpu().numpy().view("uint8"), axis=1,
                                                                  bitorder="little")[:, :V].astype(bool))).sum()
    print(f"start-state masked fraction {int(masked) / (B * V):.4f}")
    for name, fn in cases.items():
        for fl, sp in ((False, False), (True, False), (False, True), (True, True)):
            mean, med = t(fn, fl, spin=sp)
            print(f"{name:30s} flush={int(fl)} spin={int(sp)}  mean {mean:7.2f} us  median {med:7.2f} us")


if __name__ == "__main__":
    main()

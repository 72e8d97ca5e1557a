"""Dependent-walk stress: the uncached compile of
REF matcher.py:446-460 (CompileOptions(cache=False): no cached rows, every
token context-dependent) with the context classes off (GMASK_CTX_CLASSES=0),
so the fill walks EVERY non-special token of the vocabulary against each
request's full stack, per step — the reference's brute-force fill, on the
GPU.  Masks are checked against the cached engine's on the same
trajectories.  Reports K2 time per step, walked tokens/s and token bytes/s
(upper bound: every byte of every walked token).

    GMASK_CTX_CLASSES=0 python tools/walk_stress.py --vocab 128256 --batch 128 --steps 8
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--vocab", type=int, default=128256)
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--grammar", default="json")
    args = ap.parse_args()
    import bench
    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200.compat import device_vocab
    from paper_2411_15100_b200.engine import compile_on_device, get_pool
    from paper_2411_15100_b200.matcher import SlotMatcher, batch_accept, batch_fill, batch_recycle

    torch.cuda.set_device(0)
    vocab = gm.synth_vocab(args.vocab)
    dv = device_vocab(vocab)
    text = bench.grammar_text(args.grammar)

    class H:  # duck-typed CompiledGrammar for SlotMatcher
        def __init__(self, dev):
            self._dev = dev

    cached = H(compile_on_device(text, dv))
    uncached = H(compile_on_device(text, dv, uncached=True))
    pool = get_pool()
    B, V, W = args.batch, vocab.size, (vocab.size + 31) // 32
    mc = [SlotMatcher(cached, 1, pool) for _ in range(B)]
    mu = [SlotMatcher(uncached, 1, pool) for _ in range(B)]
    sc = torch.tensor([m.slot for m in mc], dtype=torch.int32, device="cuda")
    su = torch.tensor([m.slot for m in mu], dtype=torch.int32, device="cuda")
    bc = torch.empty((B, W), dtype=torch.int32, device="cuda")
    bu = torch.empty_like(bc)
    acc = torch.empty(B, dtype=torch.uint8, device="cuda")
    rows = torch.arange(B, device="cuda")
    structural = torch.from_numpy(bench.structural_flags(vocab)).cuda()
    lens = torch.tensor([len(t) for t in vocab.tokens], dtype=torch.float64)
    walked_bytes = float(lens[[t for t in range(V) if t not in vocab.special_tokens and len(vocab.tokens[t])]].sum())
    walked_tokens = sum(1 for t in range(V) if t not in vocab.special_tokens and len(vocab.tokens[t]))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    times, mism = [], 0
    for s in range(args.steps):
        batch_fill(pool, sc, bc)
        torch.cuda.synchronize()
        ev[0].record()
        batch_fill(pool, su, bu)
        ev[1].record()
        torch.cuda.synchronize()
        times.append(ev[0].elapsed_time(ev[1]) * 1e3)
        mism += int((bc != bu).any(dim=1).sum())
        toks = bench.sample_tokens(bench.unpack_allowed(bc, V), structural, s, rows).to(torch.int32)
        batch_accept(pool, sc, toks, acc)
        batch_accept(pool, su, toks, acc)
        batch_recycle(pool, sc)
        batch_recycle(pool, su)
    pool.check()
    us = sorted(times)[len(times) // 2]
    print(json.dumps({"grammar": args.grammar, "vocab": V, "batch": B, "steps": args.steps,
                      "context_classes": os.environ.get("GMASK_CTX_CLASSES", "1") != "0",
                      "k2_uncached_us_per_step_median": us, "k2_us_per_step_all": times,
                      "mask_rows_differing_from_cached": mism,
                      "walked_tokens_per_request_step": walked_tokens,
                      "walked_tokens_per_s": walked_tokens * B / (us * 1e-6),
                      "token_bytes_per_s_upper_bound": walked_bytes * B / (us * 1e-6)}))


if __name__ == "__main__":
    main()

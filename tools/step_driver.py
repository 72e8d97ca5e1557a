"""Minimal decode-loop driver for ncu captures (no timing, no sampler).

Runs the bench workload (JSON grammar, synth_vocab(128256), batch 128) for
``--steps`` decode steps through one kernel path, with tokens from a fixed
greedy-ish choice (lowest allowed non-EOS id after the first allowed word),
so ncu can capture e.g. the 10th launch of the K5 step kernel:

    ncu --set full --cache-control none -k regex:fill_kernel -s 10 -c 1 \
        -o gpurun_out/k5 python tools/step_driver.py --mode k5
"""

import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="k5", choices=["k5", "k3", "k2k0", "k4k3"])
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--grammar", default="json")
    args = ap.parse_args()
    import bench
    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200.engine import get_pool
    from paper_2411_15100_b200.matcher import batch_accept, batch_fill, batch_fill_apply, batch_step, batch_recycle

    torch.cuda.set_device(0)
    vocab = gm.synth_vocab(128256)
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    compiled = gm.GrammarCompiler(info).compile_grammar(bench.grammar_text(args.grammar))
    pool = get_pool()
    B = 128
    ms = [gm.GrammarMatcher(compiled, max_rollback_tokens=1) for _ in range(B)]
    dev = pool.device
    slots = torch.tensor([m.slot for m in ms], dtype=torch.int32, device=dev)
    rows = torch.arange(B, device=dev)
    structural = torch.from_numpy(bench.structural_flags(vocab, bench.WORKLOADS[args.grammar]["structural"])).to(dev)
    W = (vocab.size + 31) // 32
    bitmask = torch.empty((B, W), dtype=torch.int32, device=dev)
    acc = torch.empty(B, dtype=torch.uint8, device=dev)
    ring = [torch.randn((B, vocab.size), device=dev).to(torch.bfloat16) for _ in range(8)]
    toks = None
    for s in range(args.steps):
        lg = ring[s % 8]
        if args.mode == "k5":
            batch_step(pool, slots, toks, acc if toks is not None else None, bitmask, lg, recycle=True)
        else:
            if toks is not None:
                batch_accept(pool, slots, toks, acc)
                batch_recycle(pool, slots)
            if args.mode in ("k3", "k4k3"):
                batch_fill_apply(pool, slots, lg, bitmask)
            else:
                batch_fill(pool, slots, bitmask)
                gm.apply_token_bitmask_inplace(lg, bitmask)
        allowed = bench.unpack_allowed(bitmask, vocab.size)
        toks = bench.sample_tokens(allowed, structural, s, rows).to(torch.int32)
    torch.cuda.synchronize()
    pool.check()
    print("ok")


if __name__ == "__main__":
    main()

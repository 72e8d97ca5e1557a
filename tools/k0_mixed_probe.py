"""Diagnostic: K0 back to back (CUDA graph) over the bench's real decode
masks vs the same masks with every partially masked 16-byte chunk (8 bf16
tokens = one mask byte) rounded to fully masked: how much do the mixed
chunks' 2-byte stores cost?  python tools/k0_mixed_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import bench
    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200.engine import get_pool
    from paper_2411_15100_b200.matcher import batch_fill, batch_accept, batch_recycle

    dev = torch.device("cuda", 0)
    V, B, S = 128256, 128, 64
    W = (V + 31) // 32
    vocab = gm.synth_vocab(V)
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    comp = gm.GrammarCompiler(info).compile_builtin_json_grammar()
    pool = get_pool()
    ms = [gm.GrammarMatcher(comp, max_rollback_tokens=1) for _ in range(B)]
    slots = torch.tensor([m.slot for m in ms], dtype=torch.int32, device=dev)
    rows = torch.arange(B, device=dev)
    structural = torch.from_numpy(bench.structural_flags(vocab)).to(dev)
    masks = torch.empty((S, B, W), dtype=torch.int32, device=dev)
    acc = torch.empty(B, dtype=torch.uint8, device=dev)
    for s in range(S):
        batch_fill(pool, slots, masks[s])
        allowed = bench.unpack_allowed(masks[s], V)
        toks = bench.sample_tokens(allowed, structural, s, rows).to(torch.int32)
        batch_accept(pool, slots, toks, acc)
        batch_recycle(pool, slots)
    b = masks.view(torch.uint8)
    mixed = (b != 0) & (b != 255)
    print(f"mixed chunks: {int(mixed.sum())} of {b.numel()} ({float(mixed.float().mean()) * 100:.3f} %), "
          f"per step {int(mixed.sum()) / S:.0f}")
    rounded = torch.where(mixed, torch.zeros_like(b), b).view(torch.int32).view(S, B, W)
    ring = [torch.zeros(B, V, dtype=torch.bfloat16, device=dev) for _ in range(8)]

    def run(mk):
        g = torch.cuda.CUDAGraph()
        for s in range(4):
            gm.apply_token_bitmask_inplace(ring[s % 8], mk[s])
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            for s in range(S):
                gm.apply_token_bitmask_inplace(ring[s % 8], mk[s])
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / S

    for name, mk in (("real", masks), ("rounded", rounded), ("real", masks), ("rounded", rounded)):
        print(f"K0 {name:8s} {run(mk):6.2f} us/step")


if __name__ == "__main__":
    main()

"""Steady-state DRAM traffic of the K5 decode step: N
K5 steps back to back captured in ONE CUDA graph (as bench.py's value pass:
8 logits buffers of 32.8 MB, a fresh bitmask slice per step), replayed once
under ncu with --graph-profiling graph, so the -inf stores that are still
dirty in L2 when one launch ends are counted when later steps evict them.
Prints the algorithmic bytes per step (B*4W + 2*sum(masked)) so
traffic/step can be compared with it.

    ncu --graph-profiling graph --metrics dram__bytes_read.sum,dram__bytes_write.sum \\
        python tools/graph_traffic.py --steps 64
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
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--grammar", default="json")
    args = ap.parse_args()
    import bench
    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200.engine import get_pool
    from paper_2411_15100_b200.matcher import batch_step

    torch.cuda.set_device(0)
    vocab = gm.synth_vocab(128256)
    V = vocab.size
    compiled = gm.GrammarCompiler(gm.TokenizerInfo.from_vocabulary(vocab)).compile_grammar(
        bench.grammar_text(args.grammar))
    pool = get_pool()
    B, S = 128, args.steps
    ms = [gm.GrammarMatcher(compiled, max_rollback_tokens=1) for _ in range(B)]
    dev = pool.device
    slots = torch.tensor([m.slot for m in ms], dtype=torch.int32, device=dev)
    rows = torch.arange(B, device=dev)
    structural = torch.from_numpy(bench.structural_flags(vocab, bench.WORKLOADS[args.grammar]["structural"])).to(dev)
    W = (V + 31) // 32
    masks = torch.empty((S, B, W), dtype=torch.int32, device=dev)
    toks = torch.empty((S, B), dtype=torch.int32, device=dev)
    acc = torch.empty((S, B), dtype=torch.uint8, device=dev)
    ring = [torch.randn((B, V), device=dev).to(torch.bfloat16) for _ in range(8)]
    # record the trajectories (eager)
    for s in range(S):
        batch_step(pool, slots, toks[s - 1] if s else None, acc[s - 1] if s else None, masks[s], ring[s % 8],
                   recycle=True)
        toks[s] = bench.sample_tokens(bench.unpack_allowed(masks[s], V), structural, s, rows).to(torch.int32)
    torch.cuda.synchronize()
    masked = int((~bench.unpack_allowed(masks.view(-1, W), V)).sum())
    for m in ms:
        m.reset()
    stream = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    out = torch.empty_like(masks)
    with torch.cuda.stream(stream):
        batch_step(pool, slots, None, None, out[0], ring[0], recycle=True, stream=stream)  # warm-up outside
    torch.cuda.synchronize()
    for m in ms:
        m.reset()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=stream):
        for s in range(S):
            batch_step(pool, slots, toks[s - 1] if s else None, acc[s - 1] if s else None, out[s], ring[s % 8],
                       recycle=True, stream=stream)
    for m in ms:
        m.reset()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    same = bool(torch.equal(out, masks))
    algo = (B * 4 * W * S + 2 * masked) / S
    print(json.dumps({"steps": S, "batch": B, "V": V, "masks_equal_eager": same,
                      "algorithmic_bytes_per_step": algo, "masked_fraction": masked / (S * B * V)}))


if __name__ == "__main__":
    main()

"""Diagnostic: raw write / copy bandwidth and back-to-back per-launch cost.

Each case runs N launches back to back inside one CUDA-event bracket
(inputs rotate over an 8-buffer ring larger than L2) and prints the per-launch
time and GB/s.  Run on the GPU box:  python tools/write_bw_probe.py
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


GRAPH = "--graph" in sys.argv


def bracket(fn, n=200, warm=10):
    for i in range(warm):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if GRAPH:  # n launches captured once, replayed: device-side time per launch
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(n):
                fn(i)
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
    else:
        e0.record()
        for i in range(n):
            fn(i)
        e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n  # us per launch


def main():
    import paper_2411_15100_b200 as gm

    dev = torch.device("cuda", 0)
    B, V = 128, 128256
    W = (V + 31) // 32
    big = torch.empty(512 * 1024 * 1024, dtype=torch.bfloat16, device=dev)  # 1 GiB
    big2 = torch.empty_like(big)
    ring = [torch.zeros(B, V, dtype=torch.bfloat16, device=dev) for _ in range(8)]
    tiny = torch.zeros(1, device=dev)
    zero_mask = torch.zeros(B, W, dtype=torch.int32, device=dev)
    ones_mask = torch.full((B, W), -1, dtype=torch.int32, device=dev)
    half = torch.zeros(B, W, dtype=torch.int32, device=dev)
    half[::2] = -1
    # every 16-byte chunk mixed: alternate allowed/masked tokens
    mixed = torch.full((B, W), 0x55555555, dtype=torch.int32, device=dev)
    a = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
    for _ in range(100):
        a @ a
    rows_b = B * V * 2

    def rep(name, us, nbytes):
        print(f"{name:44s} {us:8.2f} us/launch   {nbytes / us / 1e3:8.1f} GB/s")

    rep("torch fill 1 GiB (write)", bracket(lambda i: big.fill_(1.0), n=20, warm=3), 2 * big.numel())
    rep("torch copy 1 GiB (read+write)", bracket(lambda i: big2.copy_(big), n=20, warm=3), 4 * big.numel())
    rep("torch fill 32.8 MB ring", bracket(lambda i: ring[i % 8].fill_(1.0)), rows_b)
    rep("tiny kernel", bracket(lambda i: tiny.add_(1)), 0.001)
    rep("K0 all masked (32.8 MB -inf + 2 MB mask)",
        bracket(lambda i: gm.apply_token_bitmask_inplace(ring[i % 8], zero_mask)), rows_b + 4 * B * W)
    rep("K0 all allowed (2 MB mask read)",
        bracket(lambda i: gm.apply_token_bitmask_inplace(ring[i % 8], ones_mask)), 4 * B * W)
    rep("K0 half rows masked",
        bracket(lambda i: gm.apply_token_bitmask_inplace(ring[i % 8], half)), rows_b // 2 + 4 * B * W)
    rep("K0 every other token masked (16.4 MB of 2-B stores)",
        bracket(lambda i: gm.apply_token_bitmask_inplace(ring[i % 8], mixed)), rows_b // 2 + 4 * B * W)
    f32 = [torch.zeros(B, V, dtype=torch.float32, device=dev) for _ in range(4)]
    rep("K0 fp32 all masked (65.7 MB)",
        bracket(lambda i: gm.apply_token_bitmask_inplace(f32[i % 4], zero_mask)), 2 * rows_b + 4 * B * W)
    # real decode-step masks: JSON start-state rows and string-interior-like rows
    if "--real" in sys.argv:
        from paper_2411_15100_b200.engine import get_pool
        from paper_2411_15100_b200.matcher import batch_fill
        info = gm.TokenizerInfo.from_vocabulary(gm.synth_vocab(V))
        comp = gm.GrammarCompiler(info).compile_builtin_json_grammar()
        ms = [gm.GrammarMatcher(comp) for _ in range(B)]
        for r, m in enumerate(ms[: B // 2]):
            m.accept_string(b'{"k": "ab')
        slots = torch.tensor([m.slot for m in ms], dtype=torch.int32, device=dev)
        real = torch.empty(B, W, dtype=torch.int32, device=dev)
        batch_fill(get_pool(), slots, real)
        allowed = ((real.unsqueeze(-1) >> torch.arange(32, device=dev, dtype=torch.int32)) & 1).reshape(B, -1)[:, :V]
        masked = int((allowed == 0).sum())
        print(f"real masks: masked fraction {masked / (B * V):.3f}")
        rep("K0 real masks (half string, half start)",
            bracket(lambda i: gm.apply_token_bitmask_inplace(ring[i % 8], real)), 2 * masked + 4 * B * W)
    rep("torch masked_fill_ bf16 (bool mask, dense)",
        bracket(lambda i: ring[i % 8].masked_fill_(ring[(i + 1) % 8] > 10, float("-inf")), n=50),
        3 * rows_b)


if __name__ == "__main__":
    main()

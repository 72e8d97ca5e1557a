"""K0 apply vs XGrammar 0.2.0's GPU apply kernels on the same B200, the same
masks and the same logits (SURVEY §2.2 names the
XGrammar Triton kernel, xgrammar/kernels/apply_token_bitmask_inplace_triton.py
:12-77, as the bar, and its CUDA kernel, ..._cuda.cu:63-113, JIT-built for the
current device, as the second one).

Masks come from real decode trajectories (bench.py's structure-biased sampler
over the engine's K3 fill), B = 128 rows, V = 128,256, bf16 logits.  Each
implementation applies S steps back to back (one fresh [B, W] mask slice and
one logits buffer of an 8-deep ring per step, inputs > L2) captured in one
CUDA graph, timed with one event pair, median of R brackets.  Every output is
compared with torch.where(bit, logits, -inf) on the first steps.

    python tools/apply_compare.py --grammar json --out gpurun_out/apply_json.json
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402


def record_masks(grammar: str, B: int, S: int, vocab_size: int):
    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200.engine import get_pool
    from paper_2411_15100_b200.matcher import batch_accept, batch_fill, batch_recycle

    dev = torch.device("cuda", 0)
    vocab = gm.synth_vocab(vocab_size)
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    compiled = gm.GrammarCompiler(info, cache_enabled=False).compile_grammar(bench.grammar_text(grammar))
    pool = get_pool()
    ms = [gm.GrammarMatcher(compiled, max_rollback_tokens=1) for _ in range(B)]
    slots = torch.tensor([m.slot for m in ms], dtype=torch.int32, device=dev)
    rows = torch.arange(B, device=dev)
    structural = torch.from_numpy(bench.structural_flags(vocab, bench.WORKLOADS[grammar]["structural"])).to(dev)
    force = bench.forced_token(vocab, grammar)
    W = (vocab.size + 31) // 32
    masks = torch.empty((S, B, W), dtype=torch.int32, device=dev)
    acc = torch.empty(B, dtype=torch.uint8, device=dev)
    for s in range(S):
        batch_fill(pool, slots, masks[s])
        allowed = bench.unpack_allowed(masks[s], vocab.size)
        toks = bench.sample_tokens(allowed, structural, s, rows, force=force).to(torch.int32)
        batch_accept(pool, slots, toks, acc)
        batch_recycle(pool, slots)
    torch.cuda.synchronize()
    del ms
    return masks, vocab.size


def time_impl(fn, masks, ring, reps: int):
    S = masks.shape[0]
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        for s in range(min(S, 3)):  # warm-up / JIT outside capture
            fn(ring[s % len(ring)], masks[s])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for s in range(S):
            fn(ring[s % len(ring)], masks[s])
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    out = []
    for _ in range(reps):
        g.replay()
        torch.cuda.synchronize()
        ev[0].record()
        g.replay()
        ev[1].record()
        torch.cuda.synchronize()
        out.append(ev[0].elapsed_time(ev[1]) * 1e3 / S)
    return statistics.median(out), out


def check_impl(fn, masks, V, n_check=6, dtype=torch.bfloat16):
    gen = torch.Generator(device="cuda").manual_seed(7)
    bad = 0
    for s in range(min(n_check, masks.shape[0])):
        x = torch.randn(masks.shape[1], V, device="cuda", generator=gen).to(dtype)
        ref = torch.where(bench.unpack_allowed(masks[s], V), x, torch.full_like(x, float("-inf")))
        y = x.clone()
        fn(y, masks[s])
        torch.cuda.synchronize()
        bad += int((y.view(torch.int16) != ref.view(torch.int16)).sum()) if dtype != torch.float32 else int(
            (y.view(torch.int32) != ref.view(torch.int32)).sum())
    return bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grammar", default="json", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--vocab", type=int, default=128256)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--out", default=None)
    ap.add_argument("--blend", type=int, nargs="*", default=[], help="also time K0 with these blend thresholds")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    import paper_2411_15100_b200 as gm

    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    masks, V = record_masks(args.grammar, args.batch, args.steps, args.vocab)
    W = masks.shape[2]
    allowed_frac = float(bench.unpack_allowed(masks.view(-1, W), V).float().mean())
    masked_total = int((~bench.unpack_allowed(masks.view(-1, W), V)).sum())
    es = 2 if dtype != torch.float32 else 4
    algo = (args.batch * 4 * W * args.steps + es * masked_total) / args.steps  # bytes per step
    phys = bench.physical_apply_bytes(masks, V, es)  # at 32-byte sector granularity
    ring = [torch.randn(args.batch, V, device="cuda").to(dtype) for _ in range(8)]
    peak, peak_kind = bench.measured_peak_hbm()

    from paper_2411_15100_b200 import _lib

    lib = _lib.load()
    default_blend = lib.gm_apply_set_blend(0)
    lib.gm_apply_set_blend(default_blend)

    def k0(blend):
        def fn(lg, bm):  # the policy is a launch parameter: captured with the graph
            old = lib.gm_apply_set_blend(blend)
            gm.apply_token_bitmask_inplace(lg, bm)
            lib.gm_apply_set_blend(old)
        return fn

    impls = {"k0_ours": k0(default_blend)}
    for n in args.blend:
        impls[f"k0_blend{n}"] = k0(n)
    errors = {}
    try:
        from xgrammar.kernels.apply_token_bitmask_inplace_triton import apply_token_bitmask_inplace_triton

        impls["xgrammar_triton"] = lambda lg, bm: apply_token_bitmask_inplace_triton(lg, bm)
    except Exception as exc:  # noqa: BLE001
        errors["xgrammar_triton"] = repr(exc)[:300]
    try:
        from xgrammar.kernels.apply_token_bitmask_inplace_cuda import apply_token_bitmask_inplace_cuda

        impls["xgrammar_cuda"] = lambda lg, bm: apply_token_bitmask_inplace_cuda(lg, bm)
    except Exception as exc:  # noqa: BLE001
        errors["xgrammar_cuda"] = repr(exc)[:300]
    res = {"grammar": args.grammar, "k0_default_blend": default_blend, "batch": args.batch, "V": V, "steps": args.steps, "dtype": args.dtype,
           "allowed_fraction": allowed_frac, "algorithmic_bytes_per_step": algo,
           "physical_bytes_per_step": phys, "peak_gbs": peak,
           "peak_source": peak_kind, "errors": errors, "impls": {}}
    for name, fn in impls.items():
        bad = check_impl(fn, masks, V, dtype=dtype)
        us, reps = time_impl(fn, masks, ring, args.reps)
        gbs = algo / (us * 1e-6) / 1e9
        pfrac = phys / (us * 1e-6) / 1e9 / peak
        res["impls"][name] = {"us_per_step": us, "reps_us": reps, "gbs": gbs, "frac_of_peak": gbs / peak,
                              "physical_frac_of_peak": pfrac, "mismatching_elements": bad}
        print(f"{args.grammar} {name}: {us:.2f} us/step  {gbs:.0f} GB/s  frac {gbs / peak:.3f}  "
              f"physical frac {pfrac:.3f}  bad {bad}", flush=True)
    if args.out:
        os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
        with open(args.out, "w") as fh:
            json.dump(res, fh, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "impls"}))


if __name__ == "__main__":
    main()

"""a batch of requests with DISTINCT JSON schemas.

1,024 schemas from a seeded mutation of the reference's SAMPLE_SCHEMA within
the supported keywords (property names, enum literals, minItems/maxItems,
optional/required split, scalar types); synth_vocab(128256); 128 requests
per GPU, each with its own schema.  Rank r of a torchrun job serves schemas
[r*128, (r+1)*128) and compiles exactly those (weak scaling: the requests a
rank serves are the only caches it needs, so the build needs no collective;
the replicated-cache path with the NCCL all-gather is bench.py's config 3).

Reports: compile ms per schema (front end + K1 cache build + assembly, one
GPU, sequential), the fill+apply step (K3) over the mixed-grammar batch, the
K5 decode step, parity with the reference (grammask, baseline/_ref) on sampled
requests over all steps, and the reference's compile
time for a sample of schemas (CPU reference, extrapolated to 1,024).

    python tools/bench_config5.py [--schemas 1024] [--per-gpu 128] [--steps 60]
"""

from __future__ import annotations

import argparse
import json
import os
import random
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402

WORDS = ["name", "unit", "count", "tags", "city", "time", "zone", "level", "mode", "query", "limit", "offset",
         "lang", "user", "id", "score", "kind", "price", "items", "notes", "start", "end", "flag", "color"]
LITS = ["get_weather", "get_time", "search", "lookup", "celsius", "fahrenheit", "fast", "slow", "on", "off",
        "red", "green", "blue", "low", "high", "auto"]


def mutate_schema(seed: int) -> dict:
    """Seeded mutation of SAMPLE_SCHEMA (REF grammars.py:53-65) within the
    supported keywords (REF schema.py:25-35)."""
    rng = random.Random(seed)
    n_props = rng.randint(2, 6)
    names = rng.sample(WORDS, n_props)
    props = {}
    for nm in names:
        kind = rng.choice(["enum", "string", "integer", "array", "number", "boolean"])
        if kind == "enum":
            props[nm] = {"enum": rng.sample(LITS, rng.randint(2, 4))}
        elif kind == "array":
            lo = rng.randint(0, 2)
            props[nm] = {"type": "array", "items": {"type": rng.choice(["string", "integer"])},
                         "minItems": lo, "maxItems": lo + rng.randint(1, 3)}
        else:
            props[nm] = {"type": kind}
    required = [nm for nm in names if rng.random() < 0.6] or [names[0]]
    return {"type": "object", "properties": props, "required": required, "additionalProperties": False}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--schemas", type=int, default=1024)
    ap.add_argument("--per-gpu", type=int, default=128)
    ap.add_argument("--vocab", type=int, default=128256)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--oracle-schemas", type=int, default=2)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))

    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200.engine import get_pool
    from paper_2411_15100_b200.matcher import batch_accept, batch_fill_apply, batch_recycle

    dev = torch.device("cuda", torch.cuda.current_device())
    vocab = gm.synth_vocab(args.vocab)
    V, W, B = vocab.size, (vocab.size + 31) // 32, args.per_gpu
    schemas = [mutate_schema(1000 + k) for k in range(args.schemas)]
    mine = schemas[rank * B:(rank + 1) * B]
    assert len(mine) == B, "not enough schemas for this rank"
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    compiler = gm.GrammarCompiler(info, cache_enabled=False)
    compiler.compile_json_schema(json.dumps(mine[0]))  # first-touch warm-up (not timed)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    compiled = []
    per_ms = []
    for sc in mine:
        t1 = time.perf_counter()
        compiled.append(compiler.compile_json_schema(json.dumps(sc)))
        torch.cuda.synchronize()
        per_ms.append((time.perf_counter() - t1) * 1e3)
    split = {k: statistics.fmean(c.compile_ms[k] for c in compiled) for k in compiled[0].compile_ms}
    keys = [c.stats.get("keys", 0) for c in compiled]
    compile_total_ms = (time.perf_counter() - t0) * 1e3
    # the same schemas compiled on host threads (GrammarCompiler.
    # compile_json_schemas: native front end + device build release the GIL)
    threaded = {}
    for nt in (4, 8):
        tc = gm.GrammarCompiler(info, cache_enabled=False, max_threads=nt)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        again = tc.compile_json_schemas([json.dumps(sc) for sc in mine])
        torch.cuda.synchronize()
        threaded[nt] = (time.perf_counter() - t1) * 1e3
        a0, b0 = compiled[0]._dev.cache.export(), again[0]._dev.cache.export()
        assert torch.equal(a0[0], b0[0]) and (a0[2] == b0[2]).all()
        del again

    pool = get_pool()
    matchers = [gm.GrammarMatcher(c, max_rollback_tokens=1) for c in compiled]
    slots = torch.tensor([m.slot for m in matchers], dtype=torch.int32, device=dev)
    rows = torch.arange(B, device=dev) + rank * B
    structural = torch.from_numpy(bench.structural_flags(vocab)).to(dev)
    bitmask = torch.empty((B, W), dtype=torch.int32, device=dev)
    gen = torch.Generator(device=dev).manual_seed(77 + rank)
    ring = [torch.randn(B, V, device=dev, generator=gen).to(torch.bfloat16) for _ in range(8)]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
    accepted = torch.empty(B, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    S = args.warmup + args.steps
    sample_rows = min(B, 4)
    keep = torch.empty((S, sample_rows, W), dtype=torch.int32, device=dev)
    masks_all = torch.empty((S, B, W), dtype=torch.int32, device=dev)
    toks_hist = torch.empty((S, B), dtype=torch.int32, device=dev)
    masked = torch.zeros(S, dtype=torch.int64, device=dev)
    ev = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(4)) for _ in range(S)]
    torch.cuda.synchronize()
    with bench.ClockSampler(torch.cuda.current_device()) as clocks:
        for s in range(S):
            flush.zero_()
            ev[s][0].record(stream)
            batch_fill_apply(pool, slots, ring[s % 8], bitmask)
            ev[s][1].record(stream)
            allowed = bench.unpack_allowed(bitmask, V)
            masked[s] = (~allowed).sum()
            keep[s] = bitmask[:sample_rows]
            masks_all[s] = bitmask
            toks = bench.sample_tokens(allowed, structural, s, rows).to(torch.int32)
            toks_hist[s] = toks
            ev[s][2].record(stream)
            batch_accept(pool, slots, toks, accepted)
            batch_recycle(pool, slots)
            ev[s][3].record(stream)
        torch.cuda.synchronize()
    pool.check()
    step_us = statistics.fmean(ev[s][0].elapsed_time(ev[s][1]) for s in range(args.warmup, S)) * 1e3
    acc_us = statistics.fmean(ev[s][2].elapsed_time(ev[s][3]) for s in range(args.warmup, S)) * 1e3

    # the same decode steps as K5 launches back to back (CUDA graph, one event
    # bracket; inputs larger than L2), every mask compared with the pass above
    from paper_2411_15100_b200.matcher import batch_step

    masks_t = torch.empty_like(masks_all)
    acc_t = torch.zeros((S, B), dtype=torch.uint8, device=dev)

    def k5(s):
        batch_step(pool, slots, toks_hist[s - 1] if s > 0 else None, acc_t[s - 1] if s > 0 else None, masks_t[s],
                   ring[s % 8], recycle=True)

    for m in matchers:
        m.reset()
    for s in range(args.warmup):
        k5(s)
    torch.cuda.synchronize()
    cap = torch.cuda.Stream(device=dev)
    g_w, g_t = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_w, stream=cap):
        for s in range(args.warmup):
            k5(s)
    with torch.cuda.graph(g_t, stream=cap):
        for s in range(args.warmup, S):
            k5(s)
    reps = []
    for _ in range(3):
        for m in matchers:
            m.reset()
        g_w.replay()
        torch.cuda.synchronize()
        ev[0][0].record(stream)
        g_t.replay()
        ev[0][1].record(stream)
        torch.cuda.synchronize()
        reps.append(ev[0][0].elapsed_time(ev[0][1]) / args.steps * 1e3)
    k5_b2b_us = statistics.median(reps)
    k5_mism = int((masks_t != masks_all).any(dim=2).sum())
    k5_acc = bool(acc_t[:S - 1].bool().all())

    # parity on the sampled rows (their own schemas) against the REFERENCE
    # itself (grammask from baseline/_ref: its schema lowering, compile and
    # Matcher), + its compile time; the oracle port only if it is missing
    toks_h = toks_hist.cpu().numpy()
    keep_h = keep.cpu().numpy()
    mism, checked, ocomp = 0, 0, []
    gmk = bench._grammask()
    kind = "reference" if gmk is not None else "port"
    for r in range(min(sample_rows, args.oracle_schemas)):
        if gmk is not None:
            from grammask.bundle import compile_bundle as ref_compile
            from grammask.matcher import Matcher as RefMatcher, TokenMask as RefMask
            from grammask.schema import schema_to_grammar_text as ref_schema
            from grammask.synthvocab import synth_vocab as ref_synth

            rv = ref_synth(V)
            t1 = time.perf_counter()
            ob = ref_compile(ref_schema(json.dumps(mine[r])), rv)
            ocomp.append(time.perf_counter() - t1)
            new_m = lambda: RefMatcher(ob, rv, history_window=1)  # noqa: E731
            mk = RefMask(V)

            def fill(m):
                m.fill_next_token_mask(mk)
                return np.frombuffer(mk.to_bytes(), dtype=np.int32)
        else:
            from oracle import compile_oracle_bundle
            from oracle.matcher import OracleMatcher
            from paper_2411_15100_b200.schema import schema_to_grammar_text

            t1 = time.perf_counter()
            ob = compile_oracle_bundle(schema_to_grammar_text(json.dumps(mine[r])), vocab)
            ocomp.append(time.perf_counter() - t1)
            new_m = lambda: OracleMatcher(ob, history_window=1)  # noqa: E731

            def fill(m):
                return m.fill().view(np.int32)
        m = new_m()
        for s in range(S):
            checked += 1
            if not np.array_equal(fill(m), keep_h[s, r]):
                mism += 1
            t = int(toks_h[s, r])
            assert m.accept_token(t)
            if t == vocab.eos_id:
                m = new_m()
    out = {
        "config": "SURVEY §8d config 5: distinct JSON schemas, synth_vocab(%d), %d requests/GPU" % (V, B),
        "schemas_total": args.schemas, "rank": rank, "world": world,
        "compile_ms_per_schema": {"mean": statistics.fmean(per_ms), "median": statistics.median(per_ms),
                                  "max": max(per_ms)},
        "compile_ms_rank_total": compile_total_ms,
        "compile_ms_rank_total_threads": threaded,
        "compile_split_ms_mean": split,
        "cache_keys_per_schema": {"mean": statistics.fmean(keys), "max": max(keys)},
        "k5_step_us_back_to_back": k5_b2b_us, "k5_mask_mismatches_vs_flushed_pass": k5_mism,
        "k5_all_accepted": k5_acc,
        "fill_apply_us_per_step_l2_flushed": step_us, "accept_recycle_us_per_step_l2_flushed": acc_us,
        "masked_fraction": float(masked[args.warmup:].double().mean().item()) / (B * V),
        "cpu_parity": {"kind": kind, "requests": min(sample_rows, args.oracle_schemas), "steps_checked": checked,
                       "mismatches": mism},
        "cpu_reference_compile_s_per_schema": statistics.fmean(ocomp) if ocomp else None,
        "cpu_reference_compile_s_1024_extrapolated_1core": (statistics.fmean(ocomp) * args.schemas) if ocomp else None,
        "cpu": bench._cpu_name(),
        "clocks": clocks.summary(),
        "l2": "k5 back to back: inputs larger than L2 (logits ring 8 x 32.8 MB); *_l2_flushed: 256 MiB flush before every step",
    }
    line = json.dumps(out)
    print(line)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(line + "\n")


if __name__ == "__main__":
    main()

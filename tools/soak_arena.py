"""Arena soak: one pool, many decode steps of
random-nesting JSON requests plus config-5 schema requests (16 distinct
mutated schemas), finished requests restarted in the step kernel, arena
collected whenever it is more than half full (MatcherPool.maybe_collect).
Reports arena occupancy over time, collections, and any per-request error
(an arena-full error would surface as flag bit 1).

    python tools/soak_arena.py --steps 1000000 --arena-log2 16
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=100000)
    ap.add_argument("--json-requests", type=int, default=32)
    ap.add_argument("--schema-requests", type=int, default=32)
    ap.add_argument("--arena-log2", type=int, default=16)
    ap.add_argument("--check-every", type=int, default=500)
    ap.add_argument("--vocab", type=int, default=32000)
    args = ap.parse_args()
    os.environ["GMASK_ARENA_LOG2"] = str(args.arena_log2)
    torch.cuda.set_device(0)
    import bench
    import paper_2411_15100_b200 as gm
    from bench_config5 import mutate_schema
    from paper_2411_15100_b200.engine import get_pool
    from paper_2411_15100_b200.matcher import batch_step

    vocab = gm.synth_vocab(args.vocab)
    comp = gm.GrammarCompiler(gm.TokenizerInfo.from_vocabulary(vocab))
    js = comp.compile_builtin_json_grammar()
    schemas = [comp.compile_json_schema(json.dumps(mutate_schema(9000 + i))) for i in range(16)]
    ms = [gm.GrammarMatcher(js, max_rollback_tokens=4) for _ in range(args.json_requests)]
    ms += [gm.GrammarMatcher(schemas[i % 16], max_rollback_tokens=4) for i in range(args.schema_requests)]
    pool = get_pool()
    B = len(ms)
    slots = torch.tensor([m.slot for m in ms], dtype=torch.int32, device="cuda")
    W = (vocab.size + 31) // 32
    bm = torch.empty((B, W), dtype=torch.int32, device="cuda")
    acc = torch.empty(B, dtype=torch.uint8, device="cuda")
    structural = torch.from_numpy(bench.structural_flags(vocab)).cuda()

    def only(chars, need):
        return torch.tensor([t != vocab.eos_id and 0 < len(tok) <= 3 and all(c in chars for c in tok)
                             and any(c in need for c in tok) for t, tok in enumerate(vocab.tokens)], device="cuda")

    openers = only(set(b'[{":, '), set(b"[{"))
    closers = only(set(b']}", '), set(b"]}"))
    is_json = torch.zeros(B, 1, dtype=torch.bool, device="cuda")
    is_json[: args.json_requests] = True
    gen = torch.Generator(device="cuda").manual_seed(11)
    rows = torch.arange(B, device="cuda")
    toks = None
    timeline, collections, err_steps = [], 0, 0
    max_occ = 0.0
    t0 = time.perf_counter()
    for s in range(args.steps):
        batch_step(pool, slots, toks, acc if toks is not None else None, bm, recycle=True)
        allowed = bench.unpack_allowed(bm, vocab.size)
        u = torch.rand(B, 1, device="cuda", generator=gen)
        deeper = (s // 40) % 2 == 0
        for pref, lo, hi in ((openers, 0.0, 0.6 if deeper else 0.1), (closers, 0.6 if deeper else 0.1, 0.75)):
            pick = (u >= lo) & (u < hi) & is_json
            sub = allowed & pref.view(1, -1)
            use = pick & sub.any(dim=1, keepdim=True)
            allowed = torch.where(use, sub, allowed)
        toks = bench.sample_tokens(allowed, structural, s, rows).to(torch.int32)
        if s % args.check_every == args.check_every - 1:
            f = acc.cpu().numpy()
            if (f & 2).any():
                err_steps += 1
                pool.raise_slot_errors(slots, f)
            st = pool.arena_stats()
            max_occ = max(max_occ, st["occupancy"])
            did = pool.maybe_collect(0.5)
            collections += did
            after = pool.arena_stats() if did else st
            timeline.append({"step": s + 1, "live": st["live"], "tombstones": st["tombstones"],
                             "occupancy": round(st["occupancy"], 4), "collected": bool(did),
                             "live_after": after["live"], "elapsed_s": round(time.perf_counter() - t0, 1)})
    torch.cuda.synchronize()
    pool.check()
    out = {"steps": args.steps, "requests": B, "json_requests": args.json_requests,
           "schema_requests": args.schema_requests, "distinct_schemas": 16, "arena_slots": 1 << args.arena_log2,
           "collections": collections, "max_occupancy": max_occ, "error_checks_with_errors": err_steps,
           "request_steps": args.steps * B, "wall_s": round(time.perf_counter() - t0, 1),
           "timeline": timeline[:: max(1, len(timeline) // 40)] + timeline[-1:]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()

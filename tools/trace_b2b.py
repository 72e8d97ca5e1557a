"""Back-to-back timeline of the K5 step (diagnostics, traced build):
  bash tools/trace.sh build         # here (tools/variants/libgmask_trace.so)
  GMASK_NO_BUILD=1 GMASK_LIB=tools/variants/libgmask_trace.so GMASK_TRACE=2 python tools/trace_b2b.py
Records S K5 steps of the bench workload (eager), replays them back to back
in one CUDA graph, and reads every CTA's stamps for the last 16 launches
(GMASK_TRACE=2 ring): per launch the span (first CTA past its grid wait ->
last CTA end), the gap to the next launch, the CTA launch-to-start wait, and
the p50 / max of every phase."""

import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

PH = ["header", "accept", "setup", "ctx", "walks", "merge", "apply"]


def main(S=48, grammar="json"):
    import bench
    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200 import _lib
    from paper_2411_15100_b200.engine import get_pool
    from paper_2411_15100_b200.matcher import batch_step

    torch.cuda.set_device(0)
    vocab = gm.synth_vocab(128256)
    V = vocab.size
    compiled = gm.GrammarCompiler(gm.TokenizerInfo.from_vocabulary(vocab)).compile_grammar(bench.grammar_text(grammar))
    pool = get_pool()
    B = 128
    ms = [gm.GrammarMatcher(compiled, max_rollback_tokens=1) for _ in range(B)]
    dev = pool.device
    slots = torch.tensor([m.slot for m in ms], dtype=torch.int32, device=dev)
    rows = torch.arange(B, device=dev)
    structural = torch.from_numpy(bench.structural_flags(vocab, bench.WORKLOADS[grammar]["structural"])).to(dev)
    force = bench.forced_token(vocab, grammar)
    W = (V + 31) // 32
    masks = torch.empty((S, B, W), dtype=torch.int32, device=dev)
    toks = torch.empty((S, B), dtype=torch.int32, device=dev)
    acc = torch.empty((S, B), dtype=torch.uint8, device=dev)
    ring = [torch.randn((B, V), device=dev).to(torch.bfloat16) for _ in range(8)]
    for s in range(S):
        batch_step(pool, slots, toks[s - 1] if s else None, acc[s - 1] if s else None, masks[s], ring[s % 8],
                   recycle=True)
        toks[s] = bench.sample_tokens(bench.unpack_allowed(masks[s], V), structural, s, rows, force=force).to(torch.int32)
    torch.cuda.synchronize()
    for m in ms:
        m.reset()
    stream = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=stream):
        for s in range(S):
            batch_step(pool, slots, toks[s - 1] if s else None, acc[s - 1] if s else None, masks[s], ring[s % 8],
                       recycle=True, stream=stream)
    for m in ms:
        m.reset()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    cap, R = pool.capacity, 16
    NB = 64 + 16 * cap * (1 + R) + cap
    buf = (C.c_uint64 * NB)()
    _lib.check(_lib.load().gm_pool_trace(pool.handle, buf, NB))
    launches = []
    for r in range(R):
        recs = []
        for c in range(B):
            base = 64 + 16 * cap * (1 + r) + 16 * c
            recs.append([buf[base + k] for k in range(16)])
        launches.append(recs)
    launches.sort(key=lambda recs: min(x[0] for x in recs))
    out = []
    for j, recs in enumerate(launches):
        t0 = min(x[0] for x in recs)
        t_launch = min(x[13] for x in recs)
        t1 = max(x[7] for x in recs)
        row = {"span_us": (t1 - t0) / 1e3, "launch_to_first_start_us": (t0 - t_launch) / 1e3}
        if j + 1 < len(launches):
            row["gap_to_next_us"] = (min(x[0] for x in launches[j + 1]) - t1) / 1e3
            row["next_resident_before_end_us"] = (t1 - min(x[13] for x in launches[j + 1])) / 1e3
        for k, name in enumerate(PH):
            d = [(x[k + 1] - x[k]) / 1e3 for x in recs if x[k] and x[k + 1] and x[k + 1] >= x[k]]
            if d:
                row[name] = (round(statistics.median(d), 2), round(max(d), 2))
        # the slowest accepts of this launch: token bytes, stacks, fresh frames
        slow = sorted(recs, key=lambda x: -(x[2] - x[1]) if x[2] and x[1] else 0)[:4]
        row["slow_accepts"] = [((x[2] - x[1]) / 1e3, x[9] & 0xFFFF, (x[9] >> 16) & 0xFF, x[9] >> 24,
                                (x[8] - x[1]) / 1e3 if x[8] else None) for x in slow if x[2] and x[1]]
        accs = [((x[2] - x[1]) / 1e3, x[9]) for x in recs if x[2] and x[1]]
        row["accept_by_kind"] = {}
        for t, info in accs:
            kind = "walked" if (info & 0xFFFF) else "no-walk"
            key = f"{kind} frames={info >> 24 if info else 0} stacks={(info >> 16) & 0xFF}"
            row["accept_by_kind"].setdefault(key, []).append(round(t, 2))
        ends = sorted((x[7] - t0) / 1e3 for x in recs)
        row["cta_end_p50_max"] = (round(ends[len(ends) // 2], 2), round(ends[-1], 2))
        # when each CTA's apply can start (its merged words are final)
        ready = sorted((x[6] - t0) / 1e3 for x in recs if x[6])
        if ready:
            row["apply_start_p10_p50_p90_max"] = tuple(round(ready[min(len(ready) - 1, int(q * len(ready)))], 2)
                                                       for q in (0.1, 0.5, 0.9, 1.0))
        walked = [(x[10] >> 40) & 0xFFFF for x in recs]
        row["deps_walked_mean_max"] = (round(sum(walked) / len(walked), 1), max(walked))
        out.append(row)
    keys = ["span_us", "gap_to_next_us", "launch_to_first_start_us", "next_resident_before_end_us"] + PH + [
        "cta_end_p50_max", "apply_start_p10_p50_p90_max"]
    summ = {}
    for k in keys:
        vals = [r[k] for r in out if k in r]
        if not vals:
            continue
        if isinstance(vals[0], tuple):
            summ[k] = tuple(round(statistics.median(v[j] for v in vals), 2) for j in range(len(vals[0])))
        else:
            summ[k] = round(statistics.median(vals), 2)
    print(json.dumps({"launches": len(out), "median_over_launches": summ, "per_launch": out}))


if __name__ == "__main__":
    g = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--grammar=")), "json")
    main(grammar=g)

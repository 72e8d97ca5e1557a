"""Diagnostics: per-phase timing of the accept (K4) and fill (K2) kernels.

Runs the bench workload (JSON grammar, synth_vocab(128256), batch 128) with
GMASK_TRACE=1 so CTA 0 of every launch records %globaltimer stamps at phase
boundaries, and prints the phase deltas for a few steps (cold L2: a 256 MiB
flush before each step, as in bench.py).

    GMASK_TRACE=1 python tools/trace_step.py
"""

import ctypes as C
import os
import sys

os.environ.setdefault("GMASK_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2411_15100_b200 as gm  # noqa: E402
from paper_2411_15100_b200 import _lib  # noqa: E402
from paper_2411_15100_b200.engine import get_pool  # noqa: E402
from paper_2411_15100_b200.matcher import (  # noqa: E402
    batch_accept, batch_fill, batch_fill_apply, batch_recycle, batch_step)


PHASES = ["header", "accept", "setup", "ctx", "walks", "merge", "apply"]


def timeline(buf, nc):
    """Per-CTA timeline (absolute %globaltimer stamps at 64 + 8c): span of
    the kernel and p50 / max of every phase over the CTAs."""
    import statistics

    rec = [[buf[64 + 16 * c + k] for k in range(16)] for c in range(nc)]
    t0 = min(r[0] for r in rec)
    t1 = max(r[7] for r in rec)
    out = [f"span {(t1 - t0) / 1e3:.2f} us, CTA start spread {(max(r[0] for r in rec) - t0) / 1e3:.2f}"]
    for k, name in enumerate(PHASES):
        d = []
        for r in rec:
            a, b = r[k], r[k + 1]
            if k == 3 and not b:  # no ctx stamp (no dependents): fold into walks
                continue
            if k == 4 and not a:
                a = r[3]
            if k == 1 and not b:
                continue
            if k == 2 and not a:
                a = r[1]
            if a and b and b >= a:
                d.append((b - a) / 1e3)
        if d:
            out.append(f"{name} {statistics.median(d):.2f}/{max(d):.2f}")
    wk = [(r[10] >> 40) & 0xFFFF for r in rec]
    out.append(f"deps walked per CTA: mean {sum(wk) / len(wk):.1f} max {max(wk)}")
    ends = sorted((r[7] - t0) / 1e3 for r in rec)
    out.append(f"CTA end p50 {ends[len(ends) // 2]:.2f} max {ends[-1]:.2f}")
    # the slowest CTAs: where their time went
    order = sorted(range(nc), key=lambda c: -(rec[c][7] - rec[c][0]))[:3]
    for c in order:
        r = rec[c]
        walk = (f"walk {(r[8] - r[1]) / 1e3:.2f} commit {(r[11] - r[8]) / 1e3:.2f} pub+ {(r[2] - r[11]) / 1e3:.2f}"
                if r[8] and r[2] and r[11] else "no reg walk")
        info = r[9]
        out.append(f"[slow {(r[7] - r[0]) / 1e3:.2f}: acc {(r[2] - r[1]) / 1e3 if r[2] else 0:.2f} ({walk}; "
                   f"len {info & 0xFFFF} stacks {(info >> 16) & 0xFF} frames {info >> 24}) "
                   f"deps {r[10] & 0xFFFFFFFF} tops {(r[10] >> 32) & 0xFF} walked {(r[10] >> 40) & 0xFFFF} walks {(r[5] - (r[4] or r[3])) / 1e3:.2f}]")
    # median split of the register-walk accept over CTAs that took it
    # (hdr -> accept_one -> walk -> prefetch -> commit -> ring -> header state)
    segs = [("pre", 1, 12), ("walk", 12, 8), ("pref", 8, 13), ("->commit", 13, 14), ("commit", 14, 11),
            ("ring", 11, 15), ("hstate+", 15, 2)]
    parts = []
    for name, a, b in segs:
        d = [(r[b] - r[a]) / 1e3 for r in rec if r[a] and r[b] and r[b] >= r[a]]
        if d:
            parts.append(f"{name} {statistics.median(d):.2f}/{max(d):.2f}")
    out.append("accept split p50/max: " + " ".join(parts))
    return " | ".join(out)


def main(steps=12, flush=True, fused=False, grammar="json", step_mode=False):
    torch.cuda.set_device(0)
    vocab = gm.synth_vocab(128256)
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    compiled = gm.GrammarCompiler(info).compile_grammar(bench.grammar_text(grammar))
    pool = get_pool()
    B = 128
    ms = [gm.GrammarMatcher(compiled, max_rollback_tokens=1) for _ in range(B)]
    dev = pool.device
    slots = torch.tensor([m.slot for m in ms], dtype=torch.int32, device=dev)
    rows = torch.arange(B, device=dev)
    structural = torch.from_numpy(bench.structural_flags(vocab, bench.WORKLOADS[grammar]["structural"])).to(dev)
    force = bench.forced_token(vocab, grammar)
    bitmask = torch.empty((B, (vocab.size + 31) // 32), dtype=torch.int32, device=dev)
    acc = torch.empty(B, dtype=torch.uint8, device=dev)
    fl = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
    logits = torch.randn((B, vocab.size), dtype=torch.bfloat16, device=dev)
    NB = 64 + 16 * pool.capacity
    buf = (C.c_uint64 * NB)()
    lib = _lib.load()
    for s in range(steps):
        if flush:
            fl.zero_()
        if step_mode:
            batch_step(pool, slots, toks if s > 0 else None, acc if s > 0 else None, bitmask,
                       logits if fused else None, recycle=True)
        elif fused:
            batch_fill_apply(pool, slots, logits, bitmask)
        else:
            batch_fill(pool, slots, bitmask)
        torch.cuda.synchronize()
        _lib.check(lib.gm_pool_trace(pool.handle, buf, NB))
        f = [buf[16 + k] for k in range(8)]
        ns = max(1, buf[63])
        nc = B * ns
        kname = ("K5" if step_mode else "K3" if fused else "K2")
        print(f"  {kname} x{ns} {timeline(buf, nc)}")
        extra = f"deps={buf[24]} key0={C.c_int64(buf[25]).value} ntops={buf[26]}"
        if buf[24]:
            ln = buf[44] & 0xFFFF
            walk = [(buf[32 + b] & 0xFFFFFFFFFFFF, buf[32 + b] >> 48) for b in range(min(ln, 12))]
            extra += f" | walk0 len={ln} spill={(buf[44] >> 16) & 0xFFFF} nchain={buf[44] >> 32} cycles/byte(n)={walk}"
            for b in range(13):
                buf[32 + b] = 0
        allowed = bench.unpack_allowed(bitmask, vocab.size)
        toks = bench.sample_tokens(allowed, structural, s, rows, force=force).to(torch.int32)
        if step_mode and s == steps - 1:
            print(f"  arena slots used: {lib.gm_pool_arena_used(pool.handle)}")
        if step_mode:
            fp = [buf[16], buf[17], buf[48], buf[18], buf[20], buf[21], buf[22], buf[23]]
            d = [(fp[k + 1] - fp[k]) / 1e3 if fp[k + 1] >= fp[k] > 0 else float("nan") for k in range(7)]
            print(f"step {s:2d} K5 CTA0 phases(us): header {d[0]:.2f} accept {d[1]:.2f} setup {d[2]:.2f} "
                  f"stage+ctx {d[3]:.2f} walks {d[4]:.2f} barrier {d[5]:.2f} merge {d[6]:.2f} "
                  f"deps={buf[24]} ntops={buf[26]}")
            a = [buf[17], buf[49], buf[3], buf[4], buf[5], buf[48]]
            da = [(a[k + 1] - a[k]) / 1e3 if a[k + 1] >= a[k] > 0 else float("nan") for k in range(5)]
            print(f"         accept split(us): stage {da[0]:.2f} walk {da[1]:.2f} commit {da[2]:.2f} "
                  f"publish {da[3]:.2f} tail {da[4]:.2f} blob_bytes={buf[50]} | dry walk {buf[51] / 1e3:.2f} us "
                  f"(n={buf[52] & 0xFFFFFFFF}, len={buf[52] >> 32}, arena loads={buf[53] & 0xFFFF}, "
                  f"frames={(buf[53] >> 16) & 0xFFFF}, spill={(buf[53] >> 32) & 0xFF}, nchain={(buf[53] >> 40) & 0xFF}, "
                  f"top0=chain0:{(buf[53] >> 48) & 1}) cycles init {buf[54]} per byte {[buf[55 + b] for b in range(min(4, buf[52] >> 32))]} | 2nd: init {buf[59]} per byte {[buf[60 + b] for b in range(min(4, buf[52] >> 32))]}")
            print(f"         load probes (cycles): generic smem {buf[46] & 0xFFFF}, again {(buf[46] >> 16) & 0xFFFF}, "
                  f"LDS {(buf[46] >> 32) & 0xFFFF}, generic fast[] {(buf[46] >> 48) & 0xFFFF}")
            for k in (3, 4, 5, 48, 49):
                buf[k] = 0
            continue
        if flush:
            fl.zero_()
        torch.cuda.synchronize()
        batch_accept(pool, slots, toks, acc)
        torch.cuda.synchronize()
        _lib.check(lib.gm_pool_trace(pool.handle, buf, NB))
        a = [buf[k] for k in range(6)]
        batch_recycle(pool, slots)

        def deltas(v):
            out = []
            for k in range(1, len(v)):
                out.append(f"{(v[k] - v[k - 1]) / 1e3:6.2f}" if v[k] and v[k - 1] and v[k] >= v[k - 1] else "   -  ")
            return " ".join(out)

        print(f"step {s:2d} fill phases(us): {deltas(f)}   accept phases(us): {deltas(a)}  tok0={int(toks[0])} {extra}")


if __name__ == "__main__":
    g = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--grammar=")), "json")
    main(flush="--warm" not in sys.argv, fused="--fused" in sys.argv, grammar=g, step_mode="--step" in sys.argv)

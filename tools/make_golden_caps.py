"""Golden fixtures for wide stack sets, from the REAL reference (grammask,
imported from /root/reference/pkg/src).  Run here:

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_caps.py

Writes tests/golden/caps.json.gz:

* ``ambig40``: ``root ::= a1 | ... | a40``, ``ai ::= "x" ai "y" | "z<i>"``.
  Every prefix x^k keeps one stack per alternative alive (40 > the engine's
  32-stack local walkers), while the reference's closure stays under its
  4096-state cap (REF matcher.py:116, 188-189).  Trajectories over a small
  vocabulary with the reference's mask after every prefix (full words).
* ``ambig_over_cap``: the same shape with 4200 alternatives: the reference's
  cache build raises StateLimitError (cap 4096, REF cache.py:58, 137-138) —
  so must ours (more than kWideCap = 4096 stacks).
* ``ambig300``: 300 alternatives (wide ring entries and batched fills).
* ``dfa_blowup``: ``[ab]* "a" [ab]{17} "."`` — its subset construction
  would need 2^18 states (over the front end's 200k limit), so the rule keeps
  an epsilon-free NFA and the walkers carry up to 18 stacks.
* ``deep_ambig``: nested ambiguity (two alternatives per level and 12
  levels of nesting: a ::= "(" a ")" | "(" b ")" ...), masks after every
  prefix.
"""

from __future__ import annotations

import gzip
import json
import random
import sys
import time
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, str(Path(__file__).resolve().parent))

import make_golden as mg  # noqa: E402  (puts the reference on sys.path)
from grammask.bundle import compile_bundle  # noqa: E402
from grammask.matcher import Matcher  # noqa: E402
from grammask.pda import StateLimitError  # noqa: E402
from grammask.vocab import vocab_from_tokens  # noqa: E402


def ambig_grammar(n: int) -> str:
    alts = " | ".join(f"a{i}" for i in range(1, n + 1))
    rules = "\n".join(f'a{i} ::= "x" a{i} "y" | "z{i}"' for i in range(1, n + 1))
    return f"root ::= {alts}\n{rules}\n"


DEEP = """root ::= item+
item ::= p | q
p ::= "(" item ")" | "(" "a" ")" | "a"
q ::= "(" item ")" | "(" "b" ")" | "b"
"""


def caps_vocab():
    toks = [b"x", b"y", b"z", b"xx", b"xxx", b"yy", b"yyy", b"(", b")", b"((", b"))", b"a", b"b", b"(a", b"b)",
            b"ab", b"ba", b"aa", b"bb", b"aab", b"bab", b"abba", b".", b"a."]
    toks += [str(d).encode() for d in range(10)]
    toks += [f"z{i}".encode() for i in range(1, 41)] + [f"{i}y".encode() for i in range(1, 41)]
    seen, out = set(), []
    for t in toks:
        if t not in seen:
            seen.add(t)
            out.append(t)
    return out + [b"<eos>"]


def record(bundle, vocab, n_traj, max_steps, seed, prefer):
    rng = random.Random(seed)
    out = []
    for _ in range(n_traj):
        m = Matcher(bundle, vocab, history_window=1)
        toks, masks, stacks = [], [], []
        for step in range(max_steps):
            mask = m.next_token_mask()
            masks.append(mg.mask_record(mask, True))
            stacks.append(len(m._tops))
            ids = [int(t) for t in mask.allowed_ids()]
            if not ids:
                break
            pref = [t for t in ids if vocab.tokens[t] and vocab.tokens[t][:1] in prefer(step)]
            pick = rng.choice(pref) if pref and rng.random() < 0.85 else rng.choice(ids)
            toks.append(pick)
            if pick == vocab.eos_id:
                break
            assert m.accept_token(pick)
        out.append({"tokens": toks, "masks": masks, "ref_stacks": stacks})
    return out


def main():
    t0 = time.time()
    toks = caps_vocab()
    vocab = vocab_from_tokens(toks, eos_id=len(toks) - 1, special=[len(toks) - 1])
    doc = {"vocab_tokens": [t.hex() for t in toks], "cases": {}}

    g40 = ambig_grammar(40)
    b = compile_bundle(g40, vocab)
    trajs = record(b, vocab, 6, 24, 11, lambda s: (b"x",) if s < 8 else (b"z", b"1", b"2", b"3", b"y"))
    doc["cases"]["ambig40"] = {"grammar": g40, "trajectories": trajs}
    print("ambig40", max(max(t["ref_stacks"]) for t in trajs), "stacks max", f"{time.time() - t0:.1f}s", flush=True)

    g300 = ambig_grammar(300)
    b = compile_bundle(g300, vocab)
    trajs = record(b, vocab, 3, 20, 13, lambda s: (b"x",) if s < 6 else (b"z", b"1", b"2", b"5", b"y"))
    doc["cases"]["ambig300"] = {"grammar": g300, "trajectories": trajs}
    print("ambig300", max(max(t["ref_stacks"]) for t in trajs), "stacks max", f"{time.time() - t0:.1f}s", flush=True)

    gdeep = DEEP
    b = compile_bundle(gdeep, vocab)
    trajs = record(b, vocab, 6, 40, 12, lambda s: (b"(",) if s < 14 else (b")", b"a", b"b"))
    doc["cases"]["deep_ambig"] = {"grammar": gdeep, "trajectories": trajs}
    print("deep", max(max(t["ref_stacks"]) for t in trajs), "stacks max", f"{time.time() - t0:.1f}s", flush=True)

    gdfa = 'root ::= [ab]* "a" [ab]{17} "."\n'
    b = compile_bundle(gdfa, vocab)
    trajs = record(b, vocab, 6, 40, 14, lambda s: (b"a", b"b"))
    doc["cases"]["dfa_blowup"] = {"grammar": gdfa, "trajectories": trajs}
    print("dfa_blowup", max(max(t["ref_stacks"]) for t in trajs), "stacks max", f"{time.time() - t0:.1f}s", flush=True)

    gbig = ambig_grammar(4200)
    try:
        compile_bundle(gbig, vocab)
        verdict = None
    except StateLimitError as exc:
        verdict = ["StateLimitError", str(exc)]
    doc["cases"]["ambig_over_cap"] = {"grammar_alternatives": 4200, "compile_error": verdict}
    print("over cap", verdict, f"{time.time() - t0:.1f}s", flush=True)

    with gzip.open(mg.OUT / "caps.json.gz", "wt", encoding="utf-8") as fh:
        json.dump(doc, fh, separators=(",", ":"))


if __name__ == "__main__":
    main()

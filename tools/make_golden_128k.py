"""Golden masks at the headline shape, from the REAL reference (grammask,
imported from /root/reference/pkg/src).  Run here (takes a few minutes):

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_128k.py

Writes tests/golden/k5_128k.json.gz: for synth_vocab(128256) (REF
synthvocab.py:63-154) and each of JSON (config 3), the function-call schema
(config 2), XML_TOY / ARITHMETIC forced to >= 32 nested parentheses / the
SQL-like grammar (config 4), 32 trajectories x up to 48 steps; plus 16
seeded schema mutations (config 5, tools/bench_config5.py:mutate_schema) x 2
trajectories.  Per step: the first 16 hex digits of sha256 over the
reference's u32 mask words (REF matcher.py:78-79) and the allowed count.
EOS is never sampled (trajectories stay long); half of the trajectories
prefer short structural tokens (tools/make_golden.py:structured_pick).
tests/test_gpu_golden_128k.py replays them through the batched K5 step and
the native decode loop at batch 32.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import random
import sys
import time
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, str(Path(__file__).resolve().parent))

import make_golden as mg  # noqa: E402  (puts the reference on sys.path)
from grammask.bundle import compile_bundle  # noqa: E402
from grammask.grammars import ARITHMETIC, JSON_ECMA404, SAMPLE_SCHEMA, XML_TOY  # noqa: E402
from grammask.matcher import Matcher  # noqa: E402
from grammask.schema import schema_to_grammar_text  # noqa: E402
from grammask.synthvocab import synth_vocab  # noqa: E402

SQL = (Path(__file__).resolve().parent.parent / "paper_2411_15100_b200" / "grammars" / "sql.gbnf").read_text()
STEPS = 48


def mutate_schema(seed: int) -> dict:
    # same generator as tools/bench_config5.py (kept in sync by a CPU test)
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from bench_config5 import mutate_schema as ms

    return ms(seed)


def trajectories(bundle, vocab, n_traj, seed, open_paren=0):
    rng = random.Random(seed)
    out = []
    paren = [t for t in range(vocab.size) if vocab.tokens[t][:1] == b"(" and t not in vocab.special_tokens]
    for k in range(n_traj):
        m = Matcher(bundle, vocab, history_window=1)
        bias = 0.7 if k % 2 else 0.0
        toks, masks = [], []
        for step in range(STEPS):
            mask = m.next_token_mask()
            raw = mask.to_bytes()
            masks.append([hashlib.sha256(raw).hexdigest()[:16], mask.count()])
            ids = [int(t) for t in mask.allowed_ids() if t != vocab.eos_id]
            if not ids:
                break
            if step < open_paren:
                cand = sorted(set(paren) & set(ids))
                pick = rng.choice(cand) if cand else mg.structured_pick(ids, vocab, rng, bias)
            else:
                pick = mg.structured_pick(ids, vocab, rng, bias)
            toks.append(pick)
            assert m.accept_token(pick)
        out.append({"tokens": toks, "masks": masks})
    return out


def main():
    t0 = time.time()
    vocab = synth_vocab(128256)
    doc = {"vocab": "128256:text", "grammars": {}, "schemas": []}
    plan = [
        ("json", JSON_ECMA404, 0),
        ("schema", schema_to_grammar_text(SAMPLE_SCHEMA), 0),
        ("xml", XML_TOY, 0),
        ("arithmetic", ARITHMETIC, 34),
        ("sql", SQL, 0),
    ]
    for name, text, open_paren in plan:
        b = compile_bundle(text, vocab)
        trajs = trajectories(b, vocab, 32, seed=sum(name.encode()), open_paren=open_paren)
        doc["grammars"][name] = {"text": text, "trajectories": trajs}
        print(name, f"{time.time() - t0:.1f}s", sum(len(t["masks"]) for t in trajs), "masks", flush=True)
    for i in range(16):
        sch = mutate_schema(5000 + i)
        text = schema_to_grammar_text(json.dumps(sch))
        b = compile_bundle(text, vocab)
        doc["schemas"].append({"schema": sch, "trajectories": trajectories(b, vocab, 2, seed=7000 + i)})
        print("schema", i, f"{time.time() - t0:.1f}s", flush=True)
    with gzip.open(mg.OUT / "k5_128k.json.gz", "wt", encoding="utf-8") as fh:
        json.dump(doc, fh, separators=(",", ":"))
    print("done", f"{time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()

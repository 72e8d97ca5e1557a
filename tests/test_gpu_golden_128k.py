"""K5 at the headline shape, pinned to the REAL reference: masks that
grammask produced at synth_vocab(128256) (tests/golden/k5_128k.json.gz,
tools/make_golden_128k.py) replayed through the fused decode step (K5:
accept + fill [+ apply], gm_step_tokens) at batch 32, through the native
decode loop (gm_decoder_*, token ids in the launch parameters) with logits,
and for 16 distinct mutated schemas in ONE batch (config 5).  Every mask of
every step is compared: first 16 hex digits of sha256 over the u32 words
(REF matcher.py:78-79) and the allowed count."""

import gzip
import hashlib
import json
from functools import lru_cache

import numpy as np
import pytest

from workloads import GOLDEN, vocab_by_name

pytestmark = pytest.mark.gpu


@lru_cache(maxsize=None)
def fixture():
    with gzip.open(GOLDEN / "k5_128k.json.gz", "rt", encoding="utf-8") as fh:
        return json.load(fh)


def digest(row: np.ndarray):
    raw = row.astype(np.int32).view(np.uint32).tobytes()
    return hashlib.sha256(raw).hexdigest()[:16], int(np.unpackbits(row.view(np.uint8)).sum())


def replay_k5(compiled_per_req, trajs, logits=False):
    """Batched K5 over requests with their own compiled grammar; returns the
    number of masks compared."""
    import torch

    import paper_2411_15100_b200 as gm

    vocab = vocab_by_name(fixture()["vocab"])
    B = len(trajs)
    ms = [gm.GrammarMatcher(c) for c in compiled_per_req]
    batch = gm.BatchGrammarMatcher()
    bm = gm.allocate_token_bitmask(B, vocab.size)
    lg = torch.zeros(B, vocab.size, dtype=torch.bfloat16, device="cuda") if logits else None
    checked = 0
    for s in range(max(len(t["masks"]) for t in trajs)):
        act = [k for k, t in enumerate(trajs) if s < len(t["masks"])]
        if not act:
            break
        sub = [ms[k] for k in act]
        toks = None if s == 0 else [trajs[k]["tokens"][s - 1] for k in act]
        if lg is not None:
            lg.zero_()
        flags = batch.batch_step(sub, toks, bitmask=bm, logits=lg[: len(act)] if lg is not None else None)
        if flags is not None:
            assert (flags.cpu().numpy() == 1).all(), ("accept", s)
        rows = bm[: len(act)].cpu().numpy()
        for j, k in enumerate(act):
            want = trajs[k]["masks"][s]
            assert list(digest(rows[j])) == want, ("mask", k, s)
            checked += 1
        if lg is not None:
            allowed = np.unpackbits(rows.view(np.uint8), axis=1, bitorder="little")[:, : vocab.size].astype(bool)
            got = lg[: len(act)].view(torch.int16).cpu().numpy()
            assert (got[allowed] == 0).all() and (got[~allowed] == np.int16(-128)).all(), ("apply", s)
    return checked


@pytest.mark.parametrize("grammar", ["json", "schema", "xml", "arithmetic", "sql"])
def test_k5_batch32_matches_reference(grammar):
    import paper_2411_15100_b200 as gm

    fx = fixture()
    vocab = vocab_by_name(fx["vocab"])
    info = gm.TokenizerInfo.from_vocabulary(vocab)
    compiled = gm.GrammarCompiler(info).compile_grammar(fx["grammars"][grammar]["text"])
    trajs = fx["grammars"][grammar]["trajectories"]
    assert len(trajs) == 32
    # the fused apply's per-key mixed-chunk policy: SQL's identifier-class
    # rows are applied blended, so the logits check below covers that path
    if grammar == "sql":
        assert compiled._dev.cache.stats["blend_keys"] > 0
    n = replay_k5([compiled] * len(trajs), trajs, logits=grammar in ("json", "sql"))
    assert n == sum(len(t["masks"]) for t in trajs)


def test_k5_sql_fused_apply_policy_off():
    """The fused apply's per-key policy follows gm_apply_set_blend at cache
    build: with the policy off no SQL key is blended and the element-store
    apply of the same golden trajectories is exact too."""
    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200 import _lib

    fx = fixture()
    vocab = vocab_by_name(fx["vocab"])
    lib = _lib.load()
    old = lib.gm_apply_set_blend(0)
    try:
        compiled = gm.GrammarCompiler(gm.TokenizerInfo.from_vocabulary(vocab)).compile_grammar(
            fx["grammars"]["sql"]["text"])
    finally:
        lib.gm_apply_set_blend(old)
    assert compiled._dev.cache.stats["blend_keys"] == 0
    trajs = fx["grammars"]["sql"]["trajectories"]
    n = replay_k5([compiled] * len(trajs), trajs, logits=True)
    assert n == sum(len(t["masks"]) for t in trajs)


def test_k5_config5_distinct_schemas_one_batch():
    """Config 5: 16 mutated schemas x 2 trajectories, each request with its
    own compiled grammar, one K5 launch per step."""
    import paper_2411_15100_b200 as gm

    fx = fixture()
    vocab = vocab_by_name(fx["vocab"])
    comp = gm.GrammarCompiler(gm.TokenizerInfo.from_vocabulary(vocab))
    per_req, trajs = [], []
    for sc in fx["schemas"]:
        c = comp.compile_json_schema(json.dumps(sc["schema"]))
        for t in sc["trajectories"]:
            per_req.append(c)
            trajs.append(t)
    assert len(trajs) == 32
    n = replay_k5(per_req, trajs, logits=True)
    assert n == sum(len(t["masks"]) for t in trajs)


@pytest.mark.parametrize("grammar", ["json", "arithmetic"])
def test_decode_loop_batch32_matches_reference(grammar):
    """The native decode loop (host token ids in, flags out) over the same
    trajectories: masks after every step equal the reference's."""
    import torch

    import paper_2411_15100_b200 as gm
    from paper_2411_15100_b200.graph import DecodeLoop

    fx = fixture()
    vocab = vocab_by_name(fx["vocab"])
    compiled = gm.GrammarCompiler(gm.TokenizerInfo.from_vocabulary(vocab)).compile_grammar(
        fx["grammars"][grammar]["text"])
    trajs = fx["grammars"][grammar]["trajectories"]
    steps = min(len(t["masks"]) for t in trajs)
    B = len(trajs)
    ms = [gm.GrammarMatcher(compiled) for _ in range(B)]
    bms = [gm.allocate_token_bitmask(B, vocab.size) for _ in range(2)]
    lgs = [torch.zeros(B, vocab.size, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    loop = DecodeLoop(ms, bms, lgs, recycle=False)
    for s in range(steps):
        i = s % 2
        loop.step(None if s == 0 else np.asarray([t["tokens"][s - 1] for t in trajs], np.int32), i)
        flags = loop.flags(i)
        if s:
            assert (flags == 1).all()
        rows = bms[i].cpu().numpy()
        for k in range(B):
            assert list(digest(rows[k])) == trajs[k]["masks"][s], (grammar, k, s)
    loop.close()

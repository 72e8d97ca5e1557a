"""GMB1 / GMC1 files: the reader/writer against bundles
written by the real reference (tests/golden/bundles, made by
tools/make_golden_bundles.py), and — on the GPU — loading them into the
engine and exporting bundles from it."""

import hashlib
import json

import numpy as np
import pytest

from paper_2411_15100_b200 import bundle_io as bio
from workloads import GOLDEN, grammar_text, load_fixture, vocab_by_name

BUNDLES = GOLDEN / "bundles"
META = json.loads((BUNDLES / "bundles.json").read_text())


@pytest.mark.parametrize("tag", sorted(META))
def test_reference_bundles_round_trip(tag):
    """read -> write reproduces the reference's bytes (REF docs/formats.md:
    'Re-serializing ... is byte-identical'); header and section facts match."""
    raw = (BUNDLES / f"{tag}.gmb").read_bytes()
    m = META[tag]
    b = bio.read_bundle(raw)
    assert bio.write_bundle(b) == raw
    assert hashlib.sha256(raw).hexdigest() == m["sha256"]
    assert b.flags == m["flags"] and b.grammar_text == m["grammar_text"] and b.vocab_hash.hex() == m["vocab_hash"]
    assert (b.pda.node_count, len(b.pda.edges), len(b.pda.rules), b.pda.root) == (
        m["pda"]["nodes"], m["pda"]["edges"], m["pda"]["rules"], m["pda"]["root"])
    if m["cache_entries"]:
        assert len(b.cache.entries) == m["cache_entries"]
        assert hashlib.sha256(bio.write_cache(b.cache)).hexdigest() == m["cache_sha256"]
    else:
        assert b.cache is None


@pytest.mark.parametrize("tag", [t for t in sorted(META) if META[t]["cache_entries"]])
def test_reference_cache_entries_partition_and_storage(tag):
    """Every GMC1 entry partitions the non-special vocabulary, and the
    adaptive encoding chosen by choose_storage is the reference's."""
    b = bio.read_bundle((BUNDLES / f"{tag}.gmb").read_bytes())
    vocab = vocab_by_name(META[tag]["vocab"])
    universe = np.asarray([i for i in range(vocab.size) if i not in vocab.special_tokens], dtype=np.uint32)
    for node, e in b.cache.entries.items():
        dep = e.dependent
        if e.variant == bio.ACCEPT_HEAVY:
            rej = e.ids
            acc = np.setdiff1d(universe, np.concatenate([rej, dep]))
        elif e.variant == bio.REJECT_HEAVY:
            acc = e.ids
            rej = np.setdiff1d(universe, np.concatenate([acc, dep]))
        else:
            acc = np.nonzero(np.unpackbits(e.bits.view(np.uint8), bitorder="little")[:vocab.size])[0]
            rej = np.setdiff1d(universe, np.concatenate([acc, dep]))
        parts = np.concatenate([acc, rej, dep])
        assert len(parts) == len(universe) and np.array_equal(np.sort(parts), universe), (tag, node)
        again = bio.choose_storage(acc, rej, dep, vocab.size)
        assert again.variant == e.variant, (tag, node)


def test_reader_rejects_bad_files():
    raw = (BUNDLES / "json_toy200.gmb").read_bytes()
    with pytest.raises(ValueError, match="not a grammask bundle"):
        bio.read_bundle(b"XXXX" + raw[4:])
    with pytest.raises(ValueError, match="unsupported bundle version"):
        bio.read_bundle(raw[:4] + (2).to_bytes(4, "little") + raw[8:])
    with pytest.raises(ValueError, match="truncated"):
        bio.read_bundle(raw[:100])
    with pytest.raises(ValueError, match="not a mask cache blob"):
        bio.read_cache(b"GMB1" + raw[4:])


def _replay(bundle, vocab, fname):
    from paper_2411_15100_b200.compat import Matcher

    fx = load_fixture(fname)
    checked = 0
    for traj in fx["trajectories"][:6]:
        m = Matcher(bundle, vocab, history_window=1)
        toks = traj["tokens"]
        for step, rec in enumerate(traj["masks"]):
            raw = m.next_token_mask().to_bytes()
            assert hashlib.sha256(raw).hexdigest() == rec["sha256"], (fname, step)
            checked += 1
            if step >= len(toks):
                break
            assert m.accept_token(toks[step])
            if toks[step] == vocab.eos_id:
                break
        m.close()
    assert checked > 0


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["json_toy200", "schema_toy200", "arithmetic_gen", "xml_gen", "json_toy200_cache0",
                                 "json_gen_inline0_merge0"])
def test_load_reference_bundle_on_device(tag):
    """compat.load_bundle(reference bytes) -> masks == the reference's golden
    masks for that grammar and vocabulary; save_bundle gives the bytes back."""
    from paper_2411_15100_b200.compat import Matcher, MatcherError, load_bundle, save_bundle

    raw = (BUNDLES / f"{tag}.gmb").read_bytes()
    m = META[tag]
    vocab = vocab_by_name(m["vocab"])
    bundle = load_bundle(raw)
    with pytest.raises(MatcherError, match="does not match"):
        Matcher(bundle, vocab_by_name("gen" if m["vocab"] == "toy200" else "toy200"))
    _replay(bundle, vocab, f"masks_{m['grammar']}_{m['vocab']}.json.gz")
    assert save_bundle(bundle) == raw


@pytest.mark.gpu
@pytest.mark.parametrize("gname,vname", [("json", "toy200"), ("arithmetic", "gen"), ("schema", "toy200")])
def test_export_bundle_round_trip(gname, vname):
    """A bundle compiled here exports to GMB1 (this engine's automaton + its
    cache as GMC1); the file parses, its cache entries agree with the device
    cache, it is deterministic, and loading it reproduces the golden masks."""
    from paper_2411_15100_b200.compat import compile_bundle, load_bundle, save_bundle

    vocab = vocab_by_name(vname)
    b = compile_bundle(grammar_text(gname), vocab)
    raw = save_bundle(b)
    assert save_bundle(b) == raw
    img = bio.read_bundle(raw)
    assert bio.write_bundle(img) == raw
    t = b.compiled.tables
    assert img.pda.node_count == t.n_nodes and len(img.pda.rules) == t.n_rules
    assert sorted(img.cache.entries) == sorted(int(k) for k in t.cache_keys)
    _replay(load_bundle(raw), vocab, f"masks_{gname}_{vname}.json.gz")

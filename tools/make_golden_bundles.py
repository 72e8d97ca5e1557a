"""Golden GMB1/GMC1 artefacts from the real reference (run HERE only — it
imports grammask from /root/reference; the outputs are committed under
tests/golden/bundles/ and nothing at test time reads /root/reference).

For each (grammar, vocabulary, options) the reference's compile_bundle +
save_bundle bytes are written as <name>.gmb, plus bundles.json with the
vocabulary names, options and per-bundle facts (sizes, entry counts, the
sha256 of the GMC1 blob) the tests check the reader against.

    python tools/make_golden_bundles.py
"""

import hashlib
import json
import struct
import sys
from pathlib import Path

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

from conftest import FIVE_GRAMMARS, build_gen_vocab, build_toy200  # noqa: E402
from grammask.bundle import CompileOptions, compile_bundle, load_bundle, save_bundle  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "bundles"


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    vocabs = {"toy200": build_toy200(), "gen": build_gen_vocab()}
    plan = [
        ("json", "toy200", {}),
        ("schema", "toy200", {}),
        ("arithmetic", "gen", {}),
        ("xml", "gen", {}),
        ("array_string", "gen", {}),
        ("json", "toy200", {"cache": False}),
        ("json", "gen", {"inline": False, "merge": False}),
    ]
    meta = {}
    for gname, vname, kw in plan:
        vocab = vocabs[vname]
        b = compile_bundle(FIVE_GRAMMARS[gname], vocab, CompileOptions(**kw))
        raw = save_bundle(b)
        assert save_bundle(load_bundle(raw)) == raw
        tag = "_".join([gname, vname] + [f"{k}{int(v)}" for k, v in sorted(kw.items())])
        (OUT / f"{tag}.gmb").write_bytes(raw)
        cache_blob = b.cache.serialize() if b.cache is not None else b""
        meta[tag] = {
            "grammar": gname, "vocab": vname, "options": kw, "flags": b.options.flags,
            "bytes": len(raw), "sha256": hashlib.sha256(raw).hexdigest(),
            "grammar_text": b.grammar_text,
            "pda": {"nodes": b.pda.node_count, "edges": len(b.pda.edges), "rules": len(b.pda.rules),
                    "root": b.pda.root},
            "cache_entries": len(b.cache.entries) if b.cache is not None else 0,
            "cache_sha256": hashlib.sha256(cache_blob).hexdigest() if cache_blob else None,
            "vocab_hash": vocab.content_hash().hex(),
        }
        print(tag, len(raw), "bytes")
    (OUT / "bundles.json").write_text(json.dumps(meta, indent=1) + "\n")


if __name__ == "__main__":
    main()

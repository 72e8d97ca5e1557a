"""Load bundles EXPORTED by this engine with the real reference (build
container only: imports grammask from /root/reference) and replay the golden
trajectories through the reference's Matcher on them: the reference's masks
over our automaton + cache must equal the golden masks it produced on its own
bundles.

    python tools/check_exports_with_reference.py gpurun_out/exports
"""
import gzip
import hashlib
import json
import sys
from pathlib import Path

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
GOLDEN = Path(__file__).resolve().parent.parent / "tests" / "golden"

from conftest import build_gen_vocab, build_toy200  # noqa: E402
from grammask.bundle import load_bundle, save_bundle  # noqa: E402
from grammask.matcher import Matcher  # noqa: E402


def main(src):
    vocabs = {"toy200": build_toy200(), "gen": build_gen_vocab()}
    total_bad = 0
    for path in sorted(Path(src).glob("*.gmb")):
        g, v = path.stem.rsplit("_", 1)
        raw = path.read_bytes()
        b = load_bundle(raw)
        assert save_bundle(b) == raw, "reference re-serialisation differs"
        vocab = vocabs[v]
        with gzip.open(GOLDEN / f"masks_{g}_{v}.json.gz", "rt") as fh:
            fx = json.load(fh)
        checked = bad = 0
        for traj in fx["trajectories"]:
            m = Matcher(b, vocab, history_window=1)
            toks = traj["tokens"]
            for step, rec in enumerate(traj["masks"]):
                raw_mask = m.next_token_mask().to_bytes()
                checked += 1
                bad += hashlib.sha256(raw_mask).hexdigest() != rec["sha256"]
                if step >= len(toks):
                    break
                assert m.accept_token(toks[step])
                if toks[step] == vocab.eos_id:
                    break
        total_bad += bad
        print(f"{path.name}: reference loads it (re-serialises byte-identical); {checked} masks replayed, "
              f"{bad} differ from golden; pda nodes {b.pda.node_count}, cache entries {len(b.cache.entries)}")
    print("ALL OK" if total_bad == 0 else f"{total_bad} MISMATCHES")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/exports")

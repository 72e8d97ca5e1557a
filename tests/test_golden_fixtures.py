"""CPU checks of the golden fixtures' provenance (no GPU): the config-5
schemas recorded from the reference by tools/make_golden_128k.py are the
same seeded mutations bench / tools/bench_config5.py generate."""

import gzip
import json
import sys
from pathlib import Path

from workloads import GOLDEN

ROOT = Path(__file__).resolve().parent.parent


def test_config5_schemas_match_generator():
    sys.path.insert(0, str(ROOT / "tools"))
    from bench_config5 import mutate_schema

    with gzip.open(GOLDEN / "k5_128k.json.gz", "rt", encoding="utf-8") as fh:
        fx = json.load(fh)
    assert len(fx["schemas"]) == 16
    for i, sc in enumerate(fx["schemas"]):
        assert sc["schema"] == mutate_schema(5000 + i)
    for g in ("json", "schema", "xml", "arithmetic", "sql"):
        assert len(fx["grammars"][g]["trajectories"]) == 32


def test_caps_fixture_shape():
    with gzip.open(GOLDEN / "caps.json.gz", "rt", encoding="utf-8") as fh:
        fx = json.load(fh)
    assert max(max(t["ref_stacks"]) for t in fx["cases"]["ambig40"]["trajectories"]) == 40
    assert max(max(t["ref_stacks"]) for t in fx["cases"]["ambig300"]["trajectories"]) == 300
    assert fx["cases"]["ambig_over_cap"]["compile_error"][0] == "StateLimitError"

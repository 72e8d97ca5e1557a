"""Export GMB1 bundles compiled by this engine (GPU box) for the reference
to load (tools/check_exports_with_reference.py runs the reference on them in
the build container):

    python tools/export_bundles.py gpurun_out/exports
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

from paper_2411_15100_b200.compat import compile_bundle, save_bundle  # noqa: E402
from workloads import grammar_text, vocab_by_name  # noqa: E402

PLAN = [("json", "toy200"), ("schema", "toy200"), ("arithmetic", "gen"), ("xml", "gen"), ("array_string", "gen")]


def main(out_dir):
    os.makedirs(out_dir, exist_ok=True)
    for g, v in PLAN:
        raw = save_bundle(compile_bundle(grammar_text(g), vocab_by_name(v)))
        with open(os.path.join(out_dir, f"{g}_{v}.gmb"), "wb") as fh:
            fh.write(raw)
        print(g, v, len(raw), "bytes")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/exports")

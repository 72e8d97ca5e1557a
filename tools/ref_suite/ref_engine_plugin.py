"""pytest plugin: the reference's OWN test files (an unmodified copy of
REF pkg/tests in baseline/_ref/tests, next to the reference install) run
against this engine — SURVEY §8b's drop-in claim, checked on the reference's
files instead of restatements.

The engine entry points of grammask are replaced by this engine's
(paper_2411_15100_b200.compat): compile_bundle / Matcher / MatcherError /
TokenMask.  Everything the tests use as their oracle — grammar parsing, the
PDA and its brute-force oracle (REF pda.py:547-594), schemas, vocabularies —
stays the reference's own; a compiled bundle carries the reference's PDA as
`.pda` for those oracle checks, while every mask, accept, rollback and branch
comes from the GPU.

Deselected (with the reason printed): tests of the reference's internal
state (its StackArena counters, its NFA stack count, its cache statistics,
its CPU timings), which this engine does not have.

    python -m pytest -p tools.ref_suite.ref_engine_plugin baseline/_ref/tests/test_matcher.py ...
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = os.path.join(ROOT, "baseline", "_ref")
for p in (REF, os.path.join(REF, "tests"), ROOT):
    if p not in sys.path:
        sys.path.insert(0, p)

import grammask  # noqa: E402  (the reference, from baseline/_ref)
import grammask.bundle as _rb  # noqa: E402
import grammask.matcher as _rm  # noqa: E402

from paper_2411_15100_b200 import compat  # noqa: E402
from paper_2411_15100_b200.vocab import vocab_from_tokens as _our_vocab_from_tokens  # noqa: E402

_REAL_COMPILE = _rb.compile_bundle
_VOCABS: dict = {}

INTERNAL = {
    "test_parallel_stack_count_on_raw_bundle": "counts the reference's NFA stacks (m._tops); this engine's automaton "
                                               "is determinised, stack counts are not a parity target (SURVEY §0.4)",
    "test_branch_cost_independent_of_depth": "reads the reference's StackArena (m._arena)",
    "test_arena_bounded_by_window": "reads the reference's StackArena counters (m._arena)",
    "test_arena_reclaims_rejected_work": "reads the reference's StackArena counters (m._arena)",
    "test_classification_statistics": "the reference's cache statistics (structure-dependent, not a parity target)",
    "test_adaptive_storage": "the reference's cache encoding sizes",
    "test_prefix_sharing": "the reference's sweep instrumentation",
    "test_ablation_ordering": "CPU timing thresholds of the reference's ablation ladder",
    "test_overlap_simulation": "CPU timing of the reference's overlap simulation",
    "test_dependent_sweep_threshold_equivalence": "the reference's CPU dependent-sweep threshold knob",
    "test_ablation_ladder_runs_and_verifies_masks": "its report rows read the reference's cache object (bytes, "
                                                    "dependent counts before/after context expansion)",
    "test_measured_counts_deterministic": "the reference's cache statistics in the bench report",
}


def _ours(v):
    """This engine's Vocabulary for a reference Vocabulary (same tokens,
    specials and EOS, hence the same content hash)."""
    key = id(v)
    hit = _VOCABS.get(key)
    if hit is None or hit[0] is not v:
        ov = _our_vocab_from_tokens(list(v.tokens), eos_id=v.eos_id, special=sorted(v.special_tokens))
        assert ov.content_hash() == v.content_hash()
        hit = _VOCABS[key] = (v, ov)
    return hit[1]


def compile_bundle(grammar_text, vocab, options=None):
    o = options or _rb.CompileOptions()
    ours = compat.compile_bundle(grammar_text, _ours(vocab),
                                 compat.CompileOptions(inline=o.inline, merge=o.merge, cache=o.cache,
                                                       ctx_expansion=o.ctx_expansion))
    # the oracle side of the tests: the reference's PDA for the same text
    ref = _REAL_COMPILE(grammar_text, vocab, _rb.CompileOptions(inline=o.inline, merge=o.merge, cache=False))
    ours.pda = ref.pda
    ours.options = o
    return ours


class Matcher(compat.Matcher):
    def __init__(self, bundle, vocab, history_window=32, **kw):
        super().__init__(bundle, _ours(vocab), history_window, **kw)

    @property
    def tops_count(self):
        return self.stack_count()


for mod in (_rb, grammask):
    mod.compile_bundle = compile_bundle
for mod in (_rm, grammask):
    mod.Matcher = Matcher
    mod.MatcherError = compat.MatcherError
    mod.TokenMask = compat.TokenMask


def pytest_collection_modifyitems(config, items):
    keep, drop = [], []
    for it in items:
        (drop if it.originalname in INTERNAL or it.name in INTERNAL else keep).append(it)
    if drop:
        config.hook.pytest_deselected(items=drop)
        items[:] = keep
        for it in drop:
            name = it.originalname or it.name
            print(f"deselected {it.nodeid}: {INTERNAL[name]}")

"""The reference's OWN test files against this engine (the
reference tests run unchanged except for the engine): test_matcher.py,
test_acceptance.py and test_bench.py from an unmodified copy of REF
pkg/tests next to the reference install (baseline/_ref/tests), with
grammask's compile_bundle / Matcher / MatcherError / TokenMask replaced by
this engine's through tools/ref_suite/ref_engine_plugin.py (tests of the
reference's internal state are deselected there, each with its reason).
Skipped when the reference copy is absent."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "tests")


@pytest.mark.skipif(not os.path.isfile(os.path.join(REF_TESTS, "test_matcher.py")),
                    reason="reference test files not installed in baseline/_ref/tests")
def test_reference_suite_against_engine():
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""))
    res = subprocess.run([sys.executable, "-m", "pytest", "-p", "tools.ref_suite.ref_engine_plugin",
                          "test_matcher.py", "test_acceptance.py", "test_bench.py", "-q", "-p", "no:cacheprovider"],
                         cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=1500)
    tail = res.stdout[-3000:]
    assert res.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail, tail

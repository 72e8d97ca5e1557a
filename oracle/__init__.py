"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain-Python restatement of the reference (grammask,
/root/reference/pkg/src/grammask) algorithm for the token-mask hot path:
Thompson PDA construction, node merging and rule inlining, the sorted-sweep
adaptive cache with context expansion, and the runtime matcher (closure,
Algorithm-1 fill with dependent resolution, accept, rollback).  Every
function cites the reference file:line it restates.

Who may use it: tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg — as the checker or the timed CPU baseline, never as
part of the product path (paper_2411_15100_b200 never imports it).

Pinning: the oracle is checked against golden vectors produced by the real
reference (tests/golden, tools/make_golden.py) in tests/test_oracle.py.

Shared piece: grammar *parsing* reuses the product's pure-Python parser
(paper_2411_15100_b200/grammar.py), whose surface semantics are pinned
independently against the reference by golden/languages.json (accept
verdicts and error messages).  Everything from the automaton on is
independent of the product.
"""

from .pda import OraclePda, build_oracle_pda
from .cache import OracleCache, build_oracle_cache
from .matcher import OracleMatcher, OracleBundle, compile_oracle_bundle, brute_force_mask

__all__ = [
    "OraclePda",
    "build_oracle_pda",
    "OracleCache",
    "build_oracle_cache",
    "OracleMatcher",
    "OracleBundle",
    "compile_oracle_bundle",
    "brute_force_mask",
]

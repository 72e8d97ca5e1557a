"""Add the SQL-like grammar of SURVEY §8(d) config 4 to tests/golden, from the
REAL reference (grammask, imported from /root/reference/pkg/src).  Run here:

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_sql.py

Adds "sql" to languages.json (grammar text + oracle_accepts verdicts for
probe strings) and writes masks_sql_toy200.json.gz (full masks) and
masks_sql_32000_text.json.gz (sha256 + popcount), with the trajectory
sampler of tools/make_golden.py.  The golden suites (CPU oracle, front end,
GPU parity) pick them up through tests/workloads.py.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, str(Path(__file__).resolve().parent))

import make_golden as mg  # noqa: E402  (puts the reference on sys.path)
from grammask.bundle import compile_bundle  # noqa: E402
from grammask.grammar import parse_grammar  # noqa: E402
from grammask.pda import build_pda, oracle_accepts  # noqa: E402
from grammask.synthvocab import synth_vocab  # noqa: E402

SQL = (Path(__file__).resolve().parent.parent / "paper_2411_15100_b200" / "grammars" / "sql.gbnf").read_text()

PROBES = [
    b"SELECT * FROM t;", b"SELECT a FROM t WHERE a = 1;", b"SELECT a,b FROM t ORDER BY a DESC, b LIMIT 5 ;",
    b"SELECT COUNT(*) AS n FROM t x LEFT JOIN u y ON x.id = y.id WHERE NOT (a > 1 OR b IS NOT NULL);",
    b"SELECT a FROM (SELECT b FROM c) d WHERE e IN (SELECT f FROM g) GROUP BY a;",
    b"SELECT a + 2 * (b - 1) FROM t WHERE s <> 'x y' AND k IN (1, -2.5, NULL);",
    b"SELECT FROM t;", b"SELECT * FROM;", b"select * from t;", b"SELECT * FROM t", b"SELECT a FROM t WHERE;",
    b"SELECT a FROM t WHERE a IS NULL NULL;", b"SELECT 'unterminated FROM t;",
]


def main():
    p = build_pda(parse_grammar(SQL))
    lang_path = mg.OUT / "languages.json"
    lang = json.loads(lang_path.read_text())
    lang["grammars"]["sql"] = SQL
    lang["accepts"] = [a for a in lang["accepts"] if a[0] != "sql"]
    alpha = list(b"SELCTFROMWHEANDIBYJ *(),;=<>'.-+0123456789abxyz_\n")
    rng = random.Random(17)
    probes = set(PROBES)
    for s in PROBES:  # prefixes and one-byte edits of the probes
        for k in range(0, len(s) + 1, 3):
            probes.add(s[:k])
        for _ in range(6):
            i = rng.randrange(len(s))
            probes.add(s[:i] + bytes([rng.choice(alpha)]) + s[i + 1:])
    for _ in range(200):
        probes.add(bytes(rng.choice(alpha) for _ in range(rng.randrange(1, 10))))
    for s in sorted(probes):
        lang["accepts"].append(["sql", s.hex(), oracle_accepts(p, s)])
    lang_path.write_text(json.dumps(lang, indent=0) + "\n")

    toy = mg.build_toy200()
    b = compile_bundle(SQL, toy)
    trajs = []
    for bias in (0.0, 0.7):
        trajs += mg.trajectories(b, toy, 12, 40, seed=31 + int(bias * 10), bias=bias, full=True)
    mg.write_gz("masks_sql_toy200.json.gz", {"grammar": "sql", "vocab": "toy200", "trajectories": trajs})
    vocab = synth_vocab(32000, profile="text")
    b = compile_bundle(SQL, vocab)
    trajs = []
    for i, bias in enumerate((0.0, 0.7)):
        trajs += mg.trajectories(b, vocab, 2, 60, seed=2000 + i, bias=bias, full=False)
    mg.write_gz("masks_sql_32000_text.json.gz",
                {"grammar": "sql", "vocab": "32000:text", "trajectories": trajs,
                 "ref_stats": {"entries": b.cache.stats.entry_count,
                               "dependent_total": b.cache.stats.dependent_total}})
    print("sql fixtures written", sum(1 for a in lang["accepts"] if a[0] == "sql"), "probes")


if __name__ == "__main__":
    main()

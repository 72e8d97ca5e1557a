"""Summarise an A/B run of library variants (run_e-style): bench value/e2e and
ncu median kernel durations per variant.  Usage: python tools/ab_summary.py libA.so libB.so ..."""
import collections
import csv
import json
import statistics
import sys

for lib in sys.argv[1:]:
    rows = list(csv.DictReader(l for l in open(f"gpurun_out/ncu_{lib}.csv") if not l.startswith("==")))
    d = collections.defaultdict(list)
    for r in rows:
        d[r["Kernel Name"][:22]].append(float(r["Metric Value"]))
    b = json.loads(open(f"gpurun_out/ab_{lib}_1.json").read())
    print(lib, round(b["value"], 2), round(b["e2e"]["value"], 2),
          {k: round(statistics.median(v) / 1000, 2) for k, v in d.items()})

#!/usr/bin/env bash
# A/B of library variants on the bench value (K5 b2b) pass, run on a GPU box:
#   bash tools/ab_libs.sh "json xml" tools/variants/libA.so tools/variants/libB.so ...
# prints grammar, library, value (us/step), e2e for each, alternating variants twice.
G=${1:-json}; shift
export GMASK_NO_BUILD=1
for rep in 1 2; do
  for g in $G; do
    for lib in "$@"; do
      out=$(GMASK_LIB=$lib timeout 300 python bench.py --grammar $g --no-cpu-baseline --repeats 5 2>/dev/null | tail -1)
      python -c "import json,sys; d=json.loads(sys.argv[1]); print('$g', '$(basename $lib)', round(d['value'],3), round(d['e2e']['value'],3))" "$out"
    done
  done
done

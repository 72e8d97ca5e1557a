#!/usr/bin/env bash
# SURVEY §8d configs 2 and 4 through the same bench step (1 GPU), one JSON
# line each into gpurun_out/configs_<tag>.jsonl:
#   bash tools/bench_configs.sh r01
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
OUT=gpurun_out/configs_${TAG}.jsonl
: > $OUT
for spec in "schema 64" "xml 128" "arithmetic 128" "json 128"; do
  set -- $spec
  timeout 900 python bench.py --grammar $1 --batch $2 --steps 100 --warmup 5 --cpu-budget-s 20 \
      >> $OUT 2> gpurun_out/configs_${TAG}_$1.err || echo "{\"grammar\": \"$1\", \"failed\": true}" >> $OUT
done
cat $OUT | cut -c1-400

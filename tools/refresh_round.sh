#!/usr/bin/env bash
# Round-end refresh on a GPU box (1 GPU): default bench line, the other
# configs, config 5, ncu launch list + --set full captures.
#   bash tools/refresh_round.sh r01
set -u
TAG=${1:-r01}
export GMASK_NO_BUILD=1
mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
: > gpurun_out/${TAG}_configs.jsonl
timeout 300 python bench.py --grammar schema --batch 64 2>/dev/null | tail -1 >> gpurun_out/${TAG}_configs.jsonl
for g in xml arithmetic sql json; do
  timeout 300 python bench.py --grammar $g 2>/dev/null | tail -1 >> gpurun_out/${TAG}_configs.jsonl
done
timeout 400 python tools/bench_config5.py --out gpurun_out/${TAG}_config5.json > gpurun_out/${TAG}_config5.log 2>&1
bash tools/profile_round.sh $TAG

#!/usr/bin/env bash
# Profile the bench workload on a GPU box (run under gpurun, 1 GPU):
#   bash tools/profile_round.sh r01
# writes gpurun_out/<tag>_launches.csv (every launch, cold-cache serialised
# durations) and gpurun_out/<tag>_<kernel>.ncu-rep (--set full) for the hot
# kernels; tools/summarize_profiles.py turns them into profiles/<tag>_*.
set -u
TAG=${1:-r01}
export GMASK_NO_BUILD=1
mkdir -p gpurun_out
CMD="python bench.py --steps 8 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"gm::|apply_tile" --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > /dev/null 2>&1
for k in "fill_kernel<true>" "fill_kernel<false>" apply_tile_kernel accept_tokens_kernel cache_build_kernel; do
  safe=$(echo "$k" | tr '<>' '__')
  ncu --set full --import-source on --clock-control none -k regex:"$k" -s 4 -c 1 \
      -o gpurun_out/${TAG}_${safe} $CMD > /dev/null 2>&1
done
ls -la gpurun_out | grep "$TAG"

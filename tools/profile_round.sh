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
    -k regex:"fill_kernel|apply_tile|accept_tokens|recycle|cache_build|dep_compact|row_popcount" --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > /dev/null 2>&1
# bench launch order: pass A = K3 fill_kernel<true> x (warmup+steps), then
# pass B = K2 fill_kernel<false> + K0 apply, then pass C; compile = 4 K1 launches
cap() {  # name regex skip tag
  ncu --set full --import-source on --clock-control none -k regex:"$1" -s "$2" -c 1 \
      -o gpurun_out/${TAG}_$3 $CMD > /dev/null 2>&1
}
cap fill_kernel 6 k3_fused_fill_apply
cap fill_kernel 17 k2_fill
cap apply_tile_kernel 4 k0_apply
cap accept_tokens_kernel 4 k4_accept
cap cache_build_kernel 1 k1_cache_build
ls -la gpurun_out | grep "$TAG"

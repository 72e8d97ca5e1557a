#!/usr/bin/env bash
# Profile the hot-path kernels on a GPU box (run under gpurun, 1 GPU):
#   bash tools/profile_round.sh r01
# writes gpurun_out/<tag>_launches.csv (every launch of the bench command:
# gpu__time_duration + DRAM bytes, cold-cache serialised) and
# gpurun_out/<tag>_<kernel>.ncu-rep (--set full, one launch each) for
#   k5_step            fill_kernel<true,true>  (the `value` kernel: accept + fill + apply)
#   k3_fused_fill_apply fill_kernel<true,false> (fill + apply)
#   k2_fill            fill_kernel<false,false>
#   k0_apply           apply_tile_kernel<2>    (bf16 apply)
#   k4_accept          accept_tokens_kernel
#   k1_cache_build     cache_build_kernel
# The --set full captures use tools/step_driver.py (plain eager decode loop
# of the bench workload, fixed launch order) so the -s skip counts are
# stable; tools/summarize_profiles.py turns everything into profiles/<tag>_*.
set -u
TAG=${1:-r01}
export GMASK_NO_BUILD=1
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"fill_kernel|step_ptok|apply_tile|accept_tokens|recycle|cache_build|dep_" --csv \
    --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 8 --warmup 3 --repeats 1 --no-cpu-baseline > /dev/null 2>&1
cap() {  # kernel-regex skip tag driver-mode
  ncu --set full --import-source on --clock-control none -k regex:"$1" -s "$2" -c 1 \
      -o gpurun_out/${TAG}_$3 python tools/step_driver.py --mode "$4" --steps 16 > /dev/null 2>&1
}
cap "fill_kernel" 10 k5_step k5
cap "fill_kernel" 10 k3_fused_fill_apply k4k3
cap "fill_kernel" 10 k2_fill k2k0
cap "apply_tile_kernel" 10 k0_apply k2k0
cap "accept_tokens_kernel" 10 k4_accept k4k3
cap "cache_build_kernel" 0 k1_cache_build k2k0
ls -la gpurun_out | grep "$TAG"

mkdir -p gpurun_out
for k in fill_kernel apply_tile_kernel accept_tokens_kernel cache_build_kernel; do
  ncu --set full --import-source on --clock-control none -k regex:$k -s 6 -c 1 -o gpurun_out/prof_$k python bench.py --steps 12 --warmup 3 --no-cpu-baseline > /dev/null 2>gpurun_out/ncu_$k.err
done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gm::" --csv --log-file gpurun_out/launches2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out

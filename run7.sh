python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-flush > gpurun_out/bench_warm.json 2>gpurun_out/bench_warm.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench_warm.json'))
for k in ['value','fill_us','apply_us','accept_us']: print('warm', k, d.get(k))
PY
ncu --set full --cache-control none --clock-control none -k regex:fill_kernel -s 6 -c 1 -o gpurun_out/prof_fill_warm python bench.py --steps 12 --warmup 3 --no-cpu-baseline --no-flush > /dev/null 2>&1
ncu --set full --cache-control all --clock-control none -k regex:fill_kernel -s 6 -c 1 -o gpurun_out/prof_fill_cold python bench.py --steps 12 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --cache-control all --clock-control none -k regex:accept_tokens -s 6 -c 1 -o gpurun_out/prof_acc_cold python bench.py --steps 12 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --cache-control all --clock-control none -k regex:apply_tile -s 6 -c 1 -o gpurun_out/prof_apply_cold python bench.py --steps 12 --warmup 3 --no-cpu-baseline > /dev/null 2>&1

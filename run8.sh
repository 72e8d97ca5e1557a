python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench8.json 2>gpurun_out/bench8.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench8.json'))
for k in ['value','fill_us','apply_us','accept_us','e2e']: print(k, d.get(k))
PY
ncu --set full --clock-control none -k regex:accept_tokens -s 6 -c 1 -o gpurun_out/prof_acc8 python bench.py --steps 12 --warmup 3 --no-cpu-baseline > /dev/null 2>&1

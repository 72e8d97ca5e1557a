export GMASK_NO_BUILD=1
python -m pytest tests -x -q -m gpu 2>&1 | tail -2
python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench20.json 2>gpurun_out/bench20.err; tail -3 gpurun_out/bench20.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench20.json'))
for k in ['value','separate_fill_then_apply_us','fill_us','apply_us','accept_us','e2e','roofline','masked_fraction']: print(k, d.get(k))
PY

export GMASK_NO_BUILD=1
for i in 1 2; do python -m pytest tests -x -q -m gpu 2>&1 | tail -2; done
GMASK_TRACE=1 python tools/trace_step.py 2>&1 | tail -8
python bench.py --steps 200 --warmup 5 > gpurun_out/bench14.json 2>gpurun_out/bench14.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench14.json'))
for k in ['value','fill_us','apply_us','accept_us','compile_ms','e2e','roofline','clocks']: print(k, d.get(k))
print('cpu', d['cpu_baseline'])
PY

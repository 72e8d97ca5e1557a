mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu 2>&1 | tail -4
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
python bench.py --steps 200 --warmup 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -3 gpurun_out/bench2.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench2.json'))
for k in ['value','fill_us','apply_us','accept_us','compile_ms','masked_fraction','e2e','roofline','clocks','all_accepted']: print(k, d.get(k))
print('cpu', d['cpu_baseline']['value'], d['cpu_baseline']['parity_mismatches'])
PY

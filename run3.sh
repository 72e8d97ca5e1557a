set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -5
python bench.py --steps 100 --warmup 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -5 gpurun_out/bench1.err
cat gpurun_out/bench1.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches1.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
tail -3 gpurun_out/launches1.csv

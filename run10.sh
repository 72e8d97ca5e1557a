GMASK_TRACE=1 python tools/trace_step.py 2>&1 | tail -14
GMASK_TRACE=1 python tools/trace_step.py --warm 2>&1 | tail -6
python -m pytest tests/test_gpu_matcher.py -x -q 2>&1 | grep -E "Error|error|passed|failed" | head -20

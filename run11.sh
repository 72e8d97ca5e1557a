GMASK_TRACE=1 python tools/trace_step.py 2>&1 | tail -12
CUDA_LAUNCH_BLOCKING=1 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_matcher.py -x -q -k "rollback_round_trip" 2>&1 | grep -vE "^=========     (Host|    )" | head -40

export GMASK_NO_BUILD=1
python -m pytest tests/test_gpu_matcher.py -x -q -k "rollback_round_trip" 2>&1 | grep -E "MatcherError|Error|passed|failed" | head -8
CUDA_LAUNCH_BLOCKING=1 compute-sanitizer --tool memcheck --print-limit 3 python -m pytest tests/test_gpu_matcher.py -x -q -k "rollback_round_trip" 2>&1 | grep -vE "^=========     (Host|    )" | head -30

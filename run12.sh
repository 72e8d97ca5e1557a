export GMASK_NO_BUILD=1
python -m pytest tests/test_gpu_matcher.py -x -q -k "rollback_round_trip" 2>&1 | grep -E "Error|error|passed|failed" | head -8
GMASK_VERIFY=1 python paper_2411_15100_b200/build.py --force > /dev/null 2>&1
python -m pytest tests/test_gpu_matcher.py -x -q -k "rollback_round_trip" 2>&1 | grep -E "Error|error|passed|failed" | head -8
python -m pytest tests/test_gpu_matcher.py tests/test_gpu_golden.py -x -q 2>&1 | tail -3

#!/usr/bin/env bash
# compute-sanitizer over the step kernels' GPU tests:
# memcheck, racecheck (shared-memory hazards) and synccheck (barrier misuse)
# on K2 fill, K3 fused fill+apply, K4 accept, K5 step (incl. the deferred
# interning collision path and the overflow walker), K0 apply, K1 build,
# and K5's blended apply (SQL at 128k: keys flagged by the per-key policy).
#   bash tools/sanitize.sh   (on the GPU box; logs in gpurun_out/sanitize_*.log)
set -u
export GMASK_NO_BUILD=1
mkdir -p gpurun_out
TESTS="tests/test_gpu_matcher.py::test_step_kernel_equals_accept_then_fill \
tests/test_gpu_matcher.py::test_fused_fill_apply_equals_separate \
tests/test_gpu_matcher.py::test_k5_small_arena_collisions \
tests/test_gpu_matcher.py::test_rollback_round_trip_and_bounds \
tests/test_gpu_caps.py::test_wide_sets_batched_and_fused \
tests/test_apply.py::test_apply_mixed_chunk_policy_exact \
tests/test_gpu_golden_128k.py::test_k5_batch32_matches_reference[sql]"
for tool in memcheck racecheck synccheck; do
  timeout 3000 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    --log-file gpurun_out/sanitize_$tool.log \
    python -m pytest $TESTS -x -q -p no:cacheprovider > gpurun_out/sanitize_${tool}_pytest.txt 2>&1
  echo "$tool exit $?"
  tail -3 gpurun_out/sanitize_$tool.log
done

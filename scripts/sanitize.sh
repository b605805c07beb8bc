#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over small parity cases of every build.
mkdir -p gpurun_out
export URG_SANITIZE=1
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -q -x -k "test_w1 or test_w2 or test_w3 or test_w4 or test_toy2_all_policies or test_calibration_fixtures or test_cudafree_fixtures or test_cpu_cores_fixtures or test_contention_fixtures or test_packed_two_scenarios_per_warp or test_classical_policies_wide or test_edge_cases" \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
  # per-task executors (R32): the cross-lane hand-over slots in shared memory
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_gpu_executors.py -q -x -k "test_pipeline_cases or test_random_workloads" \
    > gpurun_out/sanitize_te_$tool.log 2>&1
  echo "$tool (executors) rc=$?"; tail -3 gpurun_out/sanitize_te_$tool.log
done

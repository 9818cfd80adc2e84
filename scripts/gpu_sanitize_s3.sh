#!/bin/bash
# compute-sanitizer over the session-3 sampler changes (shared-memory staging of the top
# levels, thread-0 stream position, acq_rel tickets) and the scan's early trigger.
mkdir -p gpurun_out
K="test_random_updates or test_stream_without or test_sharded or test_update_sample or test_toy or test_dqn_full_size_tree or test_ppo_full_size"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_sumtree.py tests/test_gpu_returns.py -q -x -k "$K" > gpurun_out/sanitize_s3_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitize_s3_$tool.log | tail -3
done

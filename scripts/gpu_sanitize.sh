#!/bin/bash
# compute-sanitizer passes over the kernels (small shapes): memcheck, racecheck, synccheck.
mkdir -p gpurun_out
K="(test_sequences or test_sequence_shapes or test_sequence_n_active or test_transition_frames or test_toy_golden or test_random_updates_vs_oracle or test_update_seq or test_col_offset) and not tmapipe and not chunk and not lsu and not pipe14 and not pipe4"
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_gather.py tests/test_gpu_sumtree.py tests/test_gpu_returns.py -q -x -k "$K" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Error|error" gpurun_out/sanitize_$tool.log | tail -4
done

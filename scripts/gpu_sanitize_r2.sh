#!/bin/bash
# compute-sanitizer over the round-2 kernels and changes: the pipelined scans (default and
# variant 9), time-limit entries, fused sequence targets, fused sampling, the transition
# pipeline's armed-sample groups, the min-tree maintenance / rebuild, the exact sequence sum.
mkdir -p gpurun_out
K="(tl_entries and (0- or 9-)) or (discounted_and_gae_random and (0-clipped or 9-clipped)) or fused_targets or gather_sample or pipeline_skipped or pipeline_scalars or min_tree or exact_sum or time_limit_bootstrap"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_gather.py tests/test_gpu_sumtree.py tests/test_gpu_returns.py -q -x -k "$K" > gpurun_out/sanitize_r2_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitize_r2_$tool.log | tail -3
done

#!/bin/bash
# compute-sanitizer over the session-2 kernels: the dynamic-tail sequence gather (every schedule
# shape, fused sampling), the multi-CTA update (both paths, min-tree), the staged fused sampling.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 2400 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_gather_dyn.py tests/test_gpu_sumtree.py tests/test_gpu_gather.py -q -x -k "dynamic_tail or update_seq_vs_oracle or random_updates or live_only or min_tree_maintained or set_q_maxseen or gather_sample" > gpurun_out/sanitize_r2s2_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitize_r2s2_$tool.log | tail -3
done

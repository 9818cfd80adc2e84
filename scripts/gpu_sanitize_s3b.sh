#!/bin/bash
# compute-sanitizer over the session-3 launch-shape / load-order changes: sequence gather
# (4 consumers, setup before the dependency wait), transition pipeline (4 consumers),
# batched per-step |delta| loads in the update, n-step load order.
mkdir -p gpurun_out
python paper_1909_01500_b200/build.py > gpurun_out/build.log 2>&1
K="sequence or transition or r2d2 or dqn or update_seq or nstep or random_updates"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_gather.py tests/test_gpu_sumtree.py tests/test_gpu_returns.py -q -x -k "$K" > gpurun_out/sanitize_s3b_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitize_s3b_$tool.log | tail -3
done

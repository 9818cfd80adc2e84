#!/bin/bash
# compute-sanitizer over the kernels added late in round 1: fused update+sample (grid barrier),
# ring TD, initial-priority pipeline, peer-board sampler/gather (pre-filled peer: the
# sanitizer serialises kernels, so the concurrent-rank tests are left out), cluster scans.
mkdir -p gpurun_out
K="test_update_sample or test_ring_td or test_ring_append_rows or test_pipeline_initial or test_p2p_prefilled or test_ppo_full_size"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_sumtree.py tests/test_gpu_targets.py tests/test_gpu_pipeline.py tests/test_gpu_p2p.py tests/test_gpu_returns.py -q -x -k "$K" > gpurun_out/sanitize_new_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|Error|error" gpurun_out/sanitize_new_$tool.log | tail -4
done

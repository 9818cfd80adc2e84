#!/bin/bash
# Iteration call: GPU tests, tree-staging and PPO-floor A/B probes.
python paper_1909_01500_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for s in 0 1; do RPL_TREE_STAGE=$s timeout 300 python scripts/tree_probe.py > gpurun_out/tree_probe_stage$s.json 2>&1; done
for t in 0 1; do RPL_SCAN_TRIGGER=$t timeout 300 python scripts/ppo_floor_probe.py > gpurun_out/ppo_floor_trig$t.json 2>&1; done
RPL_PDL=0 timeout 300 python scripts/ppo_floor_probe.py > gpurun_out/ppo_floor_nopdl.json 2>&1
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/tree_probe_stage*.json gpurun_out/ppo_floor_*.json

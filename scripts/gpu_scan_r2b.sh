#!/bin/bash
# Scan A/B (round 2, session 2): PPO single-stage shapes x trigger, and the large-size sweep
# for the deeper-pipeline shapes.
mkdir -p gpurun_out
for trig in 1 2; do
  RPL_SCAN_TRIGGER=$trig VARIANTS=0,18,19,20,21,0 timeout 600 python scripts/scan_variants.py > gpurun_out/ppo_var_t$trig.json 2> gpurun_out/ppo_var_t$trig.err
  echo "trigger $trig"; cat gpurun_out/ppo_var_t$trig.json | tr -d '\n '; echo
done
VARIANTS="${SWEEP_VARIANTS:-0 22 23}" bash scripts/gpu_scan_ab.sh

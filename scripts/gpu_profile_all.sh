#!/bin/bash
# Profiles for profiles/: launch list of the bench step (eager), ncu --set full of the
# sequence gather (bench launch config) and of the PPO / tree kernels.
mkdir -p gpurun_out
B="python bench.py --profile --no-graph --steps 20 --warmup 10 --no-secondary --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv \
  --log-file gpurun_out/launches.csv $B > gpurun_out/launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather_seq -s 8 -c 1 \
  -o gpurun_out/prof_gather python bench.py --profile --no-graph --steps 2 --warmup 10 --no-secondary --no-cpu-baseline > gpurun_out/prof_gather.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_nstep|k_tree" -s 6 -c 8 \
  -o gpurun_out/prof_small python scripts/prof_kernels.py > gpurun_out/prof_small.log 2>&1
ls gpurun_out

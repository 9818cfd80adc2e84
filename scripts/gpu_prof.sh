#!/bin/bash
# Profiling call: HBM probes (ceilings for the write-heavy gather), ncu --set full of the
# sequence gather (default and chunked variants) and of the return / tree kernels.
set -x
mkdir -p gpurun_out
timeout 300 python scripts/hbm_probe.py > gpurun_out/hbm_probe.json 2>&1
timeout 300 python scripts/hbm_probe2.py > gpurun_out/hbm_probe2.json 2>&1
timeout 300 python scripts/hbm_probe3.py > gpurun_out/hbm_probe3.json 2>&1
B="python bench.py --profile --no-graph --steps 2 --warmup 10 --no-secondary --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather -s 8 -c 1 -o gpurun_out/prof_gather_v0 $B > gpurun_out/prof_gather_v0.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather -s 8 -c 1 -o gpurun_out/prof_gather_v1 $B --seq-variant 1 > gpurun_out/prof_gather_v1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_scan|k_nstep|k_tree" -s 6 -c 8 -o gpurun_out/prof_small python scripts/prof_kernels.py > gpurun_out/prof_small.log 2>&1
ls -la gpurun_out

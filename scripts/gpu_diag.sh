#!/bin/bash
mkdir -p gpurun_out
VARIANTS=0,5 timeout 600 python scripts/gather_diag.py > gpurun_out/gather_diag.json 2> gpurun_out/gather_diag.err
B="python bench.py --profile --no-graph --steps 2 --warmup 10 --no-secondary --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gather -s 8 -c 1 -o gpurun_out/prof_gather_meta $B > gpurun_out/prof_gather_meta.log 2>&1
cat gpurun_out/gather_diag.json; tail -3 gpurun_out/gather_diag.err

#!/bin/bash
mkdir -p gpurun_out
VARIANTS="e0=-DRPL_PDL_EARLY=0 e1=-DRPL_PDL_EARLY=1" ROUNDS=3 BENCH_ARGS="--steps 400 --fused-sample 1" bash scripts/ab_flags.sh 2>&1 | sed 's/^/fused /'
RPL_NVCC_EXTRA="-DRPL_TRACE -DRPL_PDL_EARLY=1" python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
STEP=fused python scripts/step_trace.py | tr -d '\n '; echo
python paper_1909_01500_b200/build.py --force > /dev/null 2>&1

#!/bin/bash
# PDL early-trigger masks x sampling placement (pair / fused into the gather), same box.
mkdir -p gpurun_out
VARIANTS="e0=-DRPL_PDL_EARLY=0 e4=-DRPL_PDL_EARLY=4 e5=-DRPL_PDL_EARLY=5 e7=-DRPL_PDL_EARLY=7" ROUNDS=2 BENCH_ARGS="--steps 400 --fused-sample 0" bash scripts/ab_flags.sh 2>&1 | sed 's/^/pair /'
VARIANTS="e0=-DRPL_PDL_EARLY=0 e4=-DRPL_PDL_EARLY=4 e5=-DRPL_PDL_EARLY=5" ROUNDS=2 BENCH_ARGS="--steps 400 --fused-sample 1" bash scripts/ab_flags.sh 2>&1 | sed 's/^/fused /'

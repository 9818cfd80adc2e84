#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sumtree.py tests/test_gpu_step.py tests/test_gpu_pipeline.py tests/test_gpu_append.py tests/test_gpu_targets.py -x -q > gpurun_out/pytest_upd.log 2>&1; tail -2 gpurun_out/pytest_upd.log
VARIANTS="s1=-DRPL_UPD_SINGLE=1 s0=-DRPL_UPD_SINGLE=0" ROUNDS=2 BENCH_ARGS="--steps 400 --fused-sample ${FS:-1}" bash scripts/ab_flags.sh
RPL_NVCC_EXTRA="-DRPL_TRACE" python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
STEP=fused python scripts/step_trace.py | tr -d '\n '; echo
python paper_1909_01500_b200/build.py --force > /dev/null 2>&1

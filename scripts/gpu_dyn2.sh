#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gather_dyn.py tests/test_gpu_gather.py tests/test_gpu_step.py -x -q > gpurun_out/pytest_dyn.log 2>&1; tail -3 gpurun_out/pytest_dyn.log
STEP=fused SETTINGS="-1,10,10 88,10,10 88,12,12 80,12,12" python scripts/ab_dyn_sweep.py
STEP=pair SETTINGS="-1,10,10 88,10,10 80,12,12" python scripts/ab_dyn_sweep.py
RPL_NVCC_EXTRA="-DRPL_TRACE" python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
STEADY=1 STEP=fused python scripts/step_trace.py | tr -d '\n '; echo
python paper_1909_01500_b200/build.py --force > /dev/null 2>&1

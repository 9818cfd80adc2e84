#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sumtree.py tests/test_gpu_step.py tests/test_gpu_pipeline.py tests/test_gpu_append.py tests/test_gpu_gather.py -x -q > gpurun_out/pytest_multi.log 2>&1; tail -2 gpurun_out/pytest_multi.log
KNOB=upd_multi A=0 B=1 python scripts/ab_inproc.py
KNOB=upd_multi A=1 B=0 python scripts/ab_inproc.py
BASE=upd_multi=1 KNOB=upd_trigger A=-1 B=2 python scripts/ab_inproc.py
RPL_NVCC_EXTRA="-DRPL_TRACE" python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
STEADY=1 STEP=fused python scripts/step_trace.py | tr -d '\n '; echo
python paper_1909_01500_b200/build.py --force > /dev/null 2>&1

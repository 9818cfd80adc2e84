#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gather_dyn.py tests/test_gpu_gather.py tests/test_gpu_step.py -x -q > gpurun_out/pytest_dyn.log 2>&1; tail -3 gpurun_out/pytest_dyn.log
STEP=pair KNOB=dyn_pct A=100 B=88 python scripts/ab_inproc.py
STEP=pair KNOB=dyn_pct A=80 B=70 python scripts/ab_inproc.py
STEP=pair KNOB=dyn_pct A=80 B=90 python scripts/ab_inproc.py
STEP=pair DYN_ROWS=8 KNOB=dyn_pct A=100 B=80 python scripts/ab_inproc.py
STEP=fused KNOB=dyn_pct A=100 B=80 python scripts/ab_inproc.py
RPL_NVCC_EXTRA="-DRPL_TRACE" python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
STEADY=1 STEP=pair python scripts/step_trace.py | tr -d '\n '; echo
python paper_1909_01500_b200/build.py --force > /dev/null 2>&1

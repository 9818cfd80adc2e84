#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sumtree.py tests/test_gpu_gather.py tests/test_gpu_step.py -x -q > gpurun_out/pytest_trig.log 2>&1; tail -2 gpurun_out/pytest_trig.log
VARIANTS="e0=-DRPL_PDL_EARLY=0 at3=-DRPL_PDL_EARLY=1,-DRPL_UPD_TRIGGER_AT=3" ROUNDS=2 BENCH_ARGS="--steps 400 --fused-sample 1" bash scripts/ab_flags.sh
for v in "-DRPL_PDL_EARLY=1 -DRPL_UPD_TRIGGER_AT=3"; do
  RPL_NVCC_EXTRA="-DRPL_TRACE $v" python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
  echo "$v"; STEP=fused python scripts/step_trace.py | tr -d '\n '; echo
done
python paper_1909_01500_b200/build.py --force > /dev/null 2>&1
